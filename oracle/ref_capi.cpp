// Thin extern "C" wrapper over the *unmodified* reference library (qcsim,
// /root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libqcsref.so.  TEST INFRASTRUCTURE ONLY: it is the checker that
// pins oracle/qcs_oracle.c and generates tests/golden/, and bench.py's
// `--impl reference` arm times it.  Nothing in the product path loads it.
//
// Every entry point calls only public reference API:
//   compress / decompress_into / serialize_block / parse_block  (codec.hpp:80-105)
//   parse_circuit / print_circuit / build_qft / build_grover / build_random
//                                                            (circuit.hpp:47-70)
//   run_program / CompressedState::{to_amplitudes, compressed_bytes,
//   min_stride_ratio, norm_sq_tracked, stride_scale}           (aalc.hpp:110-209)
//   run_dense / fidelity                                        (dense.hpp)
//   emit_csv                                                    (metrics.hpp:66)

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "qcs/aalc.hpp"
#include "qcs/circuit.hpp"
#include "qcs/codec.hpp"
#include "qcs/dense.hpp"
#include "qcs/metrics.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg)
{
    g_err = msg;
    return code;
}

// Return-code convention shared with include/qcs_b200.h (QCS_E_*).
int classify(const std::exception& e)
{
    if (auto* c = dynamic_cast<const qcs::CodecError*>(&e)) {
        switch (c->kind()) {
            case qcs::CodecError::Kind::bad_magic: return 10;
            case qcs::CodecError::Kind::truncated: return 11;
            case qcs::CodecError::Kind::unknown_codec: return 12;
            case qcs::CodecError::Kind::bad_value: return 13;
        }
    }
    if (dynamic_cast<const std::out_of_range*>(&e)) return 3;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 2;
    return 1;
}

int copy_text(const std::string& s, char* out, std::uint64_t cap, std::uint64_t* len)
{
    if (len) *len = s.size();
    if (!out) return 0;
    if (s.size() + 1 > cap) return fail(4, "output buffer too small");
    std::memcpy(out, s.data(), s.size());
    out[s.size()] = '\0';
    return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// Serialized QCS1 block (29-byte header + payload) of compress(x, delta).
int ref_codec_compress(const double* x, std::uint64_t n, double delta,
                       std::uint8_t* out, std::uint64_t cap, std::uint64_t* len)
{
    try {
        const qcs::CompressedBlock b =
            qcs::compress(std::span<const double>(x, n), qcs::ErrorBound(delta));
        const std::vector<std::uint8_t> bytes = qcs::serialize_block(b);
        *len = bytes.size();
        if (out) {
            if (bytes.size() > cap) return fail(4, "output buffer too small");
            std::memcpy(out, bytes.data(), bytes.size());
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// Parses one serialized block and decodes it into out[n].
int ref_codec_decompress(const std::uint8_t* blk, std::uint64_t len, double* out,
                         std::uint64_t n)
{
    try {
        std::size_t off = 0;
        const qcs::CompressedBlock b =
            qcs::parse_block(std::span<const std::uint8_t>(blk, len), off);
        if (b.scalar_count != n) return fail(2, "scalar count mismatch");
        qcs::decompress_into(b, std::span<double>(out, n));
        return 0;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// Text of a reference-built circuit: kind 0 = build_qft(n),
// 1 = build_grover(n, arg, iters), 2 = build_random(n, iters, arg).
int ref_builtin_circuit(int kind, int n, std::uint64_t arg, int iters, char* out,
                        std::uint64_t cap, std::uint64_t* len)
{
    try {
        qcs::CircuitProgram p;
        if (kind == 0) p = qcs::build_qft(n);
        else if (kind == 1) p = qcs::build_grover(n, arg, iters);
        else p = qcs::build_random(n, iters, arg);
        return copy_text(qcs::print_circuit(p), out, cap, len);
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// run_program on a circuit given in the reference text format.
//   stop_after < 0 runs the whole program.
//   csv (optional) receives emit_csv(records).
//   amps (optional) receives to_amplitudes() as interleaved re/im doubles.
//   summary[10]: gate-loop ns, amplitude updates (sum bytes_before/16),
//     init_min_ratio, threshold_violations, compressed_bytes,
//     min_stride_ratio, norm_sq_tracked, overall_min_ratio, n_records,
//     wall ns of run_program (incl. basis_state).
int ref_run(const char* circuit_text, int stride_bits, std::uint64_t basis,
            const double* ladder, int n_levels, double theta, int workers,
            std::int64_t stop_after, char* csv, std::uint64_t csv_cap,
            std::uint64_t* csv_len, double* amps, double* summary)
{
    try {
        const qcs::CircuitProgram p = qcs::parse_circuit(circuit_text);
        const qcs::StateGeometry geom = qcs::StateGeometry::make(p.n_qubits, stride_bits);
        const qcs::ErrorBoundLadder lad = qcs::ErrorBoundLadder::make(
            std::vector<double>(ladder, ladder + n_levels));
        qcs::RunOptions opt;
        opt.basis = basis;
        opt.workers = workers;
        if (stop_after >= 0) opt.stop_after = static_cast<std::size_t>(stop_after);
        const auto t0 = std::chrono::steady_clock::now();
        const qcs::RunResult r =
            qcs::run_program(p, lad, qcs::RatioThreshold(theta), geom, opt);
        const auto t1 = std::chrono::steady_clock::now();
        std::uint64_t loop_ns = 0, upd = 0;
        for (const qcs::GateRecord& g : r.metrics.records) {
            loop_ns += g.elapsed_ns;
            upd += g.bytes_before / 16;
        }
        if (summary) {
            summary[0] = static_cast<double>(loop_ns);
            summary[1] = static_cast<double>(upd);
            summary[2] = r.metrics.init_min_ratio;
            summary[3] = static_cast<double>(r.metrics.threshold_violations);
            summary[4] = static_cast<double>(r.state.compressed_bytes());
            summary[5] = r.state.min_stride_ratio();
            summary[6] = r.state.norm_sq_tracked();
            summary[7] = r.metrics.overall_min_ratio();
            summary[8] = static_cast<double>(r.metrics.records.size());
            summary[9] = static_cast<double>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
        }
        if (amps) {
            const std::vector<qcs::Amplitude> a = r.state.to_amplitudes();
            for (std::size_t i = 0; i < a.size(); ++i) {
                amps[2 * i] = a[i].real();
                amps[2 * i + 1] = a[i].imag();
            }
        }
        if (csv || csv_len) {
            int rc = copy_text(qcs::emit_csv(r.metrics.records), csv, csv_cap, csv_len);
            if (rc) return rc;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// Dense serial simulation (run_dense) of the circuit; amps interleaved re/im.
int ref_dense(const char* circuit_text, std::uint64_t basis, double* amps)
{
    try {
        const qcs::CircuitProgram p = qcs::parse_circuit(circuit_text);
        const qcs::DenseState d = qcs::run_dense(p, basis, 30);
        for (std::size_t i = 0; i < d.amplitudes.size(); ++i) {
            amps[2 * i] = d.amplitudes[i].real();
            amps[2 * i + 1] = d.amplitudes[i].imag();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// Persistent reference state for windowed timing (bench.py --impl reference):
// CompressedState::basis_state then apply_program_range over [first, last).
struct RefState {
    qcs::CircuitProgram prog;
    qcs::CompressedState state;
};

void* ref_state_create(const char* circuit_text, int stride_bits, std::uint64_t basis)
{
    try {
        auto* r = new RefState();
        r->prog = qcs::parse_circuit(circuit_text);
        r->state = qcs::CompressedState::basis_state(
            qcs::StateGeometry::make(r->prog.n_qubits, stride_bits), basis);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_state_destroy(void* h) { delete static_cast<RefState*>(h); }

// summary[4]: sum of GateRecord.elapsed_ns, amplitude updates, min ratio,
// norm_after of the last gate.
int ref_state_apply(void* h, std::uint64_t first, std::uint64_t last, const double* ladder,
                    int n_levels, double theta, int workers, double* summary)
{
    try {
        auto* r = static_cast<RefState*>(h);
        const qcs::ErrorBoundLadder lad = qcs::ErrorBoundLadder::make(
            std::vector<double>(ladder, ladder + n_levels));
        const qcs::RunMetrics m = qcs::apply_program_range(
            r->state, r->prog, first, last, lad, qcs::RatioThreshold(theta), workers);
        std::uint64_t ns = 0, upd = 0;
        double mn = 1e300, norm = 0.0;
        for (const qcs::GateRecord& g : m.records) {
            ns += g.elapsed_ns;
            upd += g.bytes_before / 16;
            mn = std::min(mn, g.min_ratio);
            norm = g.norm_after;
        }
        summary[0] = static_cast<double>(ns);
        summary[1] = static_cast<double>(upd);
        summary[2] = mn;
        summary[3] = norm;
        return 0;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// ref_state_apply plus the per-gate records as emit_csv text (parity tests).
int ref_state_apply_csv(void* h, std::uint64_t first, std::uint64_t last, const double* ladder,
                        int n_levels, double theta, int workers, char* csv, std::uint64_t cap,
                        std::uint64_t* len)
{
    try {
        auto* r = static_cast<RefState*>(h);
        const qcs::ErrorBoundLadder lad = qcs::ErrorBoundLadder::make(
            std::vector<double>(ladder, ladder + n_levels));
        const qcs::RunMetrics m = qcs::apply_program_range(
            r->state, r->prog, first, last, lad, qcs::RatioThreshold(theta), workers);
        return copy_text(qcs::emit_csv(m.records), csv, cap, len);
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// to_amplitudes of a persistent state (interleaved re/im).
int ref_state_amplitudes(void* h, double* amps)
{
    try {
        const std::vector<qcs::Amplitude> a = static_cast<RefState*>(h)->state.to_amplitudes();
        for (std::size_t i = 0; i < a.size(); ++i) {
            amps[2 * i] = a[i].real();
            amps[2 * i + 1] = a[i].imag();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

// A persistent state holding a closed-form intermediate state of the circuit
// (bench.py's late-QFT window, tests/test_gpu_window.py): amplitude
//   a_y = amp * lo[y mod L] * hi[y / L]   (complex; zero where (y & zmask) != zval)
// computed with the same IEEE operations, in the same order, as the GPU arm's
// generator (t = hr*lr - hi*li, u = hr*li + hi*lr, then amp*t, amp*u), so both
// arms start from bit-identical amplitudes.  Every stride goes through the
// reference's compress_stride_adaptive (aalc.cpp:117-138); the result is written
// as a QCKP v1 checkpoint in the reference's format (aalc.cpp:466-494: scale 1,
// sum_sq = StrideBuffer::sum_sq of the decoded blocks, as stored_sum_sq does,
// aalc.cpp:46-52) and read back with CompressedState::load (aalc.cpp:496-586).
void* ref_state_from_tables(const char* circuit_text, int stride_bits, const double* lo_re,
                            const double* lo_im, const double* hi_re, const double* hi_im,
                            double amp, std::uint64_t zmask, std::uint64_t zval,
                            const double* ladder, int n_levels, double theta, const char* path,
                            int workers)
{
    try {
        auto* r = new RefState();
        r->prog = qcs::parse_circuit(circuit_text);
        const qcs::StateGeometry geom = qcs::StateGeometry::make(r->prog.n_qubits, stride_bits);
        const qcs::ErrorBoundLadder lad = qcs::ErrorBoundLadder::make(
            std::vector<double>(ladder, ladder + n_levels));
        const std::uint64_t L = geom.stride_len(), NS = geom.n_strides();
        std::vector<std::vector<std::uint8_t>> body(NS);
        const int nt = workers > 0 ? workers : ref_max_threads();
#pragma omp parallel for schedule(dynamic) num_threads(nt)
        for (std::int64_t jj = 0; jj < static_cast<std::int64_t>(NS); ++jj) {
            const std::uint64_t j = static_cast<std::uint64_t>(jj);
            qcs::StrideBuffer buf(j, L);
            for (std::uint64_t e = 0; e < L; ++e) {
                const std::uint64_t y = j * L + e;
                if ((y & zmask) != zval) continue;  // exact +0.0
                const double t = hi_re[j] * lo_re[e] - hi_im[j] * lo_im[e];
                const double u = hi_re[j] * lo_im[e] + hi_im[j] * lo_re[e];
                buf.re[e] = amp * t;
                buf.im[e] = amp * u;
            }
            const qcs::AdaptiveResult a =
                qcs::compress_stride_adaptive(buf, lad, qcs::RatioThreshold(theta));
            qcs::decompress_into(a.re, buf.re);
            qcs::decompress_into(a.im, buf.im);
            const double ss = buf.sum_sq();
            const double one = 1.0;
            std::vector<std::uint8_t>& o = body[j];
            for (double v : {one, ss}) {
                std::uint64_t w;
                std::memcpy(&w, &v, 8);
                for (int i = 0; i < 8; ++i) o.push_back(static_cast<std::uint8_t>(w >> (8 * i)));
            }
            qcs::serialize_block_append(a.re, o);
            qcs::serialize_block_append(a.im, o);
        }
        {
            std::ofstream f(path, std::ios::binary | std::ios::trunc);
            std::vector<std::uint8_t> hdr = {'Q', 'C', 'K', 'P', 1};
            auto u32 = [&](std::uint32_t v) { for (int i = 0; i < 4; ++i) hdr.push_back(static_cast<std::uint8_t>(v >> (8 * i))); };
            auto u64 = [&](std::uint64_t v) { for (int i = 0; i < 8; ++i) hdr.push_back(static_cast<std::uint8_t>(v >> (8 * i))); };
            u32(static_cast<std::uint32_t>(geom.n_qubits));
            u32(static_cast<std::uint32_t>(geom.stride_bits));
            u64(lad.fingerprint());
            u64(NS);
            f.write(reinterpret_cast<const char*>(hdr.data()), static_cast<std::streamsize>(hdr.size()));
            for (auto& b : body) {
                f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
                std::vector<std::uint8_t>().swap(b);
            }
            if (!f) throw std::runtime_error(std::string("cannot write ") + path);
        }
        r->state = std::move(qcs::CompressedState::load(path, geom).state);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int ref_state_stats(void* h, double* out)
{
    auto* r = static_cast<RefState*>(h);
    out[0] = static_cast<double>(r->state.compressed_bytes());
    out[1] = r->state.min_stride_ratio();
    out[2] = r->state.norm_sq_tracked();
    return 0;
}

}  // extern "C"
