/*
 * qcs_b200.hpp — C++ façade over the C-ABI (qcs_b200.h) in the reference's
 * own types: what a maintainer of the reference (/root/reference/proj, C++20)
 * includes to run its per-gate hot path on a B200.
 *
 * Header-only.  It is compiled INSIDE the reference build: it includes the
 * reference's public headers (qcs/aalc.hpp and what that pulls in) and takes
 * and returns the reference's value types — GateOp, ErrorBoundLadder,
 * RatioThreshold, StateGeometry, StrideBuffer, CompressedBlock,
 * StrideCompressReport, GateRecord, RunMetrics, CircuitProgram.  The class
 * below mirrors qcs::CompressedState (aalc.hpp:110-175) method for method, and
 * the free functions mirror run_program / run_program_on /
 * apply_program_range (aalc.hpp:196-209) and the codec plugin
 * compress / decompress_into (codec.hpp:80-105).  A call site switches by
 * naming qcs::b200:: instead of qcs::.
 *
 * Errors: every QCS_E_* code is rethrown as the reference's exception type
 * (std::invalid_argument, std::out_of_range, CodecError::Kind,
 * CheckpointError::Kind, std::runtime_error); the state is unchanged when a
 * gate fails (aalc.hpp:126-129).  `workers` is accepted and ignored: the
 * reference guarantees results independent of it (aalc.hpp:127-129).
 *
 * Link: -I include -I <reference>/proj/include  -L paper_1811_05140_b200 -lqcs_b200
 * plus the reference library itself (GateOp::validate, ErrorBoundLadder).
 */
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#ifndef QCS_B200_DROPIN_API  // drop-in builds declare the engine API themselves
#include "qcs/aalc.hpp"
#endif
#include "qcs_b200.h"

namespace qcs::b200 {

// ---- errors -----------------------------------------------------------------

/// QCS_E_* -> the reference's exception kinds (codec.hpp:34-52, aalc.hpp:71-90).
[[noreturn]] inline void raise(int rc, const std::string& prefix = {})
{
    const std::string m = prefix + qcs_last_error();
    switch (rc) {
    case QCS_E_INVALID: throw std::invalid_argument(m);
    case QCS_E_RANGE: throw std::out_of_range(m);
    case QCS_E_BAD_MAGIC: throw CodecError(CodecError::Kind::bad_magic, m);
    case QCS_E_TRUNCATED: throw CodecError(CodecError::Kind::truncated, m);
    case QCS_E_UNKNOWN_CODEC: throw CodecError(CodecError::Kind::unknown_codec, m);
    case QCS_E_BAD_VALUE: throw CodecError(CodecError::Kind::bad_value, m);
    default: throw std::runtime_error(m);
    }
}

inline void check(int rc)
{
    if (rc != QCS_OK) raise(rc);
}

// ---- gate descriptors ---------------------------------------------------------

/// GateOp (gate.hpp:43-63) -> qcs_gate_desc; u in UnitaryParts order
/// (gate.cpp:141-151).
inline qcs_gate_desc to_desc(const GateOp& g)
{
    qcs_gate_desc d{};
    d.kind = static_cast<int32_t>(g.kind);
    d.target = g.target;
    d.control = g.control ? *g.control : -1;
    d.flip_index = g.flip_index;
    if (g.unitary) {
        const Unitary2x2& u = *g.unitary;
        const double p[8] = {u.u11.real(), u.u11.imag(), u.u12.real(), u.u12.imag(),
                             u.u21.real(), u.u21.imag(), u.u22.real(), u.u22.imag()};
        std::memcpy(d.u, p, sizeof p);
    }
    return d;
}

// ---- QCS1 block container (codec.hpp:54-74; codec.cpp:369-420) -------------------

namespace detail {

inline void put_le(std::vector<std::uint8_t>& out, const void* v, std::size_t n)
{
    const auto* p = static_cast<const std::uint8_t*>(v);
    out.insert(out.end(), p, p + n);  // x86-64 / aarch64: little-endian
}

inline void append_block(const CompressedBlock& b, std::vector<std::uint8_t>& out)
{
    out.insert(out.end(), {'Q', 'C', 'S', '1'});
    out.push_back(b.codec_id);
    put_le(out, &b.delta, 8);
    put_le(out, &b.scalar_count, 8);
    const std::uint64_t len = b.payload.size();
    put_le(out, &len, 8);
    out.insert(out.end(), b.payload.begin(), b.payload.end());
}

/// One serialized block at bytes[off..]; advances off.  Malformed input has
/// already been rejected by the library.
inline CompressedBlock take_block(const std::uint8_t* bytes, std::size_t& off)
{
    CompressedBlock b;
    b.codec_id = bytes[off + 4];
    std::memcpy(&b.delta, bytes + off + 5, 8);
    std::memcpy(&b.scalar_count, bytes + off + 13, 8);
    std::uint64_t len = 0;
    std::memcpy(&len, bytes + off + 21, 8);
    off += kBlockHeaderBytes;
    b.payload.assign(bytes + off, bytes + off + len);
    off += len;
    return b;
}

inline std::uint64_t now_ns()
{
    return static_cast<std::uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                          std::chrono::steady_clock::now().time_since_epoch())
                                          .count());
}

}  // namespace detail

// ---- codec plugin (codec.hpp:80-105) ----------------------------------------------

/// compress (codec.cpp:252-256) on the device: lossless when bound.delta == 0.
inline CompressedBlock compress(std::span<const double> scalars, ErrorBound bound)
{
    // worst case of the token coder: 9 bytes per scalar + run tokens
    std::uint64_t len = 0;
    std::vector<std::uint8_t> buf(kBlockHeaderBytes + 9 * scalars.size() + 64);
    int rc = qcs_codec_compress(scalars.data(), scalars.size(), bound.delta, buf.data(), buf.size(), &len);
    if (rc == QCS_E_CAPACITY) {
        buf.resize(len);
        rc = qcs_codec_compress(scalars.data(), scalars.size(), bound.delta, buf.data(), buf.size(), &len);
    }
    check(rc);
    std::size_t off = 0;
    return detail::take_block(buf.data(), off);
}

/// decompress_into (codec.cpp:344-360) on the device; out.size() must equal
/// block.scalar_count.
inline void decompress_into(const CompressedBlock& block, std::span<double> out)
{
    std::vector<std::uint8_t> buf;
    detail::append_block(block, buf);
    check(qcs_codec_decompress(buf.data(), buf.size(), out.data(), out.size()));
}

inline std::vector<double> decompress(const CompressedBlock& block)
{
    std::vector<double> out(block.scalar_count);
    b200::decompress_into(block, out);
    return out;
}

// ---- CompressedState (aalc.hpp:110-175) -------------------------------------------

class CompressedState;

struct LoadedState;

class CompressedState {
public:
    using GateResult = qcs::CompressedState::GateResult;

    CompressedState() = default;
    CompressedState(const CompressedState&) = delete;  // owns device arenas
    CompressedState& operator=(const CompressedState&) = delete;
    CompressedState(CompressedState&& o) noexcept : h_(std::exchange(o.h_, nullptr)), geom_(o.geom_) {}
    CompressedState& operator=(CompressedState&& o) noexcept
    {
        if (this != &o) {
            reset();
            h_ = std::exchange(o.h_, nullptr);
            geom_ = o.geom_;
        }
        return *this;
    }
    ~CompressedState() { reset(); }

    /// basis_state (aalc.cpp:140-174) on CUDA device `device`.
    static CompressedState basis_state(const StateGeometry& geom, std::uint64_t basis_index,
                                       int device = 0)
    {
        if (basis_index >= geom.n_amplitudes()) throw std::out_of_range("basis index out of range");
        CompressedState s;
        s.geom_ = geom;
        check(qcs_state_create(geom.n_qubits, geom.stride_bits, basis_index, device, &s.h_));
        return s;
    }

    const StateGeometry& geometry() const { return geom_; }
    qcs_dev_state_t handle() const { return h_; }

    /// apply_gate (aalc.cpp:261-420): validate, plan, decompress -> gate ->
    /// recompress with the ladder, staged commit, lazy renormalisation.
    GateResult apply_gate(const GateOp& gate, const ErrorBoundLadder& ladder, RatioThreshold theta,
                          int /*workers*/ = 0)
    {
        gate.validate(geom_);
        const qcs_gate_desc d = to_desc(gate);
        std::vector<qcs_stride_report> reps(geom_.n_strides());
        std::uint64_t nr = 0;
        double norm = 0.0;
        check(qcs_apply_gate(h_, &d, ladder.bounds.data(), static_cast<int>(ladder.bounds.size()),
                             theta.theta, reps.data(), &nr, &norm));
        GateResult out;
        out.reports.reserve(nr);
        for (std::uint64_t i = 0; i < nr; ++i) {
            StrideCompressReport r;
            r.stride_index = reps[i].stride_index;
            r.chosen_delta = reps[i].chosen_delta;
            r.ratio = reps[i].ratio;
            r.bytes_in = reps[i].bytes_in;
            r.bytes_out = reps[i].bytes_out;
            r.threshold_met = reps[i].threshold_met != 0;
            out.reports.push_back(r);
        }
        out.norm_after = norm;
        return out;
    }

    /// stored_stride / decompress_stride (aalc.cpp:191-209).
    StrideBuffer stored_stride(std::uint64_t j) const { return read(j, false); }
    StrideBuffer decompress_stride(std::uint64_t j) const { return read(j, true); }

    /// to_amplitudes (aalc.cpp:211-223).
    std::vector<Amplitude> to_amplitudes() const
    {
        std::vector<Amplitude> a(geom_.n_amplitudes());
        check(qcs_to_amplitudes(h_, reinterpret_cast<double*>(a.data())));
        return a;
    }

    /// stride_scale (aalc.cpp:225-231).
    double stride_scale(std::uint64_t j) const
    {
        if (j >= geom_.n_strides()) throw std::out_of_range("stride index out of range");
        double sc = 0, ss = 0;
        std::uint64_t a = 0, b = 0;
        check(qcs_stride_info(h_, j, &sc, &ss, &a, &b));
        return sc;
    }

    double norm_sq_tracked() const { return stats().norm; }
    std::uint64_t compressed_bytes() const { return stats().bytes; }
    double min_stride_ratio() const { return stats().min_ratio; }

    /// save (aalc.cpp:466-494): QCKP v1, byte-identical to the reference's.
    void save(const std::string& path, std::uint64_t ladder_fingerprint) const
    {
        // header: "QCKP", version 1, n u32, s u32, fingerprint u64, strides u64 (29 bytes)
        std::uint8_t hdr[29] = {'Q', 'C', 'K', 'P', 1};
        const std::uint32_t n = static_cast<std::uint32_t>(geom_.n_qubits);
        const std::uint32_t s = static_cast<std::uint32_t>(geom_.stride_bits);
        const std::uint64_t ns = geom_.n_strides();
        std::memcpy(hdr + 5, &n, 4);
        std::memcpy(hdr + 9, &s, 4);
        std::memcpy(hdr + 13, &ladder_fingerprint, 8);
        std::memcpy(hdr + 21, &ns, 8);
        std::vector<std::uint8_t> out(hdr, hdr + sizeof hdr);
        std::vector<std::uint8_t> blocks;
        for (std::uint64_t j = 0; j < ns; ++j) {
            std::uint64_t len = 0;
            double sc = 0, ss = 0;
            check(qcs_export_blocks(h_, j, nullptr, 0, &len, &sc, &ss));
            blocks.resize(len);
            check(qcs_export_blocks(h_, j, blocks.data(), len, &len, &sc, &ss));
            detail::put_le(out, &sc, 8);
            detail::put_le(out, &ss, 8);
            out.insert(out.end(), blocks.begin(), blocks.begin() + static_cast<std::ptrdiff_t>(len));
        }
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        if (!f) throw CheckpointError(CheckpointError::Kind::io, "cannot open '" + path + "' for writing");
        f.write(reinterpret_cast<const char*>(out.data()), static_cast<std::streamsize>(out.size()));
        if (!f) throw CheckpointError(CheckpointError::Kind::io, "write failed for '" + path + "'");
    }

    /// load (aalc.cpp:496-586): same validation order and error kinds.
    static LoadedState load(const std::string& path, const std::optional<StateGeometry>& expected = {},
                            int device = 0);

private:
    struct Stats {
        std::uint64_t bytes;
        double min_ratio;
        double norm;
    };
    Stats stats() const
    {
        Stats s{};
        check(qcs_state_stats(h_, &s.bytes, &s.min_ratio, &s.norm));
        return s;
    }
    StrideBuffer read(std::uint64_t j, bool apply_scale) const
    {
        if (j >= geom_.n_strides()) throw std::out_of_range("stride index out of range");
        StrideBuffer b(j, geom_.stride_len());
        check(qcs_read_stride(h_, j, apply_scale ? 1 : 0, b.re.data(), b.im.data()));
        return b;
    }
    void reset()
    {
        if (h_) qcs_state_destroy(h_);
        h_ = nullptr;
    }

    qcs_dev_state_t h_ = nullptr;
    StateGeometry geom_;
};

struct LoadedState {
    CompressedState state;
    std::uint64_t ladder_fingerprint = 0;
};

inline LoadedState CompressedState::load(const std::string& path, const std::optional<StateGeometry>& expected,
                                         int device)
{
    using K = CheckpointError::Kind;
    std::ifstream f(path, std::ios::binary);
    if (!f) throw CheckpointError(K::io, "cannot open '" + path + "' for reading");
    const std::vector<std::uint8_t> data((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (data.size() < 4 || std::memcmp(data.data(), "QCKP", 4) != 0)
        throw CheckpointError(K::bad_magic, "not a checkpoint file");
    if (data.size() < 29) throw CheckpointError(K::truncated, "checkpoint shorter than its header");
    if (data[4] != 1)
        throw CheckpointError(K::version_mismatch, "unsupported checkpoint version " + std::to_string(data[4]));
    std::uint32_t n = 0, s = 0;
    std::uint64_t fp = 0, ns = 0;
    std::memcpy(&n, data.data() + 5, 4);
    std::memcpy(&s, data.data() + 9, 4);
    std::memcpy(&fp, data.data() + 13, 8);
    std::memcpy(&ns, data.data() + 21, 8);
    StateGeometry geom;
    try {
        geom = StateGeometry::make(static_cast<int>(n), static_cast<int>(s));
    } catch (const std::exception& e) {
        throw CheckpointError(K::geometry_mismatch, e.what());
    }
    if (ns != geom.n_strides()) throw CheckpointError(K::geometry_mismatch, "stride count disagrees with geometry");
    if (expected && (expected->n_qubits != geom.n_qubits || expected->stride_bits != geom.stride_bits))
        throw CheckpointError(K::geometry_mismatch, "checkpoint geometry differs from the expected one");
    LoadedState out{CompressedState::basis_state(geom, 0, device), fp};
    std::size_t off = 29;
    for (std::uint64_t j = 0; j < ns; ++j) {
        if (off + 16 > data.size()) throw CheckpointError(K::truncated, "checkpoint ends inside stride header");
        double sc = 0, ss = 0;
        std::memcpy(&sc, data.data() + off, 8);
        std::memcpy(&ss, data.data() + off + 8, 8);
        off += 16;
        const std::size_t start = off;
        for (int b = 0; b < 2; ++b) {
            if (off + kBlockHeaderBytes > data.size())
                throw CheckpointError(K::truncated, "corrupt checkpoint: block header extends past end of data");
            if (std::memcmp(data.data() + off, "QCS1", 4) != 0)
                throw CheckpointError(K::bad_magic, "corrupt checkpoint: bad block magic");
            std::uint64_t cnt = 0, len = 0;
            std::memcpy(&cnt, data.data() + off + 13, 8);
            std::memcpy(&len, data.data() + off + 21, 8);
            off += kBlockHeaderBytes;
            if (len > data.size() - off)
                throw CheckpointError(K::truncated, "corrupt checkpoint: block payload extends past end of data");
            if (cnt != geom.stride_len()) throw CheckpointError(K::geometry_mismatch, "block length disagrees with geometry");
            off += len;
        }
        const int rc = qcs_import_blocks(out.state.h_, j, data.data() + start, off - start, sc, ss);
        if (rc != QCS_OK)
            throw CheckpointError(rc == QCS_E_TRUNCATED ? K::truncated : K::bad_magic,
                                  std::string("corrupt checkpoint: ") + qcs_last_error());
    }
    if (off != data.size()) throw CheckpointError(K::truncated, "trailing bytes after final stride");
    return out;
}

// ---- run drivers (aalc.cpp:588-676) -------------------------------------------------

struct RunResult {
    CompressedState state;
    RunMetrics metrics;
};

/// apply_program_range (aalc.cpp:588-634), batched: the gates are validated
/// up front, queued back to back on the device and synchronised once.
/// GateRecord.elapsed_ns is the gate's device time.  A gate that fails
/// leaves the gates before it applied and throws "gate i (label) failed: ...".
inline RunMetrics apply_program_range(CompressedState& state, const CircuitProgram& program, std::size_t first,
                                      std::size_t last, const ErrorBoundLadder& ladder, RatioThreshold theta,
                                      int /*workers*/ = 0)
{
    if (last > program.gates.size() || first > last) throw std::out_of_range("gate range outside program");
    RunMetrics metrics;
    std::size_t stop = last;
    std::string failure;
    std::vector<qcs_gate_desc> descs;
    descs.reserve(last - first);
    for (std::size_t i = first; i < last; ++i) {
        try {
            program.gates[i].validate(state.geometry());
        } catch (const std::exception& e) {
            stop = i;
            failure = "gate " + std::to_string(i) + " (" + program.gates[i].label + ") failed: " + e.what();
            break;
        }
        descs.push_back(to_desc(program.gates[i]));
    }
    std::vector<qcs_gate_record> recs(descs.size());
    std::uint64_t done = 0;
    int rc = QCS_OK;
    if (!descs.empty())
        rc = qcs_run_program(state.handle(), descs.data(), descs.size(), first, ladder.bounds.data(),
                             static_cast<int>(ladder.bounds.size()), theta.theta, recs.data(), &done);
    metrics.records.reserve(done);
    for (std::uint64_t k = 0; k < done; ++k) {
        const qcs_gate_record& g = recs[k];
        GateRecord r;
        r.gate_index = first + k;
        r.gate_label = program.gates[first + k].label;
        r.stride_count = g.stride_count;
        r.min_ratio = g.min_ratio;
        r.mean_ratio = g.mean_ratio;
        r.max_chosen_delta = g.max_chosen_delta;
        r.bytes_before = g.bytes_before;
        r.bytes_after = g.bytes_after;
        r.elapsed_ns = g.elapsed_ns;
        r.norm_after = g.norm_after;
        metrics.records.push_back(std::move(r));
        metrics.threshold_violations += g.threshold_violations;
        metrics.total_elapsed_ns += g.elapsed_ns;
    }
    if (rc != QCS_OK) {
        const std::size_t i = first + done;
        raise(QCS_E_RUNTIME, "gate " + std::to_string(i) + " (" + program.gates[i].label + ") failed: ");
    }
    if (stop != last) throw std::runtime_error(failure);
    return metrics;
}

/// run_program_on (aalc.cpp:653-676).
inline RunResult run_program_on(CompressedState state, const CircuitProgram& program,
                                const ErrorBoundLadder& ladder, RatioThreshold theta,
                                const RunOptions& options = {})
{
    if (program.n_qubits != state.geometry().n_qubits)
        throw std::invalid_argument("program and state disagree on qubits");
    const std::size_t last =
        options.stop_after ? std::min(*options.stop_after, program.gates.size()) : program.gates.size();
    RunResult result;
    result.metrics.init_min_ratio = state.min_stride_ratio();
    result.metrics.init_bytes = state.compressed_bytes();
    RunMetrics gm = apply_program_range(state, program, options.first_gate, last, ladder, theta, options.workers);
    result.metrics.records = std::move(gm.records);
    result.metrics.threshold_violations = gm.threshold_violations;
    result.metrics.total_elapsed_ns += gm.total_elapsed_ns;
    result.state = std::move(state);
    return result;
}

/// run_program (aalc.cpp:636-651) on CUDA device `device`.
inline RunResult run_program(const CircuitProgram& program, const ErrorBoundLadder& ladder, RatioThreshold theta,
                             const StateGeometry& geom, const RunOptions& options = {}, int device = 0)
{
    if (program.n_qubits != geom.n_qubits) throw std::invalid_argument("program and geometry disagree on qubits");
    const std::uint64_t t0 = detail::now_ns();
    CompressedState state = CompressedState::basis_state(geom, options.basis, device);
    const std::uint64_t init_ns = detail::now_ns() - t0;
    RunResult r = run_program_on(std::move(state), program, ladder, theta, options);
    r.metrics.total_elapsed_ns += init_ns;
    return r;
}

}  // namespace qcs::b200
