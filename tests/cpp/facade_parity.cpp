// C++ drop-in parity driver (test infrastructure).
//
// Runs the same programs through the UNMODIFIED reference (qcs::run_program,
// aalc.cpp:636-676, linked from oracle/_ref) and through the B200 engine via
// the C++ façade (include/qcs_b200.hpp, qcs::b200::run_program) — both fed the
// reference's own GateOp / ErrorBoundLadder / circuit builders — and compares
// everything the reference exposes: every GateRecord field except the wall
// time, the amplitudes, every stored stride, scales, state statistics,
// QCKP checkpoint bytes, the codec plugin's blocks and the error behaviour.
//
// Prints one PASS/FAIL line per case like the reference's acceptance suite
// (tests/acceptance.cpp) and exits with the number of failures.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>
#include <string>
#include <vector>

#include "qcs_b200.hpp"

namespace {

int g_fail = 0;

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

void report(const std::string& name, const std::string& err)
{
    if (err.empty()) {
        std::printf("PASS %s\n", name.c_str());
    } else {
        std::printf("FAIL %s: %s\n", name.c_str(), err.c_str());
        ++g_fail;
    }
}

std::string cmp_records(const qcs::RunMetrics& a, const qcs::RunMetrics& b)
{
    if (a.records.size() != b.records.size()) return "record count";
    for (std::size_t i = 0; i < a.records.size(); ++i) {
        const auto &x = a.records[i], &y = b.records[i];
        const std::string at = " at gate " + std::to_string(i);
        if (x.gate_index != y.gate_index || x.gate_label != y.gate_label) return "index/label" + at;
        if (x.stride_count != y.stride_count) return "stride_count" + at;
        if (!same_bits(x.min_ratio, y.min_ratio)) return "min_ratio" + at;
        if (!same_bits(x.mean_ratio, y.mean_ratio)) return "mean_ratio" + at;
        if (!same_bits(x.max_chosen_delta, y.max_chosen_delta)) return "max_chosen_delta" + at;
        if (x.bytes_before != y.bytes_before || x.bytes_after != y.bytes_after) return "bytes" + at;
        if (!same_bits(x.norm_after, y.norm_after)) return "norm_after" + at;
    }
    if (a.threshold_violations != b.threshold_violations) return "threshold_violations";
    if (!same_bits(a.init_min_ratio, b.init_min_ratio) || a.init_bytes != b.init_bytes) return "init stats";
    return {};
}

template <class S>
std::string cmp_state(const qcs::CompressedState& r, const S& g)
{
    const auto ar = r.to_amplitudes();
    const auto ag = g.to_amplitudes();
    if (ar.size() != ag.size() || std::memcmp(ar.data(), ag.data(), ar.size() * sizeof(ar[0])) != 0)
        return "amplitudes";
    if (r.compressed_bytes() != g.compressed_bytes()) return "compressed_bytes";
    if (!same_bits(r.min_stride_ratio(), g.min_stride_ratio())) return "min_stride_ratio";
    if (!same_bits(r.norm_sq_tracked(), g.norm_sq_tracked())) return "norm_sq_tracked";
    const auto& geom = r.geometry();
    for (std::uint64_t j = 0; j < geom.n_strides(); ++j) {
        if (!same_bits(r.stride_scale(j), g.stride_scale(j))) return "stride_scale " + std::to_string(j);
        const auto br = r.stored_stride(j), bg = g.stored_stride(j);
        if (br.re != bg.re || br.im != bg.im) return "stored_stride " + std::to_string(j);
    }
    return {};
}

std::vector<std::uint8_t> slurp(const std::string& p)
{
    std::ifstream f(p, std::ios::binary);
    return {std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>()};
}

void run_case(const std::string& name, const qcs::CircuitProgram& prog, int s, std::uint64_t basis,
              const qcs::ErrorBoundLadder& ladder, double theta)
{
    const auto geom = qcs::StateGeometry::make(prog.n_qubits, s);
    qcs::RunOptions opt;
    opt.basis = basis;
    opt.workers = 4;
    std::string err;
    try {
        auto ref = qcs::run_program(prog, ladder, qcs::RatioThreshold(theta), geom, opt);
        auto gpu = qcs::b200::run_program(prog, ladder, qcs::RatioThreshold(theta), geom, opt);
        err = cmp_records(ref.metrics, gpu.metrics);
        if (err.empty()) err = cmp_state(ref.state, gpu.state);
    } catch (const std::exception& e) {
        err = std::string("exception: ") + e.what();
    }
    report(name, err);
}

// save at the midpoint: both engines write the same QCKP bytes; the B200
// engine loads the reference's file and finishes bit-identically.
void checkpoint_case(const qcs::CircuitProgram& prog, int s, std::uint64_t basis, const qcs::ErrorBoundLadder& ladder)
{
    std::string err;
    try {
        const auto geom = qcs::StateGeometry::make(prog.n_qubits, s);
        const std::size_t mid = prog.gates.size() / 2;
        qcs::RunOptions a;
        a.basis = basis;
        a.stop_after = mid;
        auto ref = qcs::run_program(prog, ladder, qcs::RatioThreshold(1.0), geom, a);
        auto gpu = qcs::b200::run_program(prog, ladder, qcs::RatioThreshold(1.0), geom, a);
        const std::string pr = "/tmp/qcs_facade_ref.qckp", pg = "/tmp/qcs_facade_gpu.qckp";
        ref.state.save(pr, ladder.fingerprint());
        gpu.state.save(pg, ladder.fingerprint());
        if (slurp(pr) != slurp(pg)) err = "checkpoint bytes differ";
        if (err.empty()) {
            auto lr = qcs::CompressedState::load(pr);
            auto lg = qcs::b200::CompressedState::load(pr, geom);
            if (lg.ladder_fingerprint != lr.ladder_fingerprint) err = "fingerprint";
            qcs::RunOptions b;
            b.first_gate = mid;
            auto r2 = qcs::run_program_on(std::move(lr.state), prog, ladder, qcs::RatioThreshold(1.0), b);
            auto g2 = qcs::b200::run_program_on(std::move(lg.state), prog, ladder, qcs::RatioThreshold(1.0), b);
            if (err.empty()) err = cmp_records(r2.metrics, g2.metrics);
            if (err.empty()) err = cmp_state(r2.state, g2.state);
        }
        std::remove(pr.c_str());
        std::remove(pg.c_str());
    } catch (const std::exception& e) {
        err = std::string("exception: ") + e.what();
    }
    report("checkpoint save/load/resume (QCKP bytes identical)", err);
}

void codec_case()
{
    std::string err;
    std::mt19937_64 rng(11);
    std::normal_distribution<double> nd(0.0, 1e-3);
    for (double delta : {0.0, 1e-7, 9.765625e-7, 1e-4, 1e-2}) {
        std::vector<double> x(3000 + 17);
        double w = 0;
        for (auto& v : x) {
            w += nd(rng);
            v = w;
        }
        x[100] = 0.0;
        x[101] = -0.0;
        for (int k = 200; k < 900; ++k) x[k] = 0.25;
        const auto rb = qcs::compress(x, qcs::ErrorBound(delta));
        const auto gb = qcs::b200::compress(x, qcs::ErrorBound(delta));
        if (rb.codec_id != gb.codec_id || !same_bits(rb.delta, gb.delta) || rb.scalar_count != gb.scalar_count ||
            rb.payload != gb.payload) {
            err = "block differs at delta " + std::to_string(delta);
            break;
        }
        std::vector<double> yr(x.size()), yg(x.size());
        qcs::decompress_into(rb, yr);
        qcs::b200::decompress_into(rb, yg);
        if (yr != yg) {
            err = "decoded values differ at delta " + std::to_string(delta);
            break;
        }
    }
    if (err.empty()) {  // corrupt input: same CodecError kind
        auto blk = qcs::compress(std::vector<double>(64, 0.5), qcs::ErrorBound(1e-3));
        blk.payload.resize(blk.payload.size() / 2);
        int kr = -1, kg = -2;
        std::vector<double> out(64);
        try {
            qcs::decompress_into(blk, out);
        } catch (const qcs::CodecError& e) {
            kr = static_cast<int>(e.kind());
        }
        try {
            qcs::b200::decompress_into(blk, out);
        } catch (const qcs::CodecError& e) {
            kg = static_cast<int>(e.kind());
        }
        if (kr != kg) err = "CodecError kind differs on a truncated block";
    }
    report("codec plugin compress/decompress_into (blocks identical, 5 bounds)", err);
}

// a gate that fails leaves the state unchanged and throws the same type
void error_case()
{
    std::string err;
    const auto geom = qcs::StateGeometry::make(8, 5);
    auto ref = qcs::CompressedState::basis_state(geom, 77);
    auto gpu = qcs::b200::CompressedState::basis_state(geom, 77);
    const auto lad = qcs::ErrorBoundLadder::make({0.0, 1e-5});
    const auto h = qcs::GateOp::single(qcs::Unitary2x2::hadamard(), 6, "h");
    ref.apply_gate(h, lad, qcs::RatioThreshold(2.0));
    gpu.apply_gate(h, lad, qcs::RatioThreshold(2.0));
    qcs::GateOp bad = qcs::GateOp::single(qcs::Unitary2x2::hadamard(), 9, "h9");
    bool tr = false, tg = false;
    try {
        ref.apply_gate(bad, lad, qcs::RatioThreshold(2.0));
    } catch (const std::out_of_range&) {
        tr = true;
    } catch (const std::invalid_argument&) {
        tr = true;
    }
    try {
        gpu.apply_gate(bad, lad, qcs::RatioThreshold(2.0));
    } catch (const std::out_of_range&) {
        tg = true;
    } catch (const std::invalid_argument&) {
        tg = true;
    }
    if (tr != tg || !tr) err = "exception type differs";
    if (err.empty()) err = cmp_state(ref, gpu);
    bool rr = false, rg = false;
    try {
        (void)qcs::CompressedState::basis_state(geom, 256);
    } catch (const std::out_of_range&) {
        rr = true;
    }
    try {
        (void)qcs::b200::CompressedState::basis_state(geom, 256);
    } catch (const std::out_of_range&) {
        rg = true;
    }
    if (err.empty() && rr != rg) err = "basis_state range error differs";
    report("error atomicity and exception types", err);
}

std::string read_text(const std::string& p)
{
    std::ifstream f(p);
    return {std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>()};
}

}  // namespace

int main(int argc, char** argv)
{
    const std::string golden = argc > 1 ? argv[1] : "tests/golden/circuits";
    const double p20 = 9.5367431640625e-07;  // 2^-20
    run_case("QFT-12 s=8 single pow2 level", qcs::build_qft(12), 8, 1234, qcs::ErrorBoundLadder::make({p20}), 1.0);
    run_case("QFT-12 s=8 decimal bound 1e-6", qcs::build_qft(12), 8, 99, qcs::ErrorBoundLadder::make({1e-6}), 1.0);
    run_case("QFT-14 s=10 default ladder theta=16", qcs::build_qft(14), 10, 5, qcs::ErrorBoundLadder::default_ladder(),
             16.0);
    run_case("QFT-10 s=10 lossless", qcs::build_qft(10), 10, 3, qcs::ErrorBoundLadder::lossless_only(), 1.0);
    run_case("Grover-12 (flip + reflect_mean) s=8 default ladder theta=32", qcs::build_grover(12, 1000), 8, 0,
             qcs::ErrorBoundLadder::default_ladder(), 32.0);
    run_case("random-10 x 300 gates s=5 ladder {0,1e-6,1e-4} theta=4", qcs::build_random(10, 300, 42), 5, 17,
             qcs::ErrorBoundLadder::make({0.0, 1e-6, 1e-4}), 4.0);
    for (const char* f : {"grid3x3_pow2.txt", "grover12_gates_pow2.txt"}) {
        const std::string text = read_text(golden + "/" + f);
        if (text.empty()) {
            report(std::string("parsed ") + f, "file not found under " + golden);
            continue;
        }
        const auto prog = qcs::parse_circuit(text, f);
        run_case(std::string("parsed ") + f + " s=" + std::to_string(prog.n_qubits - 3), prog, prog.n_qubits - 3, 7,
                 qcs::ErrorBoundLadder::make({p20}), 1.0);
    }
    checkpoint_case(qcs::build_qft(12), 7, 321, qcs::ErrorBoundLadder::make({p20}));
    codec_case();
    error_case();
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
