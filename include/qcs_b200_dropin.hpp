/*
 * qcs_b200_dropin.hpp — link-level drop-in for the reference's engine API.
 *
 * The reference's hot path lives behind one header, qcs/aalc.hpp (engine:
 * CompressedState, the AALC ladder and the run drivers), plus the codec
 * functions declared in qcs/codec.hpp.  This header re-declares that engine
 * API in namespace qcs, source-compatible with the reference's call sites,
 * and paper_1811_05140_b200/host/qcs_b200_dropin.cpp implements it — and the
 * codec functions of qcs/codec.hpp — on the B200 engine through the C-ABI
 * (qcs_b200.h).  A reference build switches engines by
 *   1. putting a directory whose qcs/aalc.hpp is `#include "qcs_b200_dropin.hpp"`
 *      first on the include path (tests/cpp/dropin/ is one),
 *   2. linking qcs_b200_dropin.cpp + libqcs_b200.so instead of aalc.cpp and
 *      codec.cpp.
 * Its other sources (core, gate, circuit, dense, metrics) and its callers —
 * the acceptance suite, bench_compare, the CLI — compile unchanged
 * (oracle/Makefile builds the reference's own acceptance suite this way).
 *
 * Semantics follow the reference (aalc.hpp:18-211): bit-identical blocks,
 * reports, norms and amplitudes; exceptions of the same types; the state is
 * unchanged when a gate fails.  Differences: GateRecord.elapsed_ns is the
 * gate's device time, `workers` has no meaning on the GPU (results never
 * depend on it, as in the reference), and a CompressedState owns device
 * memory (copies are deep, through the device).
 */
#pragma once
#define QCS_B200_DROPIN_API 1

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "qcs/circuit.hpp"
#include "qcs/codec.hpp"
#include "qcs/core.hpp"
#include "qcs/gate.hpp"
#include "qcs/metrics.hpp"

namespace qcs {

namespace b200 {
class CompressedState;  // include/qcs_b200.hpp
}

// ---- AALC error-bound ladder (aalc.hpp:18-48) -------------------------------
struct ErrorBoundLadder {
    std::vector<double> bounds;  // strictly increasing, finite, >= 0

    static ErrorBoundLadder make(std::vector<double> bounds);
    static ErrorBoundLadder lossless_only() { return make({0.0}); }
    static ErrorBoundLadder default_ladder();  // 0, 1e-7 ... 1e-3
    static ErrorBoundLadder parse(const std::string& text);  // "0,1e-6,..."
    std::uint64_t fingerprint() const;  // FNV-1a over the bounds' bytes
};

// ---- ratio threshold theta (aalc.hpp:50-60) -----------------------------------
struct RatioThreshold {
    double theta = 1.0;
    RatioThreshold() = default;
    explicit RatioThreshold(double t) : theta(t)
    {
        if (!(t >= 1.0)) throw std::invalid_argument("ratio threshold must be >= 1");
    }
};

// ---- per-stride outcome of a ladder pass (aalc.hpp:62-69) ----------------------
struct StrideCompressReport {
    std::uint64_t stride_index = 0;
    double chosen_delta = 0.0;
    double ratio = 0.0;
    std::uint64_t bytes_in = 0;
    std::uint64_t bytes_out = 0;
    bool threshold_met = false;
};

// ---- checkpoint errors (aalc.hpp:71-90) ---------------------------------------
class CheckpointError : public std::runtime_error {
public:
    enum class Kind { bad_magic, version_mismatch, truncated, geometry_mismatch, io };
    CheckpointError(Kind kind, const std::string& msg) : std::runtime_error(msg), kind_(kind) {}
    Kind kind() const { return kind_; }

private:
    Kind kind_;
};

// ---- one stride through the ladder (aalc.hpp:92-102) ---------------------------
struct AdaptiveResult {
    CompressedBlock re;
    CompressedBlock im;
    StrideCompressReport report;
};

AdaptiveResult compress_stride_adaptive(StrideBuffer& buf, const ErrorBoundLadder& ladder, RatioThreshold theta);

struct LoadedState;

// ---- the compressed state, resident on a B200 (aalc.hpp:104-175) ---------------
class CompressedState {
public:
    struct GateResult {
        std::vector<StrideCompressReport> reports;  // reference unit order
        double norm_after = 0.0;
    };

    CompressedState();
    CompressedState(const CompressedState& other);
    CompressedState(CompressedState&& other) noexcept;
    CompressedState& operator=(const CompressedState& other);
    CompressedState& operator=(CompressedState&& other) noexcept;
    ~CompressedState();

    static CompressedState basis_state(const StateGeometry& geom, std::uint64_t basis_index);

    const StateGeometry& geometry() const { return geom_; }

    GateResult apply_gate(const GateOp& gate, const ErrorBoundLadder& ladder, RatioThreshold theta,
                          int workers = 0);

    StrideBuffer stored_stride(std::uint64_t stride_index) const;
    StrideBuffer decompress_stride(std::uint64_t stride_index) const;
    std::vector<Amplitude> to_amplitudes() const;
    double stride_scale(std::uint64_t stride_index) const;
    double norm_sq_tracked() const;
    std::uint64_t compressed_bytes() const;
    double min_stride_ratio() const;

    void save(const std::string& path, std::uint64_t ladder_fingerprint) const;
    static LoadedState load(const std::string& path, const std::optional<StateGeometry>& expected = {});

    /// The B200 state behind this object (null for a default-constructed one).
    b200::CompressedState* device_state() const { return impl_.get(); }

private:
    friend RunMetrics apply_program_range(CompressedState&, const CircuitProgram&, std::size_t, std::size_t,
                                          const ErrorBoundLadder&, RatioThreshold, int);
    explicit CompressedState(std::unique_ptr<b200::CompressedState> impl);
    b200::CompressedState& dev() const;

    std::unique_ptr<b200::CompressedState> impl_;
    StateGeometry geom_;
};

struct LoadedState {
    CompressedState state;
    std::uint64_t ladder_fingerprint = 0;
};

// ---- run drivers (aalc.hpp:182-209) ---------------------------------------------
struct RunOptions {
    std::uint64_t basis = 0;
    int workers = 0;
    std::size_t first_gate = 0;
    std::optional<std::size_t> stop_after;
};

struct RunResult {
    CompressedState state;
    RunMetrics metrics;
};

RunMetrics apply_program_range(CompressedState& state, const CircuitProgram& program, std::size_t first,
                               std::size_t last, const ErrorBoundLadder& ladder, RatioThreshold theta,
                               int workers = 0);

RunResult run_program(const CircuitProgram& program, const ErrorBoundLadder& ladder, RatioThreshold theta,
                      const StateGeometry& geom, const RunOptions& options = {});

RunResult run_program_on(CompressedState state, const CircuitProgram& program, const ErrorBoundLadder& ladder,
                         RatioThreshold theta, const RunOptions& options = {});

}  // namespace qcs
