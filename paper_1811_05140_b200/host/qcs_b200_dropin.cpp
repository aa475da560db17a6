// Link-level drop-in for the reference's engine and codec API on the B200
// (declarations: include/qcs_b200_dropin.hpp for aalc.hpp's API, the
// reference's own qcs/codec.hpp for the codec).  Everything here is host
// glue over the C-ABI (include/qcs_b200.h) through the C++ façade
// (include/qcs_b200.hpp): the compute runs in libqcs_b200.so.  Each function
// cites the reference definition whose contract it keeps.
#include "qcs_b200_dropin.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <sstream>

#include "qcs_b200.hpp"

namespace qcs {

// ============================== codec (codec.hpp) ==============================

// codec.cpp:111-116
ErrorBound::ErrorBound(double d) : delta(d)
{
    if (!(d >= 0.0) || !std::isfinite(d)) throw std::invalid_argument("error bound must be finite and >= 0");
}

// codec.cpp:118-147 — lossless zero-word run coder, on the device
CompressedBlock compress_lossless(std::span<const double> scalars)
{
    return b200::compress(scalars, ErrorBound());
}

// codec.cpp:206-250 — previous-value predictor + token coder, on the device
CompressedBlock compress_lossy(std::span<const double> scalars, ErrorBound bound)
{
    if (!(bound.delta > 0.0)) throw CodecError(CodecError::Kind::bad_value, "lossy compression requires delta > 0");
    return b200::compress(scalars, bound);
}

// codec.cpp:252-256
CompressedBlock compress(std::span<const double> scalars, ErrorBound bound)
{
    return b200::compress(scalars, bound);
}

// codec.cpp:344-360
void decompress_into(const CompressedBlock& block, std::span<double> out)
{
    if (out.size() != block.scalar_count) throw std::invalid_argument("output span does not match scalar count");
    if (block.codec_id != kCodecLossless && block.codec_id != kCodecLossy)
        throw CodecError(CodecError::Kind::unknown_codec, "unknown codec id " + std::to_string(block.codec_id));
    b200::decompress_into(block, out);
}

std::vector<double> decompress(const CompressedBlock& block)
{
    std::vector<double> out(block.scalar_count);
    qcs::decompress_into(block, out);
    return out;
}

// codec.cpp:369-389 — the 29-byte QCS1 container
void serialize_block_append(const CompressedBlock& block, std::vector<std::uint8_t>& out)
{
    b200::detail::append_block(block, out);
}

std::vector<std::uint8_t> serialize_block(const CompressedBlock& block)
{
    std::vector<std::uint8_t> out;
    out.reserve(block.total_bytes());
    b200::detail::append_block(block, out);
    return out;
}

// codec.cpp:391-420 (same checks, same error kinds, same order)
CompressedBlock parse_block(std::span<const std::uint8_t> bytes, std::size_t& offset)
{
    if (offset + kBlockHeaderBytes > bytes.size())
        throw CodecError(CodecError::Kind::truncated, "block header extends past end of data");
    const std::uint8_t* p = bytes.data() + offset;
    if (std::memcmp(p, "QCS1", 4) != 0) throw CodecError(CodecError::Kind::bad_magic, "bad block magic");
    if (p[4] != kCodecLossless && p[4] != kCodecLossy)
        throw CodecError(CodecError::Kind::unknown_codec, "unknown codec id " + std::to_string(p[4]));
    std::uint64_t len = 0;
    std::memcpy(&len, p + 21, 8);
    if (offset + kBlockHeaderBytes + len > bytes.size())
        throw CodecError(CodecError::Kind::truncated, "block payload extends past end of data");
    return b200::detail::take_block(bytes.data(), offset);
}

// =========================== ladder (aalc.cpp:56-115) ===========================

ErrorBoundLadder ErrorBoundLadder::make(std::vector<double> bounds)
{
    if (bounds.empty()) throw std::invalid_argument("error-bound ladder must not be empty");
    double prev = -1.0;
    for (double b : bounds) {
        if (!(b >= 0.0) || !std::isfinite(b)) throw std::invalid_argument("error bounds must be finite and >= 0");
        if (!(b > prev)) throw std::invalid_argument("error bounds must be strictly increasing");
        prev = b;
    }
    ErrorBoundLadder l;
    l.bounds = std::move(bounds);
    return l;
}

ErrorBoundLadder ErrorBoundLadder::default_ladder() { return make({0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3}); }

ErrorBoundLadder ErrorBoundLadder::parse(const std::string& text)
{
    std::vector<double> out;
    std::stringstream in(text);
    for (std::string item; std::getline(in, item, ',');) {
        std::size_t used = 0;
        double v = 0.0;
        try {
            v = std::stod(item, &used);
        } catch (const std::exception&) {
            throw std::invalid_argument("malformed error bound '" + item + "'");
        }
        while (used < item.size() && std::isspace(static_cast<unsigned char>(item[used]))) ++used;
        if (used != item.size()) throw std::invalid_argument("malformed error bound '" + item + "'");
        out.push_back(v);
    }
    return make(std::move(out));
}

// FNV-1a, 64-bit, over each bound's little-endian bytes (the QCKP header's
// ladder fingerprint)
std::uint64_t ErrorBoundLadder::fingerprint() const
{
    std::uint64_t h = 14695981039346656037ull;
    for (double b : bounds) {
        std::uint8_t bytes[8];
        std::memcpy(bytes, &b, 8);
        for (std::uint8_t c : bytes) h = (h ^ c) * 1099511628211ull;
    }
    return h;
}

// aalc.cpp:117-138 — one stride through the ladder, codec on the device
AdaptiveResult compress_stride_adaptive(StrideBuffer& buf, const ErrorBoundLadder& ladder, RatioThreshold theta)
{
    buf.snap_zeros();
    const std::uint64_t bytes_in = buf.size() * 16;
    AdaptiveResult r;
    for (double d : ladder.bounds) {
        const ErrorBound bound(d);
        r.re = b200::compress(buf.re, bound);
        r.im = b200::compress(buf.im, bound);
        r.report.chosen_delta = d;
        r.report.ratio = static_cast<double>(bytes_in) / static_cast<double>(r.re.total_bytes() + r.im.total_bytes());
        if (r.report.ratio >= theta.theta) break;
    }
    r.report.stride_index = buf.stride_index;
    r.report.bytes_in = bytes_in;
    r.report.bytes_out = r.re.total_bytes() + r.im.total_bytes();
    r.report.threshold_met = r.report.ratio >= theta.theta;
    return r;
}

// ===================== CompressedState (aalc.cpp:140-586) =====================

CompressedState::CompressedState() = default;
CompressedState::~CompressedState() = default;
CompressedState::CompressedState(CompressedState&& o) noexcept = default;
CompressedState& CompressedState::operator=(CompressedState&& o) noexcept = default;

CompressedState::CompressedState(std::unique_ptr<b200::CompressedState> impl) : impl_(std::move(impl))
{
    if (impl_) geom_ = impl_->geometry();
}

// deep copy through the device: every stride's blocks, scale and stored sum
CompressedState::CompressedState(const CompressedState& o) : geom_(o.geom_)
{
    if (!o.impl_) return;
    auto c = std::make_unique<b200::CompressedState>(b200::CompressedState::basis_state(geom_, 0));
    std::vector<std::uint8_t> buf;
    for (std::uint64_t j = 0; j < geom_.n_strides(); ++j) {
        std::uint64_t len = 0;
        double sc = 0, ss = 0;
        b200::check(qcs_export_blocks(o.impl_->handle(), j, nullptr, 0, &len, &sc, &ss));
        buf.resize(len);
        b200::check(qcs_export_blocks(o.impl_->handle(), j, buf.data(), len, &len, &sc, &ss));
        b200::check(qcs_import_blocks(c->handle(), j, buf.data(), len, sc, ss));
    }
    impl_ = std::move(c);
}

CompressedState& CompressedState::operator=(const CompressedState& o)
{
    if (this != &o) *this = CompressedState(o);
    return *this;
}

b200::CompressedState& CompressedState::dev() const
{
    if (!impl_) throw std::logic_error("empty CompressedState (default-constructed or moved from)");
    return *impl_;
}

CompressedState CompressedState::basis_state(const StateGeometry& geom, std::uint64_t basis_index)
{
    return CompressedState(
        std::make_unique<b200::CompressedState>(b200::CompressedState::basis_state(geom, basis_index)));
}

CompressedState::GateResult CompressedState::apply_gate(const GateOp& gate, const ErrorBoundLadder& ladder,
                                                        RatioThreshold theta, int workers)
{
    return dev().apply_gate(gate, ladder, theta, workers);
}

StrideBuffer CompressedState::stored_stride(std::uint64_t j) const { return dev().stored_stride(j); }
StrideBuffer CompressedState::decompress_stride(std::uint64_t j) const { return dev().decompress_stride(j); }
std::vector<Amplitude> CompressedState::to_amplitudes() const { return dev().to_amplitudes(); }
double CompressedState::stride_scale(std::uint64_t j) const { return dev().stride_scale(j); }
double CompressedState::norm_sq_tracked() const { return dev().norm_sq_tracked(); }
std::uint64_t CompressedState::compressed_bytes() const { return dev().compressed_bytes(); }
double CompressedState::min_stride_ratio() const { return dev().min_stride_ratio(); }

void CompressedState::save(const std::string& path, std::uint64_t fp) const { dev().save(path, fp); }

LoadedState CompressedState::load(const std::string& path, const std::optional<StateGeometry>& expected)
{
    b200::LoadedState l = b200::CompressedState::load(path, expected);
    LoadedState out;
    out.state = CompressedState(std::make_unique<b200::CompressedState>(std::move(l.state)));
    out.ladder_fingerprint = l.ladder_fingerprint;
    return out;
}

// ========================= run drivers (aalc.cpp:588-676) =========================

RunMetrics apply_program_range(CompressedState& state, const CircuitProgram& program, std::size_t first,
                               std::size_t last, const ErrorBoundLadder& ladder, RatioThreshold theta, int workers)
{
    return b200::apply_program_range(state.dev(), program, first, last, ladder, theta, workers);
}

RunResult run_program_on(CompressedState state, const CircuitProgram& program, const ErrorBoundLadder& ladder,
                         RatioThreshold theta, const RunOptions& options)
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

RunResult run_program(const CircuitProgram& program, const ErrorBoundLadder& ladder, RatioThreshold theta,
                      const StateGeometry& geom, const RunOptions& options)
{
    if (program.n_qubits != geom.n_qubits) throw std::invalid_argument("program and geometry disagree on qubits");
    const std::uint64_t t0 = b200::detail::now_ns();
    CompressedState state = CompressedState::basis_state(geom, options.basis);
    const std::uint64_t init_ns = b200::detail::now_ns() - t0;
    RunResult r = run_program_on(std::move(state), program, ladder, theta, options);
    r.metrics.total_elapsed_ns += init_ns;
    return r;
}

}  // namespace qcs
