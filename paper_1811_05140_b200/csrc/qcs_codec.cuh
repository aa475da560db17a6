// Codec kernels: bit-exact GPU restatement of compress_lossless /
// compress_lossy / decompress (/root/reference/proj/src/codec.cpp:118-340)
// plus the stride sum of squares (core.cpp:30-37) of what was stored.
//
// Parallel structure:
//  * One CTA encodes one stride: warps 0-3 the re plane, warps 4-7 the im
//    plane.  Each lane owns a SUB=32-element sub-chunk and runs the
//    reference's serial step (ref_step) over it, so every code is produced by
//    the reference's own arithmetic.  Only the predictor ENTERING a lane is
//    speculated (lattice_guess); lane l's guess is compared bit-for-bit with
//    lane l-1's exit predictor and any mismatching lane is re-run serially,
//    in order, before anything is emitted.  With a power-of-two bound the
//    reference's predictor lives on an exact lattice and the guesses are
//    right except next to escapes; with any other bound the repair pass
//    degenerates into the reference's serial chain.  Either way the output
//    is the reference's.
//  * Token stream: runs are maximal across lanes and CTA iterations (the
//    LossyEmitter contract, codec.cpp:153-202).  A function-composition scan
//    over lanes finds the run entering each lane; a byte-count scan places
//    each lane's tokens; words of escape/literal runs are placed by their
//    owning lanes.
//  * Side index: per sub-chunk {token offset, skip, exact predictor}, so the
//    decoder runs one independent lane per sub-chunk.
//  * sum_sq: the reference accumulates fl(s + fl(fl(re^2)+fl(im^2))) serially.
//    Within one binade of s every step adds t rounded to the ulp grid of s,
//    which is an exact integer sum; we sum those integers with a block scan
//    and fall back to one exact FP add at every binade crossing or tie.
#pragma once

#include "qcs_device.cuh"

namespace qcs {

constexpr int16_t WCODE16 = INT16_MIN;  // |q| < 32768 so -32768 is free


// ---------------------------------------------------------------------------
// Run-transfer functions for the lane scan.
//   kind 0 ID, 1 CONST(type,start), 2 PASS(type,start)
// ---------------------------------------------------------------------------
struct RunFn {
    int kt;        // kind*4 + type
    uint64_t st;   // run start (absolute element index)
};

__device__ __forceinline__ RunFn fn_compose(RunFn A, RunFn B)  // A then B
{
    const int kb = B.kt >> 2;
    if (kb == 0) return A;
    if ((A.kt >> 2) == 0) return B;
    if (kb == 1) return B;
    const int tb = B.kt & 3;
    return (A.kt & 3) == tb ? A : RunFn{(1 << 2) | tb, B.st};
}

__device__ __forceinline__ void fn_apply(RunFn F, int& ty, uint64_t& st)
{
    const int k = F.kt >> 2, t = F.kt & 3;
    if (k == 0) return;
    if (k == 1 || ty != t) {
        ty = t;
        st = F.st;
    }
}

// ---------------------------------------------------------------------------
// Shared-memory layout of the encoder CTA.
// ---------------------------------------------------------------------------
struct PlaneCarry {
    double P;            // exact predictor entering the next iteration
    double xprev;        // last input of the previous iteration (escape prediction)
    double xprev_next;
    uint64_t out_pos;    // payload bytes of closed tokens
    int open_ty;         // run still open at the end of the last iteration
    uint64_t open_start;
    uint64_t open_vmax;  // varint bytes reserved in front of an open W run
    uint64_t open_w;     // where the open W run's first word lives
    // per-iteration scratch
    double Pnext;
    uint64_t iter_bytes;
    int closes_open;     // open run closes in this iteration
    uint64_t close_vlen;
    uint64_t carry_tok;  // token offset of the run carried into this iteration
    uint64_t carry_w;    // word base of that run in its final position
    uint64_t mv_bytes;   // bytes to slide left by mv_shift
    uint64_t mv_shift;
};

// ---- block-wide helpers over 256 threads (8 warps) ------------------------

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b)
{
    const uint64_t c = a + b;
    return c > (1ull << 62) ? (1ull << 62) : c;
}

// Exclusive scan of a saturating u64 over all 256 threads; returns the
// exclusive prefix and writes the total.
// ---- bitmask view of a lane's codes (zero codes / raw words / nonzero codes)
struct LaneMasks {
    uint32_t z, w, valid;
    uint32_t cbytes;  // bytes of the lane's code tokens (varint of zigzag(q)<<2|1)
};

// varint length of code_token(q) for a 16-bit code: zigzag(q) < 2^16, so the
// token is below 2^18 and takes 1..3 bytes
__device__ __forceinline__ uint32_t code_token_len16(uint32_t c16)
{
    const int32_t q = (int32_t)(int16_t)c16;
    const uint32_t v = ((((uint32_t)q << 1) ^ (uint32_t)(q >> 31)) << 2) | 1u;
    return 1u + (v >= 128u) + (v >= 16384u);
}

// bytes of a lane's code tokens (what lane_masks<true> adds up in cbytes)
__device__ __forceinline__ uint32_t lane_cbytes(const int16_t* cl, int cnt)
{
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(cl);
    uint32_t n = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t v = c2[j];
        const uint32_t lo = v & 0xffffu, hi = v >> 16;
        const bool clo = lo != 0u && lo != 0x8000u && 2 * j < cnt;
        const bool chi = hi != 0u && hi != 0x8000u && 2 * j + 1 < cnt;
        n += (clo ? code_token_len16(lo) : 0u) + (chi ? code_token_len16(hi) : 0u);
    }
    return n;
}

// CB = false: cbytes left 0 (callers that generate the tokens count them then)
template <bool CB = true>
__device__ __forceinline__ LaneMasks lane_masks(const int16_t* cl, int cnt)
{
    LaneMasks m{0u, 0u, cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u), 0u};
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(cl);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t v = c2[j];
        const uint32_t lo = v & 0xffffu, hi = v >> 16;
        m.z |= ((uint32_t)(lo == 0u) << (2 * j)) | ((uint32_t)(hi == 0u) << (2 * j + 1));
        m.w |= ((uint32_t)(lo == 0x8000u) << (2 * j)) | ((uint32_t)(hi == 0x8000u) << (2 * j + 1));
        const bool clo = lo != 0u && lo != 0x8000u && 2 * j < cnt;
        const bool chi = hi != 0u && hi != 0x8000u && 2 * j + 1 < cnt;
        if (CB) m.cbytes += (clo ? code_token_len16(lo) : 0u) + (chi ? code_token_len16(hi) : 0u);
    }
    m.z &= m.valid;
    m.w &= m.valid;
    return m;
}

// The run tokens of lane_tokens only (same emission contract for runs):
// iterates over run starts instead of every token.
template <typename FR>
__device__ __forceinline__ void lane_runs(const LaneMasks& m, int cnt, uint64_t e0, int in_ty, uint64_t in_st,
                                          bool tail_closes, bool close_carried, FR on_run)
{
    if (cnt <= 0) return;
    const int t0 = ((m.z & 1u) ? TY_Z : ((m.w & 1u) ? TY_W : TY_C));
    const bool cont = in_ty != TY_NONE && t0 == in_ty;
    if (!cont && close_carried && in_ty != TY_NONE) on_run(in_ty, in_st, e0);
    uint32_t starts = (m.z & ~(m.z << 1)) | (m.w & ~(m.w << 1));
    while (starts) {
        const int p = __ffs(starts) - 1;
        starts &= starts - 1u;
        const bool isz = (m.z >> p) & 1u;
        const uint32_t run = (isz ? m.z : m.w) >> p;
        const int end = p + (run == 0xffffffffu ? 32 : __ffs(~run) - 1);
        const uint64_t rst = (p == 0 && cont) ? in_st : e0 + (uint64_t)p;
        if (end < cnt || tail_closes) on_run(isz ? TY_Z : TY_W, rst, e0 + (uint64_t)end);
    }
}

__device__ __forceinline__ int mask_type(const LaneMasks& m, int p)
{
    return ((m.z >> p) & 1u) ? TY_Z : (((m.w >> p) & 1u) ? TY_W : TY_C);
}

// Token enumeration over a lane with bitmasks: the same contract as
// lane_walk (runs closed by this lane -> on_run, nonzero codes -> on_code) but
// the loop runs once per token, not once per element.
template <typename FR, typename FC>
__device__ __forceinline__ void lane_tokens(const LaneMasks& m, const int16_t* cl, int cnt, uint64_t e0,
                                            int in_ty, uint64_t in_st, bool tail_closes,
                                            bool close_carried, FR on_run, FC on_code)
{
    if (cnt <= 0) return;
    const int t0 = mask_type(m, 0);
    const bool cont = in_ty != TY_NONE && t0 == in_ty;
    if (!cont && close_carried && in_ty != TY_NONE) on_run(in_ty, in_st, e0);
    const uint32_t cm = m.valid & ~(m.z | m.w);
    uint32_t rest = (cm | (m.z & ~(m.z << 1)) | (m.w & ~(m.w << 1))) & m.valid & ~1u;
    int cur = 0;
    int ty = cont ? in_ty : t0;
    uint64_t rst = cont ? in_st : e0;
    for (;;) {
        const int next = rest ? __ffs(rest) - 1 : cnt;
        if (ty == TY_C) on_code(cl[cur]);
        else if (next < cnt || tail_closes) on_run(ty, rst, e0 + next);
        if (next >= cnt) break;
        rest &= rest - 1u;
        cur = next;
        ty = mask_type(m, next);
        rst = e0 + next;
    }
}

// ---------------------------------------------------------------------------
// Decoder: one lane per sub-chunk, started from its side entry.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void decode_sub(const uint8_t* in, int codec, double td, SideEntry se,
                                           int cnt, double* o, double scale)
{
    uint64_t pos = se.off;
    uint64_t skip = se.skip;
    double P = se.pred;
    int produced = 0;
    const bool sc = scale != 1.0;
    int guard = 0;
    while (produced < cnt) {
        if (++guard > 4 * SUB + 8) break;  // corrupt side index: never spin
        const uint64_t v = get_varint(in, pos);
        if (codec == 1) {
            const unsigned tag = (unsigned)(v & 3u);
            const uint64_t arg = v >> 2;
            if (tag == 0) {
                const uint64_t m = umin64(arg - skip, (uint64_t)(cnt - produced));
                const double val = sc ? __dmul_rn(P, scale) : P;
                for (uint64_t i = 0; i < m; ++i) o[produced++] = val;
            } else if (tag == 1) {
                P = __dadd_rn(P, __dmul_rn(td, (double)unzigzag(arg)));
                o[produced++] = sc ? __dmul_rn(P, scale) : P;
            } else {
                const uint64_t m = umin64(arg - skip, (uint64_t)(cnt - produced));
                for (uint64_t i = 0; i < m; ++i) {
                    P = __longlong_as_double((long long)get_word(in + pos + 8 * (skip + i)));
                    o[produced++] = sc ? __dmul_rn(P, scale) : P;
                }
                pos += 8 * arg;
            }
        } else {
            const uint64_t run = v >> 1;
            const uint64_t m = umin64(run - skip, (uint64_t)(cnt - produced));
            if ((v & 1u) == 0) {
                for (uint64_t i = 0; i < m; ++i) o[produced++] = 0.0;
            } else {
                for (uint64_t i = 0; i < m; ++i) {
                    const double w = __longlong_as_double((long long)get_word(in + pos + 8 * (skip + i)));
                    o[produced++] = sc ? __dmul_rn(w, scale) : w;
                }
                pos += 8 * run;
            }
        }
        skip = 0;
    }
}

// 8 bytes starting at byte offset `pos` of an 8-byte-aligned base (two
// aligned loads + funnel shift; may read up to 15 bytes past pos)
__device__ __forceinline__ uint64_t load8_at(const uint8_t* base, uint64_t pos)
{
    const uint64_t* p = reinterpret_cast<const uint64_t*>(base + (pos & ~7ull));
    const int r = (int)(pos & 7) * 8;
    const uint64_t lo = p[0];
    if (r == 0) return lo;
    return (lo >> r) | (p[1] << (64 - r));
}

// decode_sub over a payload staged in SHARED memory (8-byte aligned base):
// tokens come from a 64-bit byte window, one pair of aligned loads per up to
// 8 one-byte (2-3 three-byte) tokens, instead of one dependent load per byte.
__device__ __forceinline__ void decode_sub_win(const uint8_t* in, int codec, double td, SideEntry se, int cnt,
                                               double* o, double scale)
{
    uint64_t pos = se.off;
    uint64_t w = 0;
    int avail = 0;
    uint64_t skip = se.skip;
    double P = se.pred;
    int produced = 0;
    const bool sc = scale != 1.0;
    int guard = 0;
    while (produced < cnt) {
        if (++guard > 4 * SUB + 8) break;  // corrupt side index: never spin
        if (avail < 5) {
            w = load8_at(in, pos);
            avail = 8;
        }
        const uint64_t stop = ~w & 0x8080808080808080ull;
        const int nb = stop ? (__ffsll((long long)stop) >> 3) : 9;
        uint64_t v;
        if (nb <= 4 && nb <= avail) {
            const uint64_t x = w & ((1ull << (8 * nb)) - 1);
            v = (x & 0x7full) | ((x >> 1) & (0x7full << 7)) | ((x >> 2) & (0x7full << 14)) |
                ((x >> 3) & (0x7full << 21));
            pos += nb;
            avail -= nb;
            w >>= 8 * nb;
        } else {  // long varint: byte loop
            v = get_varint(in, pos);
            avail = 0;
        }
        if (codec == 1) {
            const unsigned tag = (unsigned)(v & 3u);
            const uint64_t arg = v >> 2;
            if (tag == 0) {
                const uint64_t m = umin64(arg - skip, (uint64_t)(cnt - produced));
                const double val = sc ? __dmul_rn(P, scale) : P;
                for (uint64_t i = 0; i < m; ++i) o[produced++] = val;
            } else if (tag == 1) {
                P = __dadd_rn(P, __dmul_rn(td, (double)unzigzag(arg)));
                o[produced++] = sc ? __dmul_rn(P, scale) : P;
            } else {
                const uint64_t m = umin64(arg - skip, (uint64_t)(cnt - produced));
                for (uint64_t i = 0; i < m; ++i) {
                    P = __longlong_as_double((long long)load8_at(in, pos + 8 * (skip + i)));
                    o[produced++] = sc ? __dmul_rn(P, scale) : P;
                }
                pos += 8 * arg;
                avail = 0;
            }
        } else {
            const uint64_t run = v >> 1;
            const uint64_t m = umin64(run - skip, (uint64_t)(cnt - produced));
            if ((v & 1u) == 0) {
                for (uint64_t i = 0; i < m; ++i) o[produced++] = 0.0;
            } else {
                for (uint64_t i = 0; i < m; ++i) {
                    const double x = __longlong_as_double((long long)load8_at(in, pos + 8 * (skip + i)));
                    o[produced++] = sc ? __dmul_rn(x, scale) : x;
                }
                pos += 8 * run;
                avail = 0;
            }
        }
        skip = 0;
    }
}

// ---------------------------------------------------------------------------
// Validating serial walk of one payload (decompress_*_into, codec.cpp:260-340):
// writes the side index and, optionally, the decoded values.  Used for
// imported blocks, basis states and the codec API's decompress.
// ---------------------------------------------------------------------------
__device__ int index_plane(const uint8_t* in, uint64_t len, int codec, double delta, uint64_t n,
                           SideEntry* side, double* outv)
{
    uint64_t pos = 0, produced = 0;
    const double td = 2.0 * delta;
    double P = 0.0;
    auto varint = [&](uint64_t& v) -> int {
        v = 0;
        int shift = 0;
        for (;;) {
            if (pos >= len) return 11;
            const uint8_t bb = in[pos++];
            if (shift >= 63 && (bb & 0x7e) != 0) return 13;
            v |= (uint64_t)(bb & 0x7f) << (shift & 63);
            if (!(bb & 0x80)) return 0;
            shift += 7;
        }
    };
    auto mark = [&](uint64_t tokpos, uint64_t k, uint64_t tokfirst, double predv) {
        if (side && (k % SUB) == 0) side[k / SUB] = SideEntry{(uint32_t)tokpos, (uint32_t)(k - tokfirst), predv};
    };
    while (produced < n) {
        const uint64_t tokpos = pos;
        uint64_t v;
        int rc = varint(v);
        if (rc) return rc;
        if (codec == 0) {
            const uint64_t run = v >> 1;
            if (run == 0 || run > n - produced) return 13;
            const uint64_t first = produced;
            if ((v & 1u) == 0) {
                for (uint64_t i = 0; i < run; ++i) {
                    mark(tokpos, produced, first, 0.0);
                    if (outv) outv[produced] = 0.0;
                    ++produced;
                }
            } else {
                for (uint64_t i = 0; i < run; ++i) {
                    if (pos + 8 > len) return 11;
                    mark(tokpos, produced, first, 0.0);
                    if (outv) outv[produced] = __longlong_as_double((long long)get_word(in + pos));
                    pos += 8;
                    ++produced;
                }
            }
        } else {
            const unsigned tag = (unsigned)(v & 3u);
            const uint64_t arg = v >> 2;
            const uint64_t first = produced;
            if (tag == 0) {
                if (arg == 0 || arg > n - produced) return 13;
                for (uint64_t i = 0; i < arg; ++i) {
                    mark(tokpos, produced, first, P);
                    if (outv) outv[produced] = P;
                    ++produced;
                }
            } else if (tag == 1) {
                const int64_t q = unzigzag(arg);
                if (q == 0 || q <= -QRADIUS || q >= QRADIUS) return 13;
                mark(tokpos, produced, first, P);
                P = __dadd_rn(P, __dmul_rn(td, (double)q));
                if (outv) outv[produced] = P;
                ++produced;
            } else if (tag == 2) {
                if (arg == 0 || arg > n - produced) return 13;
                for (uint64_t i = 0; i < arg; ++i) {
                    if (pos + 8 > len) return 11;
                    mark(tokpos, produced, first, P);
                    P = __longlong_as_double((long long)get_word(in + pos));
                    pos += 8;
                    if (outv) outv[produced] = P;
                    ++produced;
                }
            } else {
                return 13;
            }
        }
    }
    if (pos != len) return 13;
    return 0;
}

}  // namespace qcs
