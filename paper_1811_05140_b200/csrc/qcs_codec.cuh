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

__device__ __forceinline__ int ty16(int16_t c) { return c == 0 ? TY_Z : (c == WCODE16 ? TY_W : TY_C); }

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

constexpr int MAXPIN = 12;  // pinned exact steps per plane and iteration (then lane-serial chains)

struct EncShared {
    double entryP[2][PLANE_LANES];
    double exitP[2][PLANE_LANES];
    RunFn fincl[2][PLANE_LANES];
    uint64_t bstart[2][PLANE_LANES];
    uint64_t runtok[2][PLANE_LANES];
    uint64_t runw[2][PLANE_LANES];
    uint32_t bytes[2][PLANE_LANES];
    int8_t ftype[2][PLANE_LANES + 1];
    RunFn wfn[8];
    long long wesc_i[8];
    double wesc_v[8];
    uint64_t wsum[8];
    long long wmin[8];
    PlaneCarry carry[2];
    long long pin_idx[2][MAXPIN];
    double pin_val[2][MAXPIN];
    int16_t pin_code[2][MAXPIN];
    int npin[2];
    int pin_over[2];
    long long wfail[8];
    double fail_prev[2];
    double s;            // exact running sum of squares of the stride
    long long kstar;
    uint64_t mvmax;
};

constexpr size_t ENC_S_OFF = ((sizeof(double) * 2 * PLANE_LANES * XS_STRIDE +
                               sizeof(int16_t) * 2 * ITER) + 15) & ~size_t(15);
constexpr size_t ENC_SMEM = ENC_S_OFF + sizeof(EncShared);

struct EncodeArgs {
    const double* X;          // input planes
    uint64_t n;               // elements per plane
    const uint64_t* job_stride;  // per CTA: stride index; planes at X + stride*stride_elems (+n)
    uint64_t stride_elems;       // null job_stride: CTA b reads X + b*2n
    const uint8_t* pending;   // per CTA: encode at this level? (null = all)
    int planes;               // 1 (codec API) or 2 (stride)
    int snap;                 // apply snap_zeros on load (engine) or not (codec API)
    uint8_t* out;             // payload of plane (b,c) at out + (2b+c)*cap
    uint64_t cap;
    SideEntry* side;          // side entries of plane (b,c) at side + (2b+c)*nsub
    uint64_t nsub;
    uint64_t* out_len;        // [2b+c]
    double* sumsq;            // [b] or null
    CodecParams cp;
    unsigned long long* counters;  // optional: [0] repaired lanes, [1] exact-sum passes,
                                   // [2] slid bytes, [3] lanes that fell back to the serial chain
};

__device__ __forceinline__ double& xs_at(double* xs, int pl, int k)
{
    return xs[pl * PLANE_LANES * XS_STRIDE + (k >> 5) * XS_STRIDE + (k & 31)];
}

// ---- block-wide helpers over 256 threads (8 warps) ------------------------

__device__ __forceinline__ long long block_min_ll(long long v, long long* wmin)
{
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = v;
    __syncthreads();
    long long r = wmin[0];
    for (int w = 1; w < 8; ++w) r = min(r, wmin[w]);
    return r;
}

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b)
{
    const uint64_t c = a + b;
    return c > (1ull << 62) ? (1ull << 62) : c;
}

// Exclusive scan of a saturating u64 over all 256 threads; returns the
// exclusive prefix and writes the total.
__device__ __forceinline__ uint64_t block_scan_sat(uint64_t v, uint64_t* wsum, uint64_t& total)
{
    const int wl = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (wl >= o) inc = sat_add(inc, u);
    }
    __syncthreads();
    if (wl == 31) wsum[w] = inc;
    __syncthreads();
    uint64_t pre = 0, tot = 0;
    for (int i = 0; i < 8; ++i) {
        if (i < w) pre = sat_add(pre, wsum[i]);
        tot = sat_add(tot, wsum[i]);
    }
    total = tot;
    // exclusive prefix from the neighbour's inclusive value (inc - v would be
    // wrong once this thread's own value saturated)
    const uint64_t prev = __shfl_up_sync(0xffffffffu, inc, 1);
    return sat_add(pre, wl ? prev : 0);
}

// t_k = fl(fl(re^2) + fl(im^2)) at iteration-local element k.
__device__ __forceinline__ double tsq(double* xs, int k)
{
    const double r = xs_at(xs, 0, k), i = xs_at(xs, 1, k);
    return __dadd_rn(__dmul_rn(r, r), __dmul_rn(i, i));
}

// Exact emulation of `for k: s += t_k` (core.cpp:33-35) over this iteration's
// n_it elements; S.s holds s in and out.  Must be called by all 256 threads.
__device__ __forceinline__ void sumsq_iteration(double* xs, int n_it, EncShared& S, unsigned long long* counters)
{
    constexpr int PER = ITER / CODEC_THREADS;  // 16 elements per thread
    const int tid = threadIdx.x;
    const int kb = tid * PER;
    int k0 = 0;
    for (;;) {
        __syncthreads();
        const double s = S.s;
        if (k0 >= n_it) break;
        if (counters && tid == 0) atomicAdd(&counters[1], 1ull);
        if (s == 0.0) {
            long long mine = LLONG_MAX;
            for (int i = 0; i < PER; ++i) {
                const int k = kb + i;
                if (k >= k0 && k < n_it && tsq(xs, k) != 0.0) {
                    mine = k;
                    break;
                }
            }
            const long long first = block_min_ll(mine, S.wmin);
            if (first == LLONG_MAX) break;
            if (tid == 0) S.s = tsq(xs, (int)first);  // 0 + t == t exactly
            k0 = (int)first + 1;
            continue;
        }
        const int e = ilogb(s);
        if (e < -960) {  // tiny sums: take exact serial steps (no unit scaling)
            if (tid == 0) S.s = __dadd_rn(s, tsq(xs, k0));
            ++k0;
            continue;
        }
        const double to_units = ldexp(1.0, 52 - e);          // 1/ulp(s)
        const uint64_t ms = (uint64_t)(s * to_units);        // exact, in [2^52, 2^53)
        const double lim = 9007199254740992.0;               // 2^53
        // pass 1: local totals
        uint64_t loc = 0;
        for (int i = 0; i < PER; ++i) {
            const int k = kb + i;
            if (k < k0 || k >= n_it) continue;
            const double y = tsq(xs, k) * to_units;          // exact scaling
            loc = sat_add(loc, y >= lim ? (1ull << 62) : (uint64_t)rint(y));
        }
        uint64_t total;
        const uint64_t off = block_scan_sat(loc, S.wsum, total);
        // pass 2: first element that ties, overflows, or crosses the binade
        long long bad = LLONG_MAX;
        uint64_t run = off;
        for (int i = 0; i < PER && bad == LLONG_MAX; ++i) {
            const int k = kb + i;
            if (k < k0 || k >= n_it) continue;
            const double y = tsq(xs, k) * to_units;
            if (y >= lim || y - floor(y) == 0.5) { bad = k; break; }
            run = sat_add(run, (uint64_t)rint(y));
            if (ms + run >= (1ull << 53)) bad = k;
        }
        const long long kstar = block_min_ll(bad, S.wmin);
#ifdef SUMSQ_TRACE
        if (tid == 0) printf("k0=%d s=%.17g e=%d ms=%llu total=%llu kstar=%lld\n", k0, s, e, (unsigned long long)ms, (unsigned long long)total, kstar);
#endif
        if (kstar == LLONG_MAX) {
            if (tid == 0) S.s = (double)(ms + total) / to_units;  // exact
            break;
        }
        // the owner of k* recomputes its prefix before k* and takes one exact step
        if (kstar >= kb && kstar < kb + PER) {
            uint64_t r2 = off;
            for (int k = max(kb, k0); k < (int)kstar; ++k) r2 += (uint64_t)rint(tsq(xs, k) * to_units);
            const double before = (double)(ms + r2) / to_units;  // exact (< 2^53 units)
            S.s = __dadd_rn(before, tsq(xs, (int)kstar));
        }
        k0 = (int)kstar + 1;
    }
}

// ---- scans over the 128 lanes of one plane (4 warps) ----------------------

__device__ __forceinline__ RunFn plane_fn_scan(RunFn F, EncShared& S, int pl)
{
    const int wl = threadIdx.x & 31, w = threadIdx.x >> 5;
    RunFn inc = F;
    for (int o = 1; o < 32; o <<= 1) {
        RunFn u;
        u.kt = __shfl_up_sync(0xffffffffu, inc.kt, o);
        u.st = __shfl_up_sync(0xffffffffu, inc.st, o);
        if (wl >= o) inc = fn_compose(u, inc);
    }
    if (wl == 31) S.wfn[w] = inc;
    __syncthreads();
    RunFn pre{0, 0};
    for (int i = pl * 4; i < w; ++i) pre = fn_compose(pre, S.wfn[i]);
    return fn_compose(pre, inc);
}

// Exclusive "last predicted escape" scan over the plane's lanes: returns the
// index (or -1) and input value of the last escape before this lane.
__device__ __forceinline__ long long plane_last_scan(long long idx, double val, EncShared& S, int pl,
                                                     double& out_val)
{
    const int wl = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long ii = idx;
    double vv = val;
    for (int o = 1; o < 32; o <<= 1) {
        const long long ui = __shfl_up_sync(0xffffffffu, ii, o);
        const double uv = __shfl_up_sync(0xffffffffu, vv, o);
        if (wl >= o && ii < 0) {
            ii = ui;
            vv = uv;
        }
    }
    // exclusive within the warp
    long long ei = __shfl_up_sync(0xffffffffu, ii, 1);
    double ev = __shfl_up_sync(0xffffffffu, vv, 1);
    if (wl == 0) ei = -1;
    __syncthreads();
    if (wl == 31) {
        S.wesc_i[w] = ii;
        S.wesc_v[w] = vv;
    }
    __syncthreads();
    if (ei < 0) {
        for (int k = w - 1; k >= pl * 4; --k) {
            if (S.wesc_i[k] >= 0) {
                ei = S.wesc_i[k];
                ev = S.wesc_v[k];
                break;
            }
        }
    }
    out_val = ev;
    return ei;
}

__device__ __forceinline__ uint64_t plane_sum_scan(uint64_t v, EncShared& S, int pl, uint64_t& total)
{
    const int wl = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (wl >= o) inc += u;
    }
    __syncthreads();
    if (wl == 31) S.wsum[w] = inc;
    __syncthreads();
    uint64_t pre = 0, tot = 0;
    for (int i = pl * 4; i < pl * 4 + 4; ++i) {
        if (i < w) pre += S.wsum[i];
        tot += S.wsum[i];
    }
    total = tot;
    return pre + inc - v;
}

// ---- the lane token walk ----------------------------------------------------
// Walks the lane's codes with the entering run state and calls
//   on_run(ty, start, endexcl)  for every run the lane closes,
//   on_code(q)                  for every nonzero code,
//   on_word(k, run_start)       for every W element (mode words only).
// Returns the run still open at the lane end in (ty, start) and whether
// the lane closes it (emit_tail).
template <typename FR, typename FC, typename FW>
__device__ __forceinline__ void lane_walk(const int16_t* cl, int cnt, uint64_t e0, int in_ty,
                                          uint64_t in_st, bool tail_closes, bool close_carried,
                                          FR on_run,
                                          FC on_code, FW on_word)
{
    int cur = TY_NONE;
    uint64_t cst = 0;
    if (cnt > 0 && in_ty != TY_NONE && ty16(cl[0]) == in_ty) {
        cur = in_ty;
        cst = in_st;
    } else if (close_carried && in_ty != TY_NONE) {
        // run carried over from the previous CTA iteration ends right here
        on_run(in_ty, in_st, e0);
    }
    for (int i = 0; i < cnt; ++i) {
        const uint64_t k = e0 + i;
        const int16_t c = cl[i];
        const int t = ty16(c);
        if (t == TY_C) {
            if (cur != TY_NONE) on_run(cur, cst, k);
            cur = TY_NONE;
            on_code(c);
        } else {
            if (t != cur) {
                if (cur != TY_NONE) on_run(cur, cst, k);
                cur = t;
                cst = k;
            }
            if (t == TY_W) on_word(k, cst);
        }
    }
    if (cur != TY_NONE && tail_closes) on_run(cur, cst, e0 + cnt);
}


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
        m.cbytes += (clo ? code_token_len16(lo) : 0u) + (chi ? code_token_len16(hi) : 0u);
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

template <bool LOSSY>
__global__ void __launch_bounds__(CODEC_THREADS, 2) k_encode(EncodeArgs a)
{
    const int b = blockIdx.x;
    if (a.pending && !a.pending[b]) return;
    extern __shared__ __align__(16) unsigned char smem[];
    double* xs = reinterpret_cast<double*>(smem);
    int16_t* code = reinterpret_cast<int16_t*>(xs + 2 * PLANE_LANES * XS_STRIDE);
    EncShared& S = *reinterpret_cast<EncShared*>(smem + ENC_S_OFF);

    const CodecParams cp = a.cp;
    const int tid = threadIdx.x;
    const int pl = tid >> 7;
    const int lane = tid & (PLANE_LANES - 1);
    const bool pact = pl < a.planes;
    const uint64_t n = a.n;
    const double* xg = a.X + (a.job_stride ? a.job_stride[b] * a.stride_elems : (uint64_t)b * 2 * n) +
                       (uint64_t)pl * n;
    uint8_t* out = a.out + ((uint64_t)b * 2 + pl) * a.cap;
    SideEntry* side = a.side + ((uint64_t)b * 2 + pl) * a.nsub;
    double* xl = xs + pl * PLANE_LANES * XS_STRIDE + lane * XS_STRIDE;
    int16_t* cl = code + pl * ITER + lane * SUB;
    PlaneCarry& C = S.carry[pl];

    if (lane == 0) {
        C.P = 0.0;
        C.xprev = 0.0;
        C.out_pos = 0;
        C.open_ty = TY_NONE;
        C.open_start = 0;
        C.open_vmax = 0;
        C.open_w = 0;
    }
    if (tid == 0) S.s = 0.0;
    __syncthreads();

    for (uint64_t base = 0; base < n; base += ITER) {
        const uint64_t e0 = base + (uint64_t)lane * SUB;
        const int cnt = (pact && e0 < n) ? (int)umin64(SUB, n - e0) : 0;
        const bool final_iter = base + ITER >= n;
        const int active = pact ? (int)umin64(PLANE_LANES, (n - base + SUB - 1) / SUB) : 0;
        const int n_it = (int)umin64(ITER, n - base);

        // 1. coalesced asynchronous load (cp.async: every copy of the
        //    iteration in flight at once), then snap_zeros in shared memory
#pragma unroll 8
        for (int i = lane; i < ITER; i += PLANE_LANES) {
            double* dst = &xs_at(xs, pl, i);
            if (pact && base + i < n) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(xg + base + i)
                             : "memory");
            } else {
                *dst = 0.0;
            }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        if (a.snap && cnt > 0) {
            for (int i = 0; i < cnt; ++i) xl[i] = snap(xl[i]);
        }
        __syncthreads();

        if (LOSSY && cp.pow2) {
            // 2-4 (power-of-two bound).  Event rounds: the reference's predictor
            // after element k is, unless something special happens, the point of
            // the current anchor's 2*delta lattice nearest x_k.  Anchors are
            // *events*: the exact predictor carried into the iteration, predicted
            // escapes (a jump beyond the escape limit + 2*delta escapes whatever
            // the predictor), and pinned exact steps.  Every non-pinned element
            // is verified by one reference step from the speculated predictor of
            // its left neighbour; all elements verified => the speculation IS the
            // reference chain (induction from the exact carried predictor).  The
            // first element that fails (rounding drift off the lattice, a missed
            // or phantom escape, a tie) is pinned with its exact reference step
            // and the plane is re-verified.  Verification is element-parallel.
            if (lane == 0) {
                S.npin[pl] = 0;
                S.pin_over[pl] = 0;
            }
            if (cnt > 0 && lane + 1 == active) C.xprev_next = xl[cnt - 1];
            __syncthreads();
            long long f = LLONG_MAX;
            for (int round = 0;; ++round) {
                const int np = S.npin[pl];
                // (a) last event of every lane, then the event entering each lane
                long long my_last = -1;
                double my_val = 0.0;
                if (cnt > 0) {
                    double xp = lane == 0 ? C.xprev : xs_at(xs, pl, lane * SUB - 1);
                    int pp = 0;
                    while (pp < np && S.pin_idx[pl][pp] < (long long)e0) ++pp;
                    for (int i = 0; i < cnt; ++i) {
                        const long long k = (long long)e0 + i;
                        const double x = xl[i];
                        if (pp < np && S.pin_idx[pl][pp] == k) {
                            my_last = k;
                            my_val = S.pin_val[pl][pp];
                            ++pp;
                        } else if (predict_escape(cp, x, xp)) {
                            my_last = k;
                            my_val = x;
                        }
                        xp = x;
                    }
                }
                double aval;
                const long long aidx = plane_last_scan(my_last, my_val, S, pl, aval);
                // (b) speculate and verify every element
                long long fail = LLONG_MAX;
                double fprev = 0.0;
                if (cnt > 0) {
                    double A = aidx >= 0 ? aval : C.P;
                    const long long Aidx = aidx >= 0 ? aidx : (long long)base - 1;
                    double Pprev = (Aidx == (long long)e0 - 1) ? A
                                   : lattice_point(cp, A, xs_at(xs, pl, lane * SUB - 1));
                    double xp = lane == 0 ? C.xprev : xs_at(xs, pl, lane * SUB - 1);
                    int pp = 0;
                    while (pp < np && S.pin_idx[pl][pp] < (long long)e0) ++pp;
#pragma unroll 4
                    for (int i = 0; i < cnt; ++i) {
                        const long long k = (long long)e0 + i;
                        const double x = xl[i];
                        double Ph;
                        int16_t c16;
                        if (pp < np && S.pin_idx[pl][pp] == k) {
                            Ph = S.pin_val[pl][pp];
                            c16 = S.pin_code[pl][pp];
                            A = Ph;
                            ++pp;
                        } else {
                            if (predict_escape(cp, x, xp)) {
                                Ph = x;
                                A = x;
                            } else {
                                Ph = lattice_step(cp, A, x);
                            }
                            double P2 = Pprev;
                            const int32_t c = ref_step(cp, P2, x);
                            c16 = c == WCODE ? WCODE16 : (int16_t)c;
                            if (!same_bits(P2, Ph) && fail == LLONG_MAX) {
                                fail = k;
                                fprev = Pprev;
                            }
                        }
                        cl[i] = c16;
                        xp = x;
                        Pprev = Ph;
                    }
                }
                // (c) first failure of the plane
                long long m = fail;
                for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
                if ((threadIdx.x & 31) == 0) S.wfail[threadIdx.x >> 5] = m;
                __syncthreads();
                f = LLONG_MAX;
                for (int w = pl * 4; w < pl * 4 + 4; ++w) f = min(f, S.wfail[w]);
                if (fail != LLONG_MAX && fail == f) S.fail_prev[pl] = fprev;
                const bool more = f != LLONG_MAX && S.npin[pl] < MAXPIN;
                if (!__syncthreads_or(more)) break;
                if (lane == 0 && more) {  // pin the exact reference step at f
                    double P = S.fail_prev[pl];
                    const int32_t c = ref_step(cp, P, xs_at(xs, pl, (int)(f - (long long)base)));
                    const int q = S.npin[pl];
                    S.pin_idx[pl][q] = f;
                    S.pin_val[pl][q] = P;
                    S.pin_code[pl][q] = c == WCODE ? WCODE16 : (int16_t)c;
                    S.npin[pl] = q + 1;
                    if (a.counters) atomicAdd(&a.counters[0], 1ull);
                }
                __syncthreads();
            }
            // (d) pin budget exhausted (e.g. a bound whose lattice never holds):
            //     the reference's serial chain from the first unverified element.
            const long long fser = f;  // LLONG_MAX unless the budget ran out
            // (e) final values: predictor of every element into xs, lane entries
            {
                const int np = S.npin[pl];
                double Pprev = 0.0, xp = 0.0, A = 0.0;
                if (cnt > 0) {
                    long long my_last = -1;
                    double my_val = 0.0;
                    (void)my_last;
                    (void)my_val;
                }
                // recompute the entering event (same as (a)) before anyone overwrites x
                long long my_last = -1;
                double my_val = 0.0;
                if (cnt > 0) {
                    double xq = lane == 0 ? C.xprev : xs_at(xs, pl, lane * SUB - 1);
                    int pp = 0;
                    while (pp < np && S.pin_idx[pl][pp] < (long long)e0) ++pp;
                    for (int i = 0; i < cnt; ++i) {
                        const long long k = (long long)e0 + i;
                        const double x = xl[i];
                        if (pp < np && S.pin_idx[pl][pp] == k) {
                            my_last = k;
                            my_val = S.pin_val[pl][pp];
                            ++pp;
                        } else if (predict_escape(cp, x, xq)) {
                            my_last = k;
                            my_val = x;
                        }
                        xq = x;
                    }
                }
                double aval;
                const long long aidx = plane_last_scan(my_last, my_val, S, pl, aval);
                if (cnt > 0) {
                    A = aidx >= 0 ? aval : C.P;
                    const long long Aidx = aidx >= 0 ? aidx : (long long)base - 1;
                    Pprev = (Aidx == (long long)e0 - 1) ? A
                            : lattice_point(cp, A, xs_at(xs, pl, lane * SUB - 1));
                    xp = lane == 0 ? C.xprev : xs_at(xs, pl, lane * SUB - 1);
                }
                __syncthreads();  // neighbours' x read; now overwrite with predictors
                if (cnt > 0) {
                    S.entryP[pl][lane] = Pprev;
                    int pp = 0;
                    while (pp < np && S.pin_idx[pl][pp] < (long long)e0) ++pp;
                    for (int i = 0; i < cnt; ++i) {
                        const long long k = (long long)e0 + i;
                        if (k >= fser) break;
                        const double x = xl[i];
                        double Ph;
                        if (pp < np && S.pin_idx[pl][pp] == k) {
                            Ph = S.pin_val[pl][pp];
                            A = Ph;
                            ++pp;
                        } else if (predict_escape(cp, x, xp)) {
                            Ph = x;
                            A = x;
                        } else {
                            Ph = lattice_step(cp, A, x);
                        }
                        xp = x;
                        xl[i] = Ph;
                        Pprev = Ph;
                    }
                    S.exitP[pl][lane] = Pprev;
                }
                __syncthreads();
                if (lane == 0 && fser != LLONG_MAX) {
                    // serial tail: x of elements >= fser is still in xs
                    if (a.counters) atomicAdd(&a.counters[3], 1ull);
                    const int k0 = (int)(fser - (long long)base);
                    double P = S.fail_prev[pl];
                    for (int k = k0; k < n_it; ++k) {
                        if ((k & (SUB - 1)) == 0) S.entryP[pl][k / SUB] = P;
                        const int32_t c = ref_step(cp, P, xs_at(xs, pl, k));
                        code[pl * ITER + k] = c == WCODE ? WCODE16 : (int16_t)c;
                        xs_at(xs, pl, k) = P;
                    }
                    S.exitP[pl][active - 1] = P;
                }
                if (lane == 0 && active > 0) C.Pnext = S.exitP[pl][active - 1];
                __syncthreads();
            }
        } else {
        // 2. entry predictor: exact for lane 0; for the others a guess on the
        //    lattice of the last *predicted* escape (|x_k - x_k-1| beyond the
        //    escape limit by more than 2*delta escapes whatever the predictor
        //    is) or, if none in this iteration, of the exact carried predictor.
        double entry = 0.0;
        double lane_anchor = C.P;
        if (LOSSY) {
            long long my_last = -1;
            double my_val = 0.0;
            if (cnt > 0) {
                const double thr = __dmul_rn(cp.td, 32769.0);
                double xp = lane == 0 ? C.xprev : xs_at(xs, pl, lane * SUB - 1);
                for (int i = 0; i < cnt; ++i) {
                    const double x = xl[i];
                    if (fabs(__dsub_rn(x, xp)) > thr) {
                        my_last = (long long)(e0 + i);
                        my_val = x;
                    }
                    xp = x;
                }
                if (lane + 1 == active) C.xprev_next = xl[cnt - 1];
            }
            double aval;
            const long long aidx = plane_last_scan(my_last, my_val, S, pl, aval);
            if (cnt > 0) {
                if (lane == 0) {
                    entry = C.P;
                } else if (aidx == (long long)e0 - 1) {
                    entry = aval;
                } else {
                    const double anchor = aidx >= 0 ? aval : C.P;
                    entry = anchored_guess(cp, anchor, xs_at(xs, pl, lane * SUB - 2),
                                           xs_at(xs, pl, lane * SUB - 1));
                }
                if (lane > 0 && aidx >= 0) lane_anchor = aval;
                S.entryP[pl][lane] = entry;
            }
        }
        __syncthreads();

        // 3. lane encode.  Lossy: every element is speculated independently
        //    (the reference's predictor after coding x_k is the point of the
        //    current anchor's 2*delta lattice nearest x_k, or x_k itself on an
        //    escape) and verified by one reference step from the speculated
        //    predictor of x_k-1.  No dependency chain, so the loop pipelines.
        //    From the first element that fails, the reference's serial chain
        //    takes over for the rest of the lane.  Codes only: x stays in shared
        //    memory for the repair passes.
        if (cnt > 0) {
            if (LOSSY) {
                const double thr = __dmul_rn(cp.td, 32769.0);
                double xp = lane == 0 ? C.xprev : xs_at(xs, pl, lane * SUB - 1);
                double anc = lane_anchor;
                double Pprev = entry, Pfail = 0.0;
                int fpos = cnt;
#pragma unroll 4
                for (int i = 0; i < cnt; ++i) {
                    const double x = xl[i];
                    const bool esc = fabs(__dsub_rn(x, xp)) > thr;
                    xp = x;
                    double Ph;
                    if (esc) {
                        Ph = x;
                        anc = x;
                    } else {
                        const double d = __dsub_rn(x, anc);
                        const double M = rint(cp.pow2 ? __dmul_rn(d, cp.inv_td) : __ddiv_rn(d, cp.td));
                        Ph = __dadd_rn(anc, __dmul_rn(cp.td, M));
                    }
                    double P2 = Pprev;
                    const int32_t c = ref_step(cp, P2, x);
                    cl[i] = c == WCODE ? WCODE16 : (int16_t)c;
                    if (!same_bits(P2, Ph) && i < fpos) {
                        fpos = i;
                        Pfail = Pprev;
                    }
                    Pprev = Ph;
                }
                if (fpos < cnt) {
                    if (a.counters) atomicAdd(&a.counters[3], 1ull);
                    double P = Pfail;
                    for (int i = fpos; i < cnt; ++i) {
                        const int32_t c = ref_step(cp, P, xl[i]);
                        cl[i] = c == WCODE ? WCODE16 : (int16_t)c;
                    }
                    Pprev = P;
                }
                S.exitP[pl][lane] = Pprev;
            } else {
                for (int i = 0; i < cnt; ++i)
                    cl[i] = __double_as_longlong(xl[i]) == 0 ? (int16_t)0 : WCODE16;
            }
        }
        __syncthreads();

        if (LOSSY) {
            // 4a. parallel repair passes: a lane whose guessed entry differs from
            //     its left neighbour's exit re-runs from that exit.  The old
            //     speculative chain is replayed in lock step; once both hold the
            //     same predictor the rest of the lane is already exact.
            for (int pass = 0; pass < 4; ++pass) {
                const bool bad = cnt > 0 && lane > 0 && !same_bits(S.entryP[pl][lane], S.exitP[pl][lane - 1]);
                const double want = bad ? S.exitP[pl][lane - 1] : 0.0;
                if (!__syncthreads_or(bad)) break;
                if (bad) {
                    if (a.counters) atomicAdd(&a.counters[0], 1ull);
                    double Pn = want, Po = S.entryP[pl][lane];
                    bool resync = false;
                    for (int i = 0; i < cnt; ++i) {
                        const double x = xl[i];
                        const int16_t co = cl[i];
                        if (co == WCODE16) Po = x;
                        else if (co != 0) Po = __dadd_rn(Po, __dmul_rn(cp.td, (double)co));
                        const int32_t c = ref_step(cp, Pn, x);
                        cl[i] = c == WCODE ? WCODE16 : (int16_t)c;
                        if (same_bits(Pn, Po)) {
                            resync = true;
                            break;
                        }
                    }
                    S.entryP[pl][lane] = want;
                    if (!resync) S.exitP[pl][lane] = Pn;
                }
                __syncthreads();
            }
            // 4b. whatever is left (long dependency chains, e.g. a bound that
            //     is not a power of two): the reference's serial order
            if (lane == 0 && active > 0) {
                for (int l = 1; l < active; ++l) {
                    const double want = S.exitP[pl][l - 1];
                    if (same_bits(want, S.entryP[pl][l])) continue;
                    if (a.counters) atomicAdd(&a.counters[0], 1ull);
                    double Pn = want, Po = S.entryP[pl][l];
                    S.entryP[pl][l] = want;
                    const int c2 = (int)umin64(SUB, n - (base + (uint64_t)l * SUB));
                    const double* xl2 = xs + pl * PLANE_LANES * XS_STRIDE + l * XS_STRIDE;
                    int16_t* cl2 = code + pl * ITER + l * SUB;
                    bool resync = false;
                    for (int i = 0; i < c2; ++i) {
                        const double x = xl2[i];
                        const int16_t co = cl2[i];
                        if (co == WCODE16) Po = x;
                        else if (co != 0) Po = __dadd_rn(Po, __dmul_rn(cp.td, (double)co));
                        const int32_t c = ref_step(cp, Pn, x);
                        cl2[i] = c == WCODE ? WCODE16 : (int16_t)c;
                        if (same_bits(Pn, Po)) {
                            resync = true;
                            break;
                        }
                    }
                    if (!resync) S.exitP[pl][l] = Pn;
                }
                C.Pnext = S.exitP[pl][active - 1];
            }
            __syncthreads();
            // 4c. replace x by the stored (reconstructed) values: the decoder's
            //     chain from the verified entry (codec.cpp:296-335)
            if (cnt > 0) {
                double P = S.entryP[pl][lane];
                for (int i = 0; i < cnt; ++i) {
                    const int16_t co = cl[i];
                    if (co == WCODE16) P = xl[i];
                    else if (co != 0) P = __dadd_rn(P, __dmul_rn(cp.td, (double)co));
                    xl[i] = P;
                }
            }
            __syncthreads();
        }

        }

        // 5. stored sum of squares (needs both planes' final values)
        if (a.sumsq) sumsq_iteration(xs, n_it, S, a.counters);

        // 6. run summary of each lane and the run entering it
        S.ftype[pl][lane] = cnt > 0 ? (int8_t)ty16(cl[0]) : (int8_t)TY_NONE;
        if (lane == 0) S.ftype[pl][PLANE_LANES] = TY_NONE;
        RunFn F{0, 0};
        if (cnt > 0) {
            const int t0 = ty16(cl[0]);
            bool full = t0 != TY_C;
            for (int i = 1; i < cnt && full; ++i) full = ty16(cl[i]) == t0;
            if (full) {
                F = RunFn{(2 << 2) | t0, e0};
            } else {
                const int tl = ty16(cl[cnt - 1]);
                if (tl == TY_C) {
                    F = RunFn{(1 << 2) | TY_NONE, 0};
                } else {
                    int j = cnt - 1;
                    while (j > 0 && ty16(cl[j - 1]) == tl) --j;
                    F = RunFn{(1 << 2) | tl, e0 + j};
                }
            }
        }
        const RunFn inc = plane_fn_scan(F, S, pl);
        S.fincl[pl][lane] = inc;
        __syncthreads();
        int in_ty = C.open_ty;
        uint64_t in_st = C.open_start;
        if (lane > 0) fn_apply(S.fincl[pl][lane - 1], in_ty, in_st);
        // does this lane close the run open at its end?
        bool tail_closes;
        if (lane + 1 < active) {
            tail_closes = true;  // decided per run type below via ftype
        } else {
            tail_closes = final_iter;
        }
        const int next_ft = (lane + 1 < active) ? S.ftype[pl][lane + 1] : TY_NONE;

        // 7. byte count of the tokens this lane closes
        uint32_t nbytes = 0;
        int closes_open = 0;
        uint64_t close_vlen = 0;
        int tail_ty = TY_NONE;
        uint64_t tail_st = 0;
        {
            // find the lane's final open run first (to resolve tail_closes)
            int cur = TY_NONE;
            uint64_t cst = 0;
            // recompute the tail (cheap): last run state
            if (cnt > 0) {
                const int tl = ty16(cl[cnt - 1]);
                if (tl != TY_C) {
                    int j = cnt - 1;
                    while (j > 0 && ty16(cl[j - 1]) == tl) --j;
                    cur = tl;
                    cst = e0 + j;
                    if (j == 0 && in_ty == tl) cst = in_st;
                }
            }
            tail_ty = cur;
            tail_st = cst;
            if (lane + 1 < active) tail_closes = (cur != TY_NONE) && (next_ft != cur);
            lane_walk(
                cl, cnt, e0, in_ty, in_st, tail_closes, lane == 0,
                [&](int t, uint64_t st, uint64_t end) {
                    const uint64_t len = end - st;
                    const int vl = varint_len(run_token(LOSSY, t, len));
                    nbytes += vl + (t == TY_W ? 8u * (uint32_t)len : 0u);
                    if (st < base) {
                        closes_open = 1;
                        close_vlen = vl;
                    }
                },
                [&](int16_t q) { nbytes += varint_len(code_token(q)); }, [&](uint64_t, uint64_t) {});
        }
        S.bytes[pl][lane] = nbytes;
        if (closes_open) {
            C.closes_open = 1;
            C.close_vlen = close_vlen;
        }
        uint64_t tot;
        const uint64_t excl = plane_sum_scan(nbytes, S, pl, tot);
        const uint64_t bstart = C.out_pos + excl;
        S.bstart[pl][lane] = bstart;
        if (lane == 0) {
            C.iter_bytes = tot;
            // where the run carried into this iteration ends up
            C.carry_tok = C.out_pos;
            C.mv_bytes = 0;
            C.mv_shift = 0;
        }
        __syncthreads();
        if (lane == 0) {
            if (C.open_ty != TY_NONE && C.closes_open) {
                C.carry_w = C.out_pos + C.close_vlen;
                if (C.open_ty == TY_W && C.open_vmax > C.close_vlen) {
                    C.mv_bytes = 8 * (base - C.open_start);
                    C.mv_shift = C.open_vmax - C.close_vlen;
                }
            } else {
                C.carry_w = C.open_w;
            }
        }
        __syncthreads();

        // 8. slide words of a carried W run left if its varint came out shorter
        if (tid == 0) {
            S.mvmax = max(S.carry[0].mv_bytes, a.planes > 1 ? S.carry[1].mv_bytes : 0);
            if (a.counters && S.mvmax) atomicAdd(&a.counters[2], (unsigned long long)S.mvmax);
        }
        __syncthreads();
        for (uint64_t o = 0; o < S.mvmax; o += PLANE_LANES * 8) {
            uint8_t tmp[8];
            const uint64_t src0 = C.out_pos + C.open_vmax + o + lane * 8;
            int m = 0;
            if (o + lane * 8 < C.mv_bytes) {
                m = (int)umin64(8, C.mv_bytes - o - lane * 8);
                for (int i = 0; i < m; ++i) tmp[i] = out[src0 + i];
            }
            __syncthreads();
            for (int i = 0; i < m; ++i) out[src0 - C.mv_shift + i] = tmp[i];
            __syncthreads();
        }

        // 9. write tokens.  The lane that closes a run writes its varint and
        //    the words of its own elements; runs that span lanes publish their
        //    token/word position under the lane they started in (unique: a
        //    lane has at most one run reaching past its end).
        {
            uint64_t pos = bstart;
            lane_walk(
                cl, cnt, e0, in_ty, in_st, tail_closes, lane == 0,
                [&](int t, uint64_t st, uint64_t end) {
                    const uint64_t len = end - st;
                    const uint64_t v = run_token(LOSSY, t, len);
                    const int vl = varint_len(v);
                    put_varint(out + pos, v);
                    if (t == TY_W) {
                        for (uint64_t k = (st > e0 ? st : e0); k < end; ++k)
                            put_word(out + pos + vl + 8 * (k - st),
                                     (uint64_t)__double_as_longlong(xl[k - e0]));
                    }
                    if (st < e0 && st >= base) {
                        const int sl = (int)((st - base) / SUB);
                        S.runtok[pl][sl] = pos;
                        S.runw[pl][sl] = pos + vl;
                    }
                    pos += vl + (t == TY_W ? 8 * len : 0);
                },
                [&](int16_t q) {
                    const uint64_t v = code_token(q);
                    put_varint(out + pos, v);
                    pos += varint_len(v);
                },
                [&](uint64_t, uint64_t) {});
            // a run left open at the end of the iteration starts right after all closed tokens
            if (lane + 1 == active && !final_iter && tail_ty != TY_NONE && tail_st >= base) {
                const uint64_t tokpos = C.out_pos + C.iter_bytes;
                const uint64_t vmax = tail_ty == TY_W ? varint_len(run_token(LOSSY, TY_W, n - tail_st)) : 0;
                const int sl = (int)((tail_st - base) / SUB);
                S.runtok[pl][sl] = tokpos;
                S.runw[pl][sl] = tokpos + vmax;
            }
        }
        __syncthreads();

        // 10. words of a W run that reaches past this lane (closed later, or
        //     carried into the next iteration)
        if (cnt > 0 && tail_ty == TY_W && !tail_closes) {
            const uint64_t wb = tail_st < base ? C.carry_w : S.runw[pl][(tail_st - base) / SUB];
            for (uint64_t k = (tail_st > e0 ? tail_st : e0); k < e0 + cnt; ++k)
                put_word(out + wb + 8 * (k - tail_st), (uint64_t)__double_as_longlong(xl[k - e0]));
        }

        // 11. side index
        if (cnt > 0) {
            SideEntry se;
            const int t0 = ty16(cl[0]);
            if (in_ty != TY_NONE && t0 == in_ty) {
                se.off = (uint32_t)(in_st < base ? C.carry_tok : S.runtok[pl][(in_st - base) / SUB]);
                se.skip = (uint32_t)(e0 - in_st);
            } else {
                bool full = t0 != TY_C;
                for (int i = 1; i < cnt && full; ++i) full = ty16(cl[i]) == t0;
                const bool emitted_here = !full || tail_closes;
                uint64_t cover = bstart;
                if (lane == 0 && in_ty != TY_NONE) {  // carried run closed at e0 precedes us
                    const uint64_t len = e0 - in_st;
                    cover += varint_len(run_token(LOSSY, in_ty, len)) + (in_ty == TY_W ? 8 * len : 0);
                }
                se.off = (uint32_t)(emitted_here ? cover : S.runtok[pl][lane]);
                se.skip = 0;
            }
            se.pred = LOSSY ? S.entryP[pl][lane] : 0.0;
            side[e0 / SUB] = se;
        }

        // 12. carry to the next iteration
        __syncthreads();
        if (lane == 0 && active > 0) {
            const int last = active - 1;
            C.P = LOSSY ? C.Pnext : 0.0;
            C.xprev = C.xprev_next;
            const uint64_t new_pos = C.out_pos + C.iter_bytes;
            // state of the run open after the last lane
            int oty = C.open_ty;
            uint64_t ost = C.open_start;
            fn_apply(S.fincl[pl][last], oty, ost);
            if (final_iter || oty == TY_NONE) {
                C.open_ty = TY_NONE;
            } else if (ost < base) {
                // the old carried run is still open: keep its reservation
            } else {
                C.open_ty = oty;
                C.open_start = ost;
                C.open_vmax = oty == TY_W ? varint_len(run_token(LOSSY, TY_W, n - ost)) : 0;
                C.open_w = new_pos + C.open_vmax;
            }
            C.out_pos = new_pos;
            C.closes_open = 0;
        }
        __syncthreads();
    }

    if (lane == 0 && pact) a.out_len[(uint64_t)b * 2 + pl] = C.out_pos;
    if (tid == 0 && a.sumsq) a.sumsq[b] = S.s;
}

// ---------------------------------------------------------------------------
// Decoder: one lane per sub-chunk, started from its side entry.
// ---------------------------------------------------------------------------
struct PlaneRef {
    const uint8_t* payload;
    uint64_t len;
    int codec;
    double delta;
};

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
