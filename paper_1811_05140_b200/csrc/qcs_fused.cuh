// Fused per-gate kernel: decompress -> scale -> gate -> snap -> recompress
// (+ stored sum of squares, side index) in ONE kernel per ladder level.
//
// Restates, per unit of make_stride_plan (gate.cpp:313-403), the body of
// CompressedState::apply_gate's worker loop (aalc.cpp:315-382):
//   decompress_into + scale   aalc.cpp:176-189, codec.cpp:288-340
//   run_plan_unit             gate.cpp:405-454 (apply_pair order, no FMA)
//   snap_zeros                core.cpp:39-47
//   compress (one ladder level) codec.cpp:118-250
//   stored_sum_sq             aalc.cpp:46-52, core.cpp:30-37
// MODE_LOCAL keeps everything on chip between the compressed input and the
// compressed output.  MODE_RAW encodes planes already decompressed and gated
// into HBM (k_decode_gate, the split path for cross-chunk partners; or the
// codec API's input).
//
// CTA shapes (template NPL planes x LPL lanes, SUB = 32 elements per lane):
//   2 x 128  one stride per CTA, two CTAs per SM (the usual case)
//   2 x 256  one stride per CTA, one per SM: gates with fewer units than SMs
//   1 x 256  codec API, one plane
// The encoder: self-correcting event rounds over lane-serial reference
// chains, an exact emulation of the stored sum of squares, and a bitmask
// tokenizer.
#pragma once

#include "qcs_codec.cuh"

namespace qcs {

constexpr int GRP = 4;  // elements per independent group in the chain loops

enum : int { MODE_RAW = 0, MODE_LOCAL = 1 };

// Shared state of one encoder CTA with NT = planes x lanes threads.
template <int NT>
struct FusedSharedT {
    double entryP[NT];
    double exitP[NT];
    RunFn fincl[NT];
    uint64_t bstart[NT];
    uint64_t runtok[NT];
    uint64_t runw[NT];
    int8_t ftype[NT + 8];
    RunFn wfn[NT / 32];
    long long wesc_i[NT / 32];
    double wesc_v[NT / 32];
    uint64_t wsum[NT / 32];
    long long wmin[NT / 32];
    PlaneCarry carry[4];
    double s[2];  // exact running sum of squares per stride
    double s_pre;  // fused_sumsq's serial prefix (not s[0]: every thread reads s[0] on entry)
    uint64_t bar[4];  // per-plane mbarrier of the payload bulk copy (MODE_LOCAL)
    uint8_t repaired[NT];  // lane's codes rewritten by a repair pass (resync chain)
};

// code rows padded to 34 int16 (17 words) so the lanes' row accesses (32-bit
// pairs in lane_masks, 16-bit in the chain) hit distinct banks
constexpr int CODE_STRIDE = SUB + 2;
template <int NT>
struct FusedLayout {
    static constexpr size_t XS_BYTES = sizeof(double) * NT * XS_STRIDE;
    static constexpr size_t CODE_BYTES = sizeof(int16_t) * NT * CODE_STRIDE;
    static constexpr size_t S_OFF = (XS_BYTES + CODE_BYTES + 15) & ~size_t(15);
    static constexpr size_t SMEM = S_OFF + sizeof(FusedSharedT<NT>);
};
static_assert(FusedLayout<256>::SMEM <= 113 * 1024, "two 256-thread encoder CTAs per SM");
static_assert(FusedLayout<512>::SMEM <= 227 * 1024, "one 512-thread encoder CTA per SM");

struct FusedArgs {
    // ---- input: block store (MODE_LOCAL/FAR/PAIR) ----
    const uint8_t* arena0;        // the two payload arenas
    const uint8_t* arena1;
    const int* arena_cur;         // device scalar: which one is live
    const uint64_t* p_off;
    const uint64_t* p_len;
    const int8_t* p_codec;
    const double* p_delta;
    const SideEntry* side_in;     // [plane][nsub]
    const double* scale;          // [stride]
    const uint64_t* job_stride;   // [slot]
    // ---- input: raw planes (MODE_RAW) ----
    const double* X;
    uint64_t x_plane_stride;      // elements between a CTA's planes
    // ---- serial-chain mode (non-power-of-two bounds) ----
    double* dump_x;               // MODE_LOCAL: write the gated, snapped planes
                                  // here ([slot][plane][n]) and stop
    const int16_t* pre_codes;     // MODE_RAW: the reference chain's codes,
    const double* pre_pred;       // [slot][plane][n] and its predictor entering
                                  // every sub-chunk [slot][plane][nsub]
                                  // (k_serial_chain); no event rounds
    const int* chain_on;          // device flag gating pre_codes (null = always)
    // zero-imaginary-plane mode: per global slot, 1 = the slot's output im
    // plane is identically zero (real gate, zero input im planes); the CTA
    // then encodes the re plane with all its lanes and writes the im plane's
    // one-token encoding directly (null = off)
    const uint8_t* im_zero;
    // zero-stride pass: per global slot, 1 = the slot's output stride is all
    // zero (k_make_jobs); the CTA writes both planes' zero encodings only
    const uint8_t* zero_slot;
    const uint32_t* order;        // [slot] CTA -> global slot within each launch (null = identity)
    const int* err;               // device error word (non-zero: the gate failed or is suspended; no-op)
    double ladder_theta;          // > 0: a level before the last; give up once theta is out of reach
    // ---- gate ----
    double u[8];
    int kind;                     // GateKind
    // diagonal gate (u12 = u21 = 0) on far partners, MODE_LOCAL: every element
    // is gated on its own (0 = pairs inside the chunk; 1 = in-stride target,
    // the side is bit t of the element; 2 = pair unit, the side is the slot's)
    int diag;
    int t;                        // target (in-stride bit for LOCAL/FAR)
    int local_ctl;                // in-stride control bit, -1 none
    uint64_t flip_off;
    const double* mean;           // reflect_mean: {re, im}
    // ---- encoder ----
    uint64_t n;                   // elements per plane (stride length)
    const uint8_t* pending;       // per slot (null = all)
    const uint8_t* redo_only;     // per slot (null = all): only the slots the streaming kernel left (qcs_stream.cuh)
    int max_rounds;               // event rounds before the neighbour-exit repair (>= 1)
    int pool;                     // small layout: out / side / side_in are the plane
                                  // slot pools (two slots per plane, p_off selects)
    uint64_t slot_base;           // first slot of this launch (tables are global,
                                  // out / side / X buffers are launch-local)
    int snap;
    uint8_t* out;
    uint64_t cap;
    SideEntry* side;              // output side entries per slot plane
    uint64_t nsub;
    uint64_t* out_len;
    double* sumsq;
    CodecParams cp;
    unsigned long long* counters;
    unsigned long long* cta_trace;  // debug: [global slot][8] phase cycles (null = off)
};

template <int LPL>
__device__ __forceinline__ double& xrow(double* xs, int row_plane, int k)
{
    return xs[(row_plane * LPL + (k >> 5)) * XS_STRIDE + (k & 31)];
}

// n consecutive little-endian words (the doubles' bits) at an arbitrary byte
// address: byte stores for the unaligned head and tail, 8-byte aligned
// stores for the body (each built from two neighbouring words).
__device__ __forceinline__ void put_words(uint8_t* p, const double* v, int n)
{
    if (n <= 0) return;
    const int r = (int)(reinterpret_cast<uintptr_t>(p) & 7u);
    auto w = [&](int j) { return (uint64_t)__double_as_longlong(v[j]); };
    if (r == 0) {
        uint64_t* q = reinterpret_cast<uint64_t*>(p);
        for (int j = 0; j < n; ++j) q[j] = w(j);
        return;
    }
    const int d = 8 - r;  // bytes of word 0 before the first 8-byte boundary
    uint64_t cur = w(0);
    for (int i = 0; i < d; ++i) p[i] = (uint8_t)(cur >> (8 * i));
    uint64_t* q = reinterpret_cast<uint64_t*>(p + d);
    for (int j = 0; j + 1 < n; ++j) {
        const uint64_t nxt = w(j + 1);
        q[j] = (cur >> (8 * d)) | (nxt << (8 * r));
        cur = nxt;
    }
    uint8_t* t = p + d + 8 * (n - 1);
    for (int i = 0; i < r; ++i) t[i] = (uint8_t)(cur >> (8 * (d + i)));
}

// ---- scans over the WPL warps of one plane --------------------------------
template <int WPL, typename FS>
__device__ __forceinline__ RunFn fscan_fn(RunFn F, FS& S, int pl)
{
    const int wl = threadIdx.x & 31, w = threadIdx.x >> 5;
    RunFn inc = F;
    for (int o = 1; o < 32; o <<= 1) {
        RunFn u;
        u.kt = __shfl_up_sync(0xffffffffu, inc.kt, o);
        u.st = __shfl_up_sync(0xffffffffu, inc.st, o);
        if (wl >= o) inc = fn_compose(u, inc);
    }
    __syncthreads();
    if (wl == 31) S.wfn[w] = inc;
    __syncthreads();
    RunFn pre{0, 0};
    for (int i = pl * WPL; i < w; ++i) pre = fn_compose(pre, S.wfn[i]);
    return fn_compose(pre, inc);
}

template <int WPL, typename FS>
__device__ __forceinline__ uint64_t fscan_sum(uint64_t v, FS& S, int pl, uint64_t& total)
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
    for (int i = pl * WPL; i < pl * WPL + WPL; ++i) {
        if (i < w) pre += S.wsum[i];
        tot += S.wsum[i];
    }
    total = tot;
    return pre + inc - v;
}

template <int WPL, typename FS>
__device__ __forceinline__ long long fscan_last(long long idx, double val, FS& S, int pl,
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
        for (int k = w - 1; k >= pl * WPL; --k) {
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

// ---- exact stored sum of squares over a stride group ------------------------
// group g = planes (2g, 2g+1), threads [g*GT, (g+1)*GT), GT = 2*LPL; each thread
// owns 16 consecutive elements of the chunk.  Same algorithm as
// the integer-sum argument of DESIGN.md §4, restricted to the group's warps.
// IMZ: the im plane is identically zero (re^2 + 0*0, the reference's sum)
template <int LPL, bool IMZ = false>
__device__ __forceinline__ double tsq_g(double* xs, int g, int k)
{
    const double r = xrow<LPL>(xs, 2 * g, k);
    if (IMZ) return __dmul_rn(r, r);  // fl(r*r + 0*0) == fl(r*r): r*r >= +0
    const double i = xrow<LPL>(xs, 2 * g + 1, k);
    return __dadd_rn(__dmul_rn(r, r), __dmul_rn(i, i));
}

// units of 2^(e-52) of one term x*x (tu = 2^(52-e)); a tie or a term beyond
// the binade saturates
__device__ __forceinline__ uint64_t sq_units_y(double y)
{
    const double ry = rint(y);
    return (y >= 9007199254740992.0 || fabs(y - ry) == 0.5) ? (1ull << 62) : (uint64_t)ry;
}
__device__ __forceinline__ uint64_t sq_units(double x, double tu) { return sq_units_y(__dmul_rn(x, x) * tu); }

// pre_ok: every thread's units over its own elements for the binade of the
// entering sum are already in pre_loc (IMZ: formed during reconstruction)
template <int LPL, bool IMZ, typename FS>
__device__ __forceinline__ void fused_sumsq(double* xs, int n_it, FS& S, unsigned long long* counters,
                                            bool pre_ok = false, uint64_t pre_loc = 0)
{
    constexpr int GT = IMZ ? LPL : 2 * LPL;  // threads (the CTA: one stride)
    constexpr int GW = GT / 32;            // warps
    constexpr int PER = (LPL * SUB) / GT;  // 16 elements per thread
    constexpr uint64_t SAT = 1ull << 62;
    const int tid = threadIdx.x;
    const int wl = tid & 31, w = tid >> 5;
    const int kb = tid * PER;
    // (entered right after a CTA barrier: every step-4 branch ends with one)
    double s = S.s[0];  // uniform across the CTA from here on
    int k0 = 0;
#ifdef QCS_WATCHDOG
    if ((tid & 31) == 31 && !(s == 0.0) && n_it <= 512)
        printf("[qcs watchdog] sumsq entry block %d tid %d s=%a n_it=%d imz=%d\n", (int)blockIdx.x, tid, s, n_it, (int)IMZ);
#endif
    // While s is still 0 the next elements double it again and again (a binade
    // crossing, i.e. a parallel pass, per doubling): sum the first SERIAL_SUM
    // elements of a stride in the reference's order on one thread instead.
    constexpr int SERIAL_SUM = 512;
    if (s == 0.0) {
        const int m = min(n_it, SERIAL_SUM);
        // (written to s_pre: a thread still to read s[0] on entry would see
        // the prefix and skip this branch — a read-after-write race)
        if (tid == 0) {
            double acc = 0.0;
#pragma unroll 4
            for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, tsq_g<LPL, IMZ>(xs, 0, k));
            S.s_pre = acc;
        }
        __syncthreads();
        s = S.s_pre;
        k0 = m;
    }
#ifdef QCS_WATCHDOG
    int wd_passes = 0;
#endif
    while (k0 < n_it) {
#ifdef QCS_WATCHDOG
        if (++wd_passes > 100000 && (tid & 31) == 0)
            printf("[qcs watchdog] fused_sumsq block %d tid %d s=%a k0=%d n_it=%d S.s0=%a imz=%d\n", (int)blockIdx.x, tid, s, k0, n_it,
                   S.s[0], (int)IMZ);
        if (wd_passes > 100000) __trap();
#endif
        if (counters && tid == 0) atomicAdd(&counters[1], 1ull);
        long long mine = LLONG_MAX;  // this thread's event candidate
        const int state = s == 0.0 ? 1 : (ilogb(s) < -960 ? 2 : 3);
        if (state == 3) {
            const int e = ilogb(s);
            const double to_units = ldexp(1.0, 52 - e);
            const uint64_t ms = (uint64_t)(s * to_units);
            uint64_t loc = 0;
            if (pre_ok && k0 == 0) {
                loc = pre_loc;
            } else {
                for (int i = 0; i < PER; ++i) {
                    const int k = kb + i;
                    if (k < k0 || k >= n_it) continue;
                    const double y = tsq_g<LPL, IMZ>(xs, 0, k) * to_units;
                    const double ry = rint(y);
                    // a tie (or an element beyond the binade) saturates the total
                    loc = sat_add(loc, (y >= 9007199254740992.0 || fabs(y - ry) == 0.5) ? SAT : (uint64_t)ry);
                }
            }
            uint64_t inc = loc;
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t u = __shfl_up_sync(0xffffffffu, inc, o);
                if (wl >= o) inc = sat_add(inc, u);
            }
            const uint64_t prev = __shfl_up_sync(0xffffffffu, inc, 1);
            // (S.wsum's last readers are behind a barrier already: the
            // caller's, the serial prefix's, or the previous event's)
            if (wl == 31) S.wsum[w] = inc;
            __syncthreads();
            uint64_t pre = 0, total = 0;
            for (int i = 0; i < GW; ++i) {
                if (i < w) pre = sat_add(pre, S.wsum[i]);
                total = sat_add(total, S.wsum[i]);
            }
            if (ms + total < (1ull << 53)) {  // no event: the rest of the iteration
                s = (double)(ms + total) / to_units;  // < 2^53 units: exact
                break;
            }
            // An event (binade crossing or tie) lies in this pass.  It is in
            // the one thread whose inclusive prefix reaches the binade's end
            // (the threads before it hold neither a tie nor the crossing): that
            // thread's warp finds it — one of the thread's elements per lane,
            // a scan of their units and a ballot — and adds it exactly.
            const uint64_t off = sat_add(pre, wl ? prev : 0);
            const uint64_t LIM = (1ull << 53) - ms;
            const unsigned ob = __ballot_sync(0xffffffffu, off < LIM && sat_add(off, loc) >= LIM);
            if (ob) {
                const int ol = __ffs(ob) - 1;
                const uint64_t off_o = __shfl_sync(0xffffffffu, off, ol);
                const int k = (tid - wl + ol) * PER + wl;  // the owner's element of this lane
                const bool valid = wl < PER && k >= k0 && k < n_it;
                const double t = valid ? tsq_g<LPL, IMZ>(xs, 0, k) : 0.0;
                const double y = t * to_units;
                const double ry = rint(y);
                const bool beyond = y >= 9007199254740992.0;
                const bool tie = valid && !beyond && fabs(y - ry) == 0.5;
                const uint64_t c = beyond ? (1ull << 53) : (uint64_t)ry;
                uint64_t incl = c;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t u = __shfl_up_sync(0xffffffffu, incl, o);
                    if (wl >= o) incl += u;
                }
                const bool ev = valid && (beyond || tie || ms + off_o + incl >= (1ull << 53));
                const unsigned eb = __ballot_sync(0xffffffffu, ev);
                if (eb && wl == __ffs(eb) - 1) {
                    S.s[0] = __dadd_rn((double)(ms + off_o + (incl - c)) / to_units, t);
                    S.wmin[0] = k;
                    if (counters) atomicAdd(&counters[tie ? 6 : 7], 1ull);
                }
            }
            __syncthreads();
            s = S.s[0];
            k0 = (int)S.wmin[0] + 1;
        } else if (state == 1) {  // 0 + t = t exactly: the first non-zero term starts the sum
            for (int i = 0; i < PER; ++i) {
                const int k = kb + i;
                if (k >= k0 && k < n_it && tsq_g<LPL, IMZ>(xs, 0, k) != 0.0) {
                    mine = k;
                    break;
                }
            }
            long long m = mine;
            for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
            __syncthreads();
            if (wl == 0) S.wmin[w] = m;
            __syncthreads();
            long long kstar = LLONG_MAX;
            for (int i = 0; i < GW; ++i) kstar = min(kstar, S.wmin[i]);
            if (kstar == LLONG_MAX) break;  // all zero: s stays 0
            s = tsq_g<LPL, IMZ>(xs, 0, (int)kstar);
            k0 = (int)kstar + 1;
        } else {  // far below any practical state: one term at a time, in order
            s = __dadd_rn(s, tsq_g<LPL, IMZ>(xs, 0, k0));
            ++k0;
        }
    }
    __syncthreads();
    if (tid == 0) S.s[0] = s;
}

// The reference chain (LossyEmitter, codec.cpp:153-250) over one lane's c
// elements from predictor Pin: writes the codes, returns the exit predictor
// and the lane's last event (ev_i lane-relative, -1 none; ev_v the predictor
// it set).  For a power-of-two bound a step is PROVEN equal to the reference
// step when, with P = A + 2d*Mprev exactly on the anchor's lattice,
// y = (x-A)/2d has |y| < 2^30, its fractional part is >= 2^-19 away from a
// half and |rint(y) - Mprev| <= 32766 (see lattice_step_m); GRP such steps run
// as a group with independent arithmetic.  Any other step is the reference
// step itself and an event (the anchor moves to its predictor).
// resync: a repair run from the left neighbour's exit; the old codes (from
// entry Pold) give the old chain, and once the new predictor equals the old
// one the rest of the lane is unchanged (synced).
__device__ __forceinline__ double lane_chain(const CodecParams& cp, const double* xr, int16_t* cr, int c, double Pin,
                                             bool resync, double Pold, bool& synced, long long& ev_i, double& ev_v)
{
    double P = Pin, A = Pin, Mprev = 0.0, Po = Pold;
    synced = false;
    ev_i = -1;
    ev_v = 0.0;
    for (int i0 = 0; i0 < c; i0 += GRP) {
        if (cp.pow2 && !resync) {
            double Mv[GRP], Pv[GRP];
            bool ok = true;
#pragma unroll
            for (int k = 0; k < GRP; ++k) {
                const double x = xr[i0 + k];  // rows are padded: i0 + k < 32
                const double y = __dmul_rn(__dsub_rn(x, A), cp.inv_td);
                const double M = rint(y);
                const double fr = fabs(__dsub_rn(y, M));
                const double yv = __dmul_rn(cp.td, M);
                const double v = __dadd_rn(A, yv);
                const double q = __dsub_rn(M, k == 0 ? Mprev : Mv[k - 1]);
                const bool good = fabs(y) < 1073741824.0 && fr < 0.5 - 1.9073486328125e-06 && fabs(q) <= 32766.0 &&
                                  add_exact(A, yv, v);
                ok &= good | (i0 + k >= c);
                Mv[k] = M;
                Pv[k] = v;
            }
            if (ok) {
#pragma unroll
                for (int k = 0; k < GRP; ++k)
                    if (i0 + k < c) {
                        cr[i0 + k] = (int16_t)__dsub_rn(Mv[k], k == 0 ? Mprev : Mv[k - 1]);
                        P = Pv[k];
                        Mprev = Mv[k];
                    }
                continue;
            }
        }
        for (int i = i0; i < i0 + GRP && i < c; ++i) {
            const double x = xr[i];
            if (resync) {  // the old chain's predictor after this element
                const int16_t co = cr[i];
                if (co == WCODE16) Po = x;
                else if (co != 0) Po = __dadd_rn(Po, __dmul_rn(cp.td, (double)co));
            }
            bool done = false;
            if (cp.pow2) {
                const double y = __dmul_rn(__dsub_rn(x, A), cp.inv_td);
                const double M = rint(y);
                const double fr = fabs(__dsub_rn(y, M));
                const double q = __dsub_rn(M, Mprev);
                if (fabs(y) < 1073741824.0 && fr < 0.5 - 1.9073486328125e-06 && fabs(q) <= 32766.0) {
                    const double yv = __dmul_rn(cp.td, M);
                    const double v = __dadd_rn(A, yv);
                    cr[i] = (int16_t)q;
                    P = v;
                    if (add_exact(A, yv, v)) {
                        Mprev = M;
                    } else {  // the chain rounds here: re-anchor
                        A = v;
                        Mprev = 0.0;
                        ev_i = i;
                        ev_v = v;
                    }
                    done = true;
                }
            }
            if (!done) {
                const int32_t k = ref_step(cp, P, x);
                cr[i] = k == WCODE ? WCODE16 : (int16_t)k;
                A = P;  // re-anchor at the reference predictor
                Mprev = 0.0;
                ev_i = i;
                ev_v = P;
            }
            if (resync && same_bits(P, Po)) {
                synced = true;
                return P;
            }
        }
    }
    return P;
}

// Per-phase cycle accounting (thread 0 of each CTA) into counters[8..15].
#define QCS_PHASE(id)                                                        \
    do {                                                                     \
        if (tid == 0 && a.counters) {                                        \
            const long long now_ = clock64();                                \
            ph_acc[id] += (unsigned long long)(now_ - ph_t);                 \
            ph_t = now_;                                                     \
        }                                                                    \
    } while (0)

// An all-zero plane's encoding: one zero run of n elements (lossless
// codec.cpp:129-145 / lossy :224-247 both emit a single run token); every
// sub-chunk starts inside it with predictor 0.  Written by nt threads.
template <bool LOSSY>
__device__ __forceinline__ void write_zero_plane(const FusedArgs& a, uint64_t slot, uint64_t gslot, int comp, int tid,
                                                 int nt)
{
    uint8_t* o;
    SideEntry* sd;
    if (a.pool) {
        const uint64_t g = 2 * a.job_stride[gslot] + comp;
        const int ls = (int)((a.p_off[g] / a.cap) & 1);
        o = a.out + (2 * g + 1 - ls) * a.cap;
        sd = a.side + (2 * g + 1 - ls) * a.nsub;
    } else {
        o = a.out + (2 * slot + comp) * a.cap;
        sd = a.side + (2 * slot + comp) * a.nsub;
    }
    const uint64_t n = a.n;
    const uint64_t tok = run_token(LOSSY, TY_Z, n);
    if (tid == 0) {
        put_varint(o, tok);
        a.out_len[2 * gslot + comp] = (uint64_t)varint_len(tok);
    }
    const uint64_t nsub_n = (n + SUB - 1) / SUB;
    for (uint64_t sc = tid; sc < nsub_n; sc += nt) {
        SideEntry se;
        se.off = 0;
        se.skip = (uint32_t)(sc * SUB);
        se.pred = 0.0;
        sd[sc] = se;
    }
}

// The encoder body.  IMZ (zero-imaginary-plane mode): NPL = 1 and the CTA's
// LPL lanes all work on the re plane of a stride whose im plane is zero
// before and after the gate; the im plane's encoding (one zero-run token) is
// written directly.
template <bool LOSSY, int NPL, int LPL, int MODE, bool IMZ>
__device__ __forceinline__ void fused_body(const FusedArgs& a, const int b)
{
    unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long ph_t = clock64();
    constexpr int ITP = LPL * SUB;   // elements per plane per CTA iteration
    constexpr int WPL = LPL / 32;    // warps per plane
    const int tid = threadIdx.x;
    const int pl = tid / LPL;
    const int lane = tid % LPL;
    // output slot of this plane
    const uint64_t slot = (uint64_t)b;
    const int comp = pl;
    const uint64_t gslot = a.slot_base + slot;  // global slot (tables)
    const uint64_t row = IMZ ? 2 * slot : (uint64_t)b * NPL + pl;  // launch-local plane row (X, scratch)
    if (a.pending && !a.pending[a.slot_base + (uint64_t)b]) return;

    extern __shared__ __align__(16) unsigned char smem[];
    double* xs = reinterpret_cast<double*>(smem);
    using FS = FusedSharedT<NPL * LPL>;
    using LY = FusedLayout<NPL * LPL>;
    int16_t* code = reinterpret_cast<int16_t*>(smem + LY::XS_BYTES);
    FS& S = *reinterpret_cast<FS*>(smem + LY::S_OFF);

    const CodecParams cp = a.cp;
    const uint64_t n = a.n;
    uint8_t* out;
    SideEntry* side;
    int live_sel = 0;
    if (a.pool) {  // write the plane's other slot; the commit flips
        const uint64_t g = 2 * a.job_stride[gslot] + comp;
        live_sel = (int)((a.p_off[g] / a.cap) & 1);
        out = a.out + (2 * g + 1 - live_sel) * a.cap;
        side = a.side + (2 * g + 1 - live_sel) * a.nsub;
    } else {
        out = a.out + (2 * slot + comp) * a.cap;
        side = a.side + (2 * slot + comp) * a.nsub;
    }
    double* xl = xs + (pl * LPL + lane) * XS_STRIDE;
    int16_t* cl = code + (pl * LPL + lane) * CODE_STRIDE;
    PlaneCarry& C = S.carry[pl];

    // input plane of this thread (block store modes)
    uint64_t in_stride = 0;
    const uint8_t* in_bytes = nullptr;
    int in_codec = 0;
    double in_td = 0.0, in_scale = 1.0;
    const SideEntry* in_side = nullptr;
    const double* xg = nullptr;
    if (MODE == MODE_RAW) {
        xg = a.X + row * a.x_plane_stride;
    } else {
        in_stride = a.job_stride[gslot];
        const uint64_t gpl = 2 * in_stride + comp;
        in_bytes = (*a.arena_cur ? a.arena1 : a.arena0) + a.p_off[gpl];
        in_codec = a.p_codec[gpl];
        in_td = 2.0 * a.p_delta[gpl];
        in_scale = a.scale[in_stride];
        in_side = a.pool ? a.side_in + (2 * gpl + live_sel) * a.nsub : a.side_in + gpl * a.nsub;
    }
    double m8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m8[i] = a.u[i];
    const uint64_t hb = MODE == MODE_LOCAL && a.kind <= 1 ? (1ull << a.t) : 0;

    if (lane == 0) {
        C.P = 0.0;
        C.xprev = 0.0;
        C.out_pos = 0;
        C.open_ty = TY_NONE;
        C.open_start = 0;
        C.open_vmax = 0;
        C.open_w = 0;
        C.closes_open = 0;
    }
    if (tid < 2) S.s[tid] = 0.0;
    if (MODE == MODE_LOCAL && tid < NPL) mbar_init(&S.bar[tid], 1);
    unsigned stage_phase = 0;  // parity of this plane's next bulk copy
    __syncthreads();

    for (uint64_t base = 0; base < n; base += ITP) {
        const uint64_t e0 = base + (uint64_t)lane * SUB;
        const int cnt = e0 < n ? (int)umin64(SUB, n - e0) : 0;
        const bool final_iter = base + ITP >= n;
        const int active = (int)umin64(LPL, (n - base + SUB - 1) / SUB);
        const int n_it = (int)umin64(ITP, n - base);

        // 1. input: decode (+ gate) or raw load, then snap_zeros
        if (MODE == MODE_RAW) {
            // pull the NEXT chunk of this plane towards L2 while this one is
            // processed (one bulk prefetch per plane; no shared memory needed)
            if (lane == 0 && base + ITP < n) {
                const uint64_t nb = umin64((uint64_t)ITP, n - base - ITP) * 8;
                if ((nb & 15) == 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(xg + base + ITP), "r"((unsigned)nb)
                                 : "memory");
            }
#pragma unroll 8
            for (int i = lane; i < ITP; i += LPL) {
                double* dst = &xrow<LPL>(xs, pl, i);
                if (base + i < n) {
                    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(xg + base + i)
                                 : "memory");
                } else {
                    *dst = 0.0;
                }
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncthreads();
        } else {
            // Stage this iteration's payload bytes of the plane in shared memory
            // (the code buffer is free until the chain runs) with one TMA bulk
            // copy (cp.async.bulk + mbarrier), so the lanes' serial token walks read shared
            // memory instead of waiting on L2 per byte.  The range runs from
            // the token covering the iteration's first element to the token
            // covering the next iteration's first one, plus that token's
            // varint and the words it owns for this iteration's elements.
            const uint8_t* src = in_bytes;
            bool staged = false;
            if (MODE == MODE_LOCAL) {
                // staging room: everything dead between an iteration's end
                // and its decode — the code rows, and the per-iteration lane
                // arrays at the head of S (entryP .. runw).  One plane in the
                // CTA: all of it; two: the code rows for plane 0, the lane
                // arrays for plane 1
                uint8_t* const lane_arrays = reinterpret_cast<uint8_t*>(&S.entryP[0]);
                uint8_t* const lane_end = reinterpret_cast<uint8_t*>(&S.ftype[0]);
                uint8_t* stage;
                uint64_t STAGE;
                if (NPL == 1) {
                    stage = reinterpret_cast<uint8_t*>(code);
                    STAGE = (uint64_t)(lane_end - stage) & ~uint64_t(15);
                } else if (pl == 0) {
                    stage = reinterpret_cast<uint8_t*>(code);
                    STAGE = LY::CODE_BYTES & ~size_t(15);
                } else {
                    stage = lane_arrays;
                    STAGE = (uint64_t)(lane_end - lane_arrays) & ~uint64_t(15);
                }
                const uint64_t sc0 = base / SUB;
                const uint64_t lo = in_side[sc0].off & ~uint64_t(15);
                uint64_t hi;
                if (final_iter) {
                    hi = a.p_len[2 * in_stride + comp];
                } else {
                    const SideEntry nx = in_side[sc0 + LPL];
                    hi = (uint64_t)nx.off + 10 + 8 * (uint64_t)nx.skip;
                }
                const uint64_t nb = hi > lo ? ((hi - lo + 15) & ~uint64_t(15)) : 0;
                if (nb > 0 && nb <= STAGE) {  // uniform over the plane's lanes
                    // one TMA bulk copy per plane (payloads start 16-byte
                    // aligned; the code rows are free: the previous
                    // iteration ended with a barrier)
                    if (lane == 0) bulk_g2s(stage, in_bytes + lo, (unsigned)nb, &S.bar[pl]);
                    mbar_wait(&S.bar[pl], stage_phase);
                    stage_phase ^= 1u;
                    src = stage - lo;  // token offsets stay plane-relative
                    staged = true;
                }
            }
            if (cnt > 0) {
                if (staged && !IMZ)  // measured: helps two-plane CTAs (C1), not whole-CTA re planes (C2)
                    decode_sub_win(src, in_codec, in_td, in_side[e0 / SUB], cnt, xl, in_scale);
                else
                    decode_sub(src, in_codec, in_td, in_side[e0 / SUB], cnt, xl, in_scale);
            }
            __syncthreads();
            // gate (run_plan_unit, gate.cpp:405-454)
            {  // MODE_LOCAL
                if (a.kind <= 1 && a.diag) {
                    // A diagonal unitary's apply_pair (gate.cpp:153-162) adds the
                    // partner's terms multiplied by exact zeros: for a non-zero
                    // result they vanish exactly, a zero result is snapped to
                    // +0.0 (core.cpp:39-47) whatever its sign -- so each side is
                    // apply_pair with a zero partner, bit for bit after the snap
                    const int fixed_side = a.diag == 2 ? (int)(gslot & 1) : -1;
                    for (int i = tid; i < n_it; i += NPL * LPL) {
                        const uint64_t gi = base + (uint64_t)i;
                        if (a.local_ctl >= 0 && !((gi >> a.local_ctl) & 1)) continue;
                        const int side = fixed_side >= 0 ? fixed_side : (int)((gi >> a.t) & 1);
                        double& xr = xrow<LPL>(xs, 0, i);
                        double xi_ = IMZ ? 0.0 : xrow<LPL>(xs, 1, i);
                        double orr, oi;
                        if (side == 0) pair_lo(m8, xr, xi_, 0.0, 0.0, orr, oi);
                        else pair_hi(m8, 0.0, 0.0, xr, xi_, orr, oi);
                        xr = orr;
                        if (!IMZ) xrow<LPL>(xs, 1, i) = oi;
                    }
                } else if (a.kind <= 1) {
                    const uint64_t lo_mask = hb - 1;
                    for (int q = tid; q < n_it / 2; q += NPL * LPL) {
                        const int i0 = (int)((((uint64_t)q & ~lo_mask) << 1) | ((uint64_t)q & lo_mask));
                        const int i1 = i0 | (int)hb;
                        if (a.local_ctl >= 0 && !(((base + i0) >> a.local_ctl) & 1)) continue;
                        if (IMZ) {  // the reference's arithmetic with zero im inputs
                            double z0 = 0.0, z1 = 0.0;
                            pair_update(m8, xrow<LPL>(xs, 0, i0), z0, xrow<LPL>(xs, 0, i1), z1);
                        } else {
                            pair_update(m8, xrow<LPL>(xs, 0, i0), xrow<LPL>(xs, 1, i0), xrow<LPL>(xs, 0, i1),
                                        xrow<LPL>(xs, 1, i1));
                        }
                    }
                } else if (a.kind == 2) {
                    if (tid == 0 && a.flip_off >= base && a.flip_off < base + n_it) {
                        const int k = (int)(a.flip_off - base);
                        xrow<LPL>(xs, 0, k) = -xrow<LPL>(xs, 0, k);
                        if (!IMZ) xrow<LPL>(xs, 1, k) = -xrow<LPL>(xs, 1, k);
                    }
                } else {
                    const double mr2 = 2.0 * a.mean[0], mi2 = 2.0 * a.mean[1];
                    for (int i = tid; i < n_it; i += NPL * LPL) {
                        xrow<LPL>(xs, 0, i) = __dsub_rn(mr2, xrow<LPL>(xs, 0, i));
                        if (!IMZ) xrow<LPL>(xs, 1, i) = __dsub_rn(mi2, xrow<LPL>(xs, 1, i));
                    }
                }
            }
            __syncthreads();
        }
        if (a.snap && cnt > 0) {
            for (int i = 0; i < cnt; ++i) xl[i] = snap(xl[i]);
        }
        if (MODE == MODE_LOCAL && a.dump_x) {  // serial-chain mode: input only
            double* dx = a.dump_x + row * n + e0;
            for (int i = 0; i < cnt; ++i) dx[i] = xl[i];
            __syncthreads();
            continue;
        }
        __syncthreads();

        QCS_PHASE(0);
        bool pre_ok = false;   // IMZ: this thread's first-pass sum units ...
        uint64_t pre_loc = 0;  // ... formed during reconstruction
        // 2-4. codes and exact predictors
        if (LOSSY && MODE == MODE_RAW && a.pre_codes && (!a.chain_on || *a.chain_on)) {
            // serial-chain mode: the codes and sub-chunk entry predictors of
            // the reference chain were computed by k_serial_chain
            if (cnt > 0) {
                const int16_t* pc = a.pre_codes + row * n + e0;
                for (int i = 0; i < cnt; ++i) cl[i] = pc[i];
                const double P0 = a.pre_pred[row * a.nsub + e0 / SUB];
                S.entryP[tid] = P0;
                double P = P0;
                for (int i = 0; i < cnt; ++i) {  // reconstructed values
                    const int16_t co = cl[i];
                    if (co == WCODE16) P = xl[i];
                    else if (co != 0) P = __dadd_rn(P, __dmul_rn(cp.td, (double)co));
                    xl[i] = P;
                }
            }
            __syncthreads();
        } else if (LOSSY) {
            // Self-correcting event rounds.  Every lane runs the
            // reference chain from an entry predictor derived from the last
            // EVENT before it (an escape, a rounding re-anchor or any step the
            // lattice test could not prove — the anchors the chain's predictor
            // is exactly defined by).  Round 0 uses predicted escapes as events;
            // later rounds the events the lanes' chains actually produced, and
            // only lanes whose entry changes re-run.  The chain is exact when
            // its entry is, so when every lane's entry equals its left
            // neighbour's exit the iteration is the reference's.  By induction
            // each round fixes at least the first wrong lane; after max_rounds
            // the remaining lanes are repaired from their neighbours' exits.
            if (cnt > 0 && lane + 1 == active) C.xprev_next = xl[cnt - 1];
            const double x_left = cnt > 0 ? (lane == 0 ? C.xprev : xrow<LPL>(xs, pl, lane * SUB - 1)) : 0.0;
            long long ev_idx = -1;  // this lane's last event (absolute index)
            double ev_val = 0.0;
            {
                double xp = x_left;
                for (int i = 0; i < cnt; ++i) {
                    const double x = xl[i];
                    if (predict_escape(cp, x, xp)) {
                        ev_idx = (long long)e0 + i;
                        ev_val = x;
                    }
                    xp = x;
                }
            }
            double used = __longlong_as_double(0x7ff8000000000000ll);  // entry of the last run
            S.repaired[tid] = 0;
            for (int round = 0;; ++round) {
                double aval = 0.0;
                const long long aidx = fscan_last<WPL>(cnt > 0 ? ev_idx : -1, ev_val, S, pl, aval);
                if (cnt > 0) {
                    const double A = aidx >= 0 ? aval : C.P;
                    const long long Aidx = aidx >= 0 ? aidx : (long long)base - 1;
                    const double entry = (Aidx == (long long)e0 - 1) ? A : lattice_point(cp, A, x_left);
                    if (!same_bits(entry, used)) {
                        used = entry;
                        bool sy;
                        long long li = -1;
                        double lv = 0.0;
                        S.exitP[tid] = lane_chain(cp, xl, cl, cnt, entry, false, 0.0, sy, li, lv);
                        if (li >= 0) {
                            ev_idx = (long long)e0 + li;
                            ev_val = lv;
                        } else {
                            ev_idx = -1;
                        }
                    }
                    S.entryP[tid] = used;
                }
                __syncthreads();
                const bool bad = cnt > 0 && lane > 0 && !same_bits(S.entryP[tid], S.exitP[tid - 1]);
                if (!__syncthreads_or(bad)) break;
                if (bad && a.counters) atomicAdd(&a.counters[0], 1ull);
                if (round + 1 < a.max_rounds) continue;
                // repair from the neighbours' exits (parallel passes, then in order)
                for (int pass = 0; pass < 4; ++pass) {
                    const bool bad2 = cnt > 0 && lane > 0 && !same_bits(S.entryP[tid], S.exitP[tid - 1]);
                    const double want = bad2 ? S.exitP[tid - 1] : 0.0;
                    if (!__syncthreads_or(bad2)) break;
                    if (bad2) {
                        bool sy;
                        long long li;
                        double lv;
                        const double Pn = lane_chain(cp, xl, cl, cnt, want, true, S.entryP[tid], sy, li, lv);
                        S.repaired[tid] = 1;
                        S.entryP[tid] = want;
                        if (!sy) S.exitP[tid] = Pn;
                    }
                    __syncthreads();
                }
                if (lane == 0 && active > 0) {
                    for (int l = 1; l < active; ++l) {
                        const int id = pl * LPL + l;
                        const double want = S.exitP[id - 1];
                        if (same_bits(want, S.entryP[id])) continue;
                        if (a.counters) atomicAdd(&a.counters[3], 1ull);
                        const int c2 = (int)umin64(SUB, n - (base + (uint64_t)l * SUB));
                        bool sy;
                        long long li;
                        double lv;
                        const double Pn = lane_chain(cp, xs + id * XS_STRIDE, code + id * CODE_STRIDE, c2, want, true,
                                                     S.entryP[id], sy, li, lv);
                        S.entryP[id] = want;
                        S.repaired[id] = 1;
                        if (!sy) S.exitP[id] = Pn;
                    }
                }
                __syncthreads();
                break;
            }
            QCS_PHASE(1);
            if (lane == 0 && active > 0) C.Pnext = S.exitP[pl * LPL + active - 1];
            // IMZ: the lane's row is its share of the stride's sum of squares
            // (fused_sumsq's first pass over it, formed here from registers)
            double tu = 0.0;
            if (IMZ && a.sumsq) {
                const double s0 = S.s[0];  // the running sum entering this iteration
                if (s0 > 0.0 && ilogb(s0) >= -960) {
                    tu = ldexp(1.0, 52 - ilogb(s0));
                    pre_ok = true;
                }
            }
            if (cnt > 0) {  // the reference's reconstructed predictors from the codes
                const double P0 = S.entryP[tid];
                if (cp.pow2 && ev_idx < 0 && !S.repaired[tid]) {
                    // the lane's last chain had no event: every step was a
                    // proven lattice step from its entry (lane_chain), so the
                    // predictor after element i is exactly entry + 2d*M_i with
                    // M_i the integer prefix of the codes — independent
                    // products and sums instead of a serial FP chain
                    int M = 0;
#pragma unroll 8
                    for (int i = 0; i < cnt; ++i) {
                        M += cl[i];
                        const double xv = __dadd_rn(P0, __dmul_rn(cp.td, (double)M));
                        xl[i] = xv;
                        if (IMZ) pre_loc = sat_add(pre_loc, sq_units(xv, tu));
                    }
                } else {
                    double P = P0;
                    for (int i = 0; i < cnt; ++i) {
                        const int16_t co = cl[i];
                        if (co == WCODE16) P = xl[i];
                        else if (co != 0) P = __dadd_rn(P, __dmul_rn(cp.td, (double)co));
                        xl[i] = P;
                        if (IMZ) pre_loc = sat_add(pre_loc, sq_units(P, tu));
                    }
                }
            }
            __syncthreads();
        } else {
            if (cnt > 0)
                for (int i = 0; i < cnt; ++i) cl[i] = __double_as_longlong(xl[i]) == 0 ? (int16_t)0 : WCODE16;
            __syncthreads();
        }

        QCS_PHASE(2);
        // 5. stored sum of squares per stride
        if (a.sumsq) fused_sumsq<LPL, IMZ>(xs, n_it, S, a.counters, pre_ok, pre_loc);

        QCS_PHASE(3);
        // 6. run summary of each lane (bitmasks) and the run entering it
        const LaneMasks lm = cnt > 0 ? lane_masks<false>(cl, cnt) : LaneMasks{0u, 0u, 0u};
        const int t0 = cnt > 0 ? mask_type(lm, 0) : TY_NONE;
        const bool full = cnt > 0 && (lm.z == lm.valid || lm.w == lm.valid);
        S.ftype[pl * (LPL + 1) + lane] = (int8_t)t0;
        if (lane == 0) S.ftype[pl * (LPL + 1) + LPL] = TY_NONE;
        // tail run of the lane (lane-local start)
        int tail_ty = TY_NONE, tail_j = 0;
        if (cnt > 0) {
            const int last = cnt - 1;
            tail_ty = mask_type(lm, last);
            if (tail_ty != TY_C) {
                const uint32_t mm = tail_ty == TY_Z ? lm.z : lm.w;
                const uint32_t below = (~mm) & ((1u << last) - 1u);
                tail_j = below ? (32 - __clz(below)) : 0;
            } else {
                tail_ty = TY_NONE;
            }
        }
        RunFn F{0, 0};
        if (cnt > 0) {
            if (full) F = RunFn{(2 << 2) | t0, e0};
            else if (tail_ty != TY_NONE) F = RunFn{(1 << 2) | tail_ty, e0 + tail_j};
            else F = RunFn{(1 << 2) | TY_NONE, 0};
        }
        const RunFn inc = fscan_fn<WPL>(F, S, pl);
        S.fincl[tid] = inc;
        __syncthreads();
        int in_ty = C.open_ty;
        uint64_t in_st = C.open_start;
        if (lane > 0) fn_apply(S.fincl[tid - 1], in_ty, in_st);
        const int next_ft = (lane + 1 < active) ? S.ftype[pl * (LPL + 1) + lane + 1] : TY_NONE;
        uint64_t tail_st = e0 + tail_j;
        if (tail_ty != TY_NONE && tail_j == 0 && in_ty == tail_ty) tail_st = in_st;
        const bool tail_closes = lane + 1 < active ? (tail_ty != TY_NONE && next_ft != tail_ty) : final_iter;

        // 7. byte count of the tokens this lane closes.  A lane without raw
        // words (no W element, no carried W run closing here) emits only code
        // and zero-run tokens, contiguous at its byte offset: it generates them
        // right here into its own x row (free after the sum; <= 160 bytes) and
        // the warp copies them out coalesced in step 9
        uint32_t nbytes = 0;
        int closes_open = 0;
        uint64_t close_vlen = 0;
        const bool staged = cnt > 0 && lm.w == 0u && !(lane == 0 && in_ty == TY_W);
        int rt_rel = -1, rt_vl = 0, rt_sl = 0;  // staged: token of a run begun in an earlier lane
        if (staged) {
            uint8_t* const bufp = reinterpret_cast<uint8_t*>(xl);
            uint32_t rp = 0;
            lane_tokens(
                lm, cl, cnt, e0, in_ty, in_st, tail_closes, lane == 0,
                [&](int t, uint64_t st, uint64_t end) {
                    const uint64_t v = run_token(LOSSY, t, end - st);
                    const int vl = varint_len(v);
                    put_varint(bufp + rp, v);
                    if (st < e0 && st >= base) {
                        rt_rel = (int)rp;
                        rt_vl = vl;
                        rt_sl = pl * LPL + (int)((st - base) / SUB);
                    }
                    if (st < base) {
                        closes_open = 1;
                        close_vlen = vl;
                    }
                    rp += vl;
                },
                [&](int16_t q) {
                    const int32_t qq = q;
                    const uint32_t v = ((((uint32_t)qq << 1) ^ (uint32_t)(qq >> 31)) << 2) | 1u;
                    const uint32_t len = 1u + (v >= 128u) + (v >= 16384u);
                    uint8_t* o = bufp + rp;
                    o[0] = (uint8_t)((v & 0x7fu) | (len > 1u ? 0x80u : 0u));
                    if (len > 1u) o[1] = (uint8_t)(((v >> 7) & 0x7fu) | (len > 2u ? 0x80u : 0u));
                    if (len > 2u) o[2] = (uint8_t)(v >> 14);
                    rp += len;
                });
            nbytes = rp;
        } else {
            nbytes = lane_cbytes(cl, cnt);
            lane_runs(lm, cnt, e0, in_ty, in_st, tail_closes, lane == 0, [&](int t, uint64_t st, uint64_t end) {
                const uint64_t len = end - st;
                const int vl = varint_len(run_token(LOSSY, t, len));
                nbytes += vl + (t == TY_W ? 8u * (uint32_t)len : 0u);
                if (st < base) {
                    closes_open = 1;
                    close_vlen = vl;
                }
            });
        }
        if (closes_open) {
            C.closes_open = 1;
            C.close_vlen = close_vlen;
        }
        uint64_t tot;
        const uint64_t excl = fscan_sum<WPL>(nbytes, S, pl, tot);
        const uint64_t bstart = C.out_pos + excl;
        S.bstart[tid] = bstart;
        if (lane == 0) {
            C.iter_bytes = tot;
            C.carry_tok = C.out_pos;
            C.mv_bytes = 0;
            C.mv_shift = 0;
            // (same thread: closes_open is visible since fscan_sum's barrier)
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

        QCS_PHASE(4);
        // 8. slide words of a carried W run left if its varint came out shorter
        uint64_t mvmax = 0;
        for (int p = 0; p < NPL; ++p) mvmax = max(mvmax, S.carry[p].mv_bytes);
        if (tid == 0 && a.counters && mvmax) atomicAdd(&a.counters[2], (unsigned long long)mvmax);
        QCS_WD(mvmax > (1ull << 32), "slide");
        for (uint64_t o = 0; o < mvmax; o += LPL * 8) {
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

        // 9. write tokens (see qcs_codec.cuh for the placement rules)
        if (staged && rt_rel >= 0) {
            S.runtok[rt_sl] = bstart + (uint64_t)rt_rel;
            S.runw[rt_sl] = bstart + (uint64_t)(rt_rel + rt_vl);
        }
        {
            // staged lanes: the warp copies each lane's bytes, 32 consecutive
            // bytes per store
            const int wl = tid & 31;
            const uint32_t my_nb = staged ? nbytes : 0u;
            for (unsigned todo = __ballot_sync(0xffffffffu, my_nb != 0u); todo; todo &= todo - 1u) {
                const int j = __ffs(todo) - 1;
                const uint32_t nb = __shfl_sync(0xffffffffu, my_nb, j);
                const uint64_t bs = __shfl_sync(0xffffffffu, bstart, j);
                const uint8_t* src = reinterpret_cast<const uint8_t*>(xs + (uint64_t)((tid & ~31) + j) * XS_STRIDE);
                // <= 160 bytes (32 tokens of <= 5): predicated rounds, loads
                // first; two rounds cover the usual lane (warp-uniform test)
                if (nb <= 64u) {
                    const uint8_t b0 = wl < nb ? src[wl] : (uint8_t)0;
                    const uint8_t b1 = wl + 32u < nb ? src[wl + 32u] : (uint8_t)0;
                    if (wl < nb) out[bs + wl] = b0;
                    if (wl + 32u < nb) out[bs + wl + 32u] = b1;
                } else {
                    uint8_t b[5];
#pragma unroll
                    for (int r = 0; r < 5; ++r) b[r] = wl + 32u * r < nb ? src[wl + 32u * r] : (uint8_t)0;
#pragma unroll
                    for (int r = 0; r < 5; ++r)
                        if (wl + 32u * r < nb) out[bs + wl + 32u * r] = b[r];
                    for (uint32_t k = wl + 160u; k < nb; k += 32) out[bs + k] = src[k];
                }
            }
        }
        if (!staged) {
            uint64_t pos = bstart;
            lane_tokens(
                lm, cl, cnt, e0, in_ty, in_st, tail_closes, lane == 0,
                [&](int t, uint64_t st, uint64_t end) {
                    const uint64_t len = end - st;
                    const uint64_t v = run_token(LOSSY, t, len);
                    const int vl = varint_len(v);
                    put_varint(out + pos, v);
                    if (t == TY_W) {
                        const uint64_t k0 = st > e0 ? st : e0;
                        put_words(out + pos + vl + 8 * (k0 - st), xl + (k0 - e0), (int)(end - k0));
                    }
                    if (st < e0 && st >= base) {
                        const int sl = pl * LPL + (int)((st - base) / SUB);
                        S.runtok[sl] = pos;
                        S.runw[sl] = pos + vl;
                    }
                    pos += vl + (t == TY_W ? 8 * len : 0);
                },
                [&](int16_t q) {
                    // code token: < 2^18, 1..3 varint bytes, stored without a loop
                    const int32_t qq = q;
                    const uint32_t v = ((((uint32_t)qq << 1) ^ (uint32_t)(qq >> 31)) << 2) | 1u;
                    const uint32_t len = 1u + (v >= 128u) + (v >= 16384u);
                    uint8_t* o = out + pos;
                    o[0] = (uint8_t)((v & 0x7fu) | (len > 1u ? 0x80u : 0u));
                    if (len > 1u) o[1] = (uint8_t)(((v >> 7) & 0x7fu) | (len > 2u ? 0x80u : 0u));
                    if (len > 2u) o[2] = (uint8_t)(v >> 14);
                    pos += len;
                });
        }
        if (lane + 1 == active && !final_iter && tail_ty != TY_NONE && tail_st >= base) {
            const uint64_t tokpos = C.out_pos + C.iter_bytes;
            const uint64_t vmax = tail_ty == TY_W ? varint_len(run_token(LOSSY, TY_W, n - tail_st)) : 0;
            const int sl = pl * LPL + (int)((tail_st - base) / SUB);
            S.runtok[sl] = tokpos;
            S.runw[sl] = tokpos + vmax;
        }
        __syncthreads();

        // 10. words of a W run reaching past this lane
        if (cnt > 0 && tail_ty == TY_W && !tail_closes) {
            const uint64_t wb = tail_st < base ? C.carry_w : S.runw[pl * LPL + (tail_st - base) / SUB];
            const uint64_t k0 = tail_st > e0 ? tail_st : e0;
            put_words(out + wb + 8 * (k0 - tail_st), xl + (k0 - e0), (int)(e0 + cnt - k0));
        }

        // 11. side index
        if (cnt > 0) {
            SideEntry se;
            if (in_ty != TY_NONE && t0 == in_ty) {
                se.off = (uint32_t)(in_st < base ? C.carry_tok : S.runtok[pl * LPL + (in_st - base) / SUB]);
                se.skip = (uint32_t)(e0 - in_st);
            } else {
                const bool emitted_here = !full || tail_closes;
                uint64_t cover = bstart;
                if (lane == 0 && in_ty != TY_NONE) {
                    const uint64_t len = e0 - in_st;
                    cover += varint_len(run_token(LOSSY, in_ty, len)) + (in_ty == TY_W ? 8 * len : 0);
                }
                se.off = (uint32_t)(emitted_here ? cover : S.runtok[tid]);
                se.skip = 0;
            }
            se.pred = LOSSY ? S.entryP[tid] : 0.0;
            side[e0 / SUB] = se;
        }

        QCS_PHASE(5);
        // 12. carry to the next iteration
        __syncthreads();
        if (lane == 0 && active > 0) {
            const int last = pl * LPL + active - 1;
            C.P = LOSSY ? C.Pnext : 0.0;
            C.xprev = C.xprev_next;
            const uint64_t new_pos = C.out_pos + C.iter_bytes;
            int oty = C.open_ty;
            uint64_t ost = C.open_start;
            fn_apply(S.fincl[last], oty, ost);
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
        // Ladder early exit (not the last level): the closed tokens are a
        // lower bound of the final payload, so once 16L / (headers + them)
        // falls below theta the level can no longer be chosen
        // (block_pair_ratio, aalc.cpp:37-42; pairs: min of both) -- stop and
        // leave the unit pending for the next level (uniform over the CTA)
        if (a.ladder_theta > 0.0 && !final_iter) {
            uint64_t lb = 2 * HEADER_BYTES;
            for (int p = 0; p < NPL; ++p) lb += S.carry[p].out_pos;
            if ((double)(16 * n) / (double)lb < a.ladder_theta) {
                if (tid == 0) {
                    a.out_len[2 * gslot] = 1ull << 50;  // ratio ~ 0: the ladder moves on
                    a.out_len[2 * gslot + 1] = 1ull << 50;
                    if (a.counters) atomicAdd(&a.counters[15], 1ull);
                }
                return;
            }
        }
    }

    if (MODE == MODE_LOCAL && a.dump_x) return;
    QCS_PHASE(6);
    if (tid == 0 && a.counters)
        for (int i = 0; i < 8; ++i) atomicAdd(&a.counters[8 + i], ph_acc[i]);
    if (tid == 0 && a.cta_trace)
        for (int i = 0; i < 8; ++i) a.cta_trace[8 * (a.slot_base + (uint64_t)b) + i] = ph_acc[i];
    if (lane == 0) a.out_len[2 * gslot + comp] = C.out_pos;
    if (a.sumsq && tid == 0) a.sumsq[gslot] = S.s[0];
    if (IMZ) write_zero_plane<LOSSY>(a, slot, gslot, 1, tid, NPL * LPL);
}

template <bool LOSSY, int NPL, int LPL, int MODE>
__global__ void __launch_bounds__(NPL * LPL, (NPL * LPL > 256 ? 1 : (NPL * LPL > 128 ? 2 : 4))) k_fused(FusedArgs a)
{
    // the launch-local slot of this CTA: block order, or the dense-first
    // permutation of the launch's slots (k_slot_order) so that all-zero
    // strides do not pile the costly ones onto the same SMs
    if (a.err && *a.err) return;
    const int b = a.order ? (int)(a.order[a.slot_base + blockIdx.x] - a.slot_base) : (int)blockIdx.x;
    const uint64_t gslot = a.slot_base + (uint64_t)b;
    if (a.pending && !a.pending[gslot]) return;
    if (a.redo_only && !a.redo_only[gslot]) return;
    // zero-stride pass: an all-zero output stride is its two zero encodings
    // and a stored sum of squares of +0.0 (core.cpp:30-37 over zeros)
    if (NPL == 2 && a.zero_slot && a.zero_slot[gslot]) {
        for (int c = 0; c < 2; ++c) write_zero_plane<LOSSY>(a, (uint64_t)b, gslot, c, threadIdx.x, NPL * LPL);
        if (a.sumsq && threadIdx.x == 0) a.sumsq[gslot] = 0.0;
        return;
    }
    // a stride whose im plane stays zero gets all of the CTA's lanes for its
    // re plane (same thread count and shared-memory layout)
    if (NPL == 2 && a.im_zero && a.im_zero[gslot])
        fused_body<LOSSY, 1, NPL * LPL, MODE, true>(a, b);
    else
        fused_body<LOSSY, NPL, LPL, MODE, false>(a, b);
}

// The reference chain of compress_lossy (codec.cpp:206-250) for bounds whose
// 2*delta is not a power of two: there the predictor `pred + 2d*q` leaves
// any fixed lattice and every step depends on the rounding history, so the
// chain is computed serially, one thread per (slot, plane, level) — all
// ladder levels of a gate at once.  x: the gated, snapped planes
// [slot][plane][n]; out: codes [level][slot][plane][n] (WCODE16 = escape)
// and the predictor entering every SUB-element sub-chunk
// [level][slot][plane][nsub].  The quotient fl(diff/2d) is formed as
// diff * fl(1/2d) when that provably rounds to the same integer (it is at
// least 2^-40 relative away from a half-integer; the two differ by < 2^-51
// relative), else by the exact division — fewer cycles on the serial path.
struct ChainLevels {
    double delta[8];
    double td[8];
    double inv[8];
    double lim[8];
    int n;
};

// rare path of the quotient (kept out of line so the compiler does not
// compute the division speculatively on every step)
__device__ __noinline__ double chain_div(double diff, double td) { return __ddiv_rn(diff, td); }

__global__ void __launch_bounds__(128) k_serial_chain(const double* __restrict__ x, uint64_t rows, uint64_t n,
                                                      uint64_t nsub, ChainLevels lv, int16_t* __restrict__ codes,
                                                      double* __restrict__ preds, const uint8_t* pending,
                                                      uint64_t slot_base, const int* on, const int* err)
{
    if ((on && !*on) || (err && *err)) return;
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= rows * (uint64_t)lv.n) return;
    const int lev = (int)(c / rows);
    const uint64_t row = c % rows;  // slot * 2 + plane
    if (pending && !pending[slot_base + row / 2]) return;
    const double delta = lv.delta[lev], td = lv.td[lev], inv = lv.inv[lev], lim = lv.lim[lev];
    const double* xr = x + row * n;
    int16_t* cr = codes + ((uint64_t)lev * rows + row) * n;
    double* pr = preds + ((uint64_t)lev * rows + row) * nsub;
    double P = 0.0;
    constexpr int G = 8;
    double nx[G];  // the next group's inputs, loaded one group ahead
#pragma unroll
    for (int k = 0; k < G; ++k) nx[k] = (uint64_t)k < n ? xr[k] : 0.0;
    for (uint64_t e0 = 0; e0 < n; e0 += G) {
        double xv[G];
#pragma unroll
        for (int k = 0; k < G; ++k) xv[k] = nx[k];
#pragma unroll
        for (int k = 0; k < G; ++k) nx[k] = e0 + G + k < n ? __ldcs(xr + e0 + G + k) : 0.0;
        if ((e0 & (SUB - 1)) == 0) pr[e0 / SUB] = P;
        uint32_t cw[G / 2];
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const double xx = xv[k];
            const double diff = __dsub_rn(xx, P);
            // fast quotient and llround (half away from zero) with the
            // candidates formed in parallel; `slow` flags a quotient within
            // 2^-40 (relative) of a half-integer: that step is redone with
            // the exact division (off the critical path otherwise)
            const double qd = __dmul_rn(diff, inv);
            const double t0 = trunc(qd);
            const double fr = fabs(__dsub_rn(qd, t0));
            const double tu = __dadd_rn(t0, copysign(1.0, qd));
            const bool slow = fabs(__dsub_rn(fr, 0.5)) <= fabs(qd) * 9.094947017729282e-13;  // 2^-40
            double t = fr >= 0.5 ? tu : t0;
            if (slow) {
                const double qx = chain_div(diff, td);
                t = trunc(qx);
                if (fabs(__dsub_rn(qx, t)) >= 0.5) t = __dadd_rn(t, copysign(1.0, qx));
            }
            const double recon = __dadd_rn(P, __dmul_rn(td, t));
            const bool ok = fabs(diff) < lim && t > -32768.0 && t < 32768.0 && fabs(__dsub_rn(xx, recon)) <= delta;
            P = ok ? recon : xx;
            const uint32_t code = ok ? (uint32_t)(uint16_t)(int16_t)t : 0x8000u;  // 0x8000 = WCODE16
            if (k & 1) cw[k / 2] |= code << 16;
            else cw[k / 2] = code;
        }
        const uint64_t m = umin64(G, n - e0);
        if (m == G && (reinterpret_cast<uintptr_t>(cr + e0) & 15) == 0) {
            *reinterpret_cast<uint4*>(cr + e0) = make_uint4(cw[0], cw[1], cw[2], cw[3]);
        } else {
            for (uint64_t k = 0; k < m; ++k) cr[e0 + k] = (int16_t)(uint16_t)(cw[k / 2] >> (16 * (k & 1)));
        }
    }
}

}  // namespace qcs
