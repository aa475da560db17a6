// B200 compressed-state gate engine: device block store + per-gate pipeline
// + the C-ABI declared in include/qcs_b200.h.
//
// Per gate (CompressedState::apply_gate, aalc.cpp:261-420):
//   k_make_jobs     unit list of make_stride_plan (gate.cpp:313-403), on device
//   [k_stride_partial, k_mean]  reflect_mean's mean pass (aalc.cpp:270-295)
//   per wave of units:
//     [k_decode_gate]  split path: decompress_into + scale + run_plan_unit +
//                      snap_zeros for cross-chunk partners, into scratch X
//     per ladder level: k_fused (decode + gate + snap + compress + stored
//                       sum_sq + side index, or the same from X) and
//                       k_ladder (compress_stride_adaptive / joint pair
//                       ladder, aalc.cpp:117-138, 337-356)
//     [k_wave_commit]  wave layout: install the wave's blocks
//   k_pool_commit   staged commit (small layout: flip each plane to its other slot)
//   k_norm          lazy renormalisation + GateRecord (aalc.cpp:410-419, 612-631)
// All launches are stream-ordered; in the small layout the host only
// synchronises at API boundaries.  A device error word makes every later
// kernel a no-op and keeps the state as it was before the failing gate.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/qcs_b200.h"
#include "qcs_stream.cuh"

using namespace qcs;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_err(QCS_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct Plan {
    uint64_t n_units;
    int pair;        // units are (lo, hi) stride pairs
    int npos;        // fixed stride-index bits (0..2)
    int pos[2];      // ascending bit positions
    int val[2];
    int64_t fixed;   // >= 0: the single unit's stride (phase flip)
    int pb;          // pair bit (pair units)
    int kind;        // gate kind
    int t, c;        // target, control (-1 none)
    int local_ctl;   // in-stride control mask bit (c < s), else -1
    uint64_t flip_off;
    int reflect;
    uint64_t first;  // LOAD: first stride of the range (0 for gates)
};

// Plan.kind of qcs_load_strides_device (not a GateKind): the units are the
// strides [first, first + n_units), their input is the caller's raw planes
constexpr int KIND_LOAD = 4;
// Device error word value of a wave-layout gate whose next wave did not fit in
// the arena: every later kernel is a no-op, the host compacts the arena and
// re-enqueues the gate from that wave (internal, never returned).
constexpr int QCS_SUSPEND = 99;
// susp_unit of a gate suspended inside the persistent streaming kernel: the flag, plus the
// strides installed so far (progress: the same value twice means the state does not fit)
constexpr uint64_t SUSP_PERSIST = 1ull << 62;

__host__ __device__ inline uint64_t insert_bit(uint64_t j, int pos, int v)
{
    const uint64_t lo = j & ((1ull << pos) - 1);
    return ((j >> pos) << (pos + 1)) | ((uint64_t)v << pos) | lo;
}

__host__ __device__ inline uint64_t unit_lo(const Plan& p, uint64_t u)
{
    if (p.fixed >= 0) return (uint64_t)p.fixed;
    uint64_t j = u;
    for (int i = 0; i < p.npos; ++i) j = insert_bit(j, p.pos[i], p.val[i]);
    return j + p.first;
}

__host__ __device__ inline uint64_t round16d(uint64_t x) { return (x + 15) & ~uint64_t(15); }
// capacity of a freshly placed block of r (16-byte-rounded) bytes: 1/256 + 64 bytes of slack, so
// that the stride's next encodings fit it in place (StreamCommit in qcs_stream.cuh uses the same)
__host__ __device__ inline uint64_t slack16(uint64_t r) { return (r + (r >> 8) + 64 + 15) & ~uint64_t(15); }

// job/slot s -> stride
__host__ __device__ inline uint64_t slot_stride(const Plan& p, uint64_t s)
{
    if (!p.pair) return unit_lo(p, s);
    const uint64_t lo = unit_lo(p, s >> 1);
    return (s & 1) ? (lo | (1ull << p.pb)) : lo;
}

struct GateParams {
    double u[8];
};

// ---------------------------------------------------------------------------
// device state arrays
// ---------------------------------------------------------------------------
struct Dev {
    // geometry
    int n, s;
    // small layout: every plane owns two fixed slots (slot_cap bytes, nsub side
    // entries each) in arena[0] / side; the live one is p_off / slot_cap & 1,
    // the encoder writes the other and the commit flips (no copy)
    int pool;
    uint64_t L, NS, nsub;
    // block store
    uint8_t* arena[2];
    uint64_t arena_cap;
    uint64_t* p_off;     // [2NS]
    uint64_t* p_len;     // [2NS]
    int8_t* p_codec;     // [2NS]
    double* p_delta;     // [2NS]
    SideEntry* side;     // [2NS][nsub]
    double* scale;       // [NS]
    double* sum_sq;      // [NS]
    // per-gate scratch
    double* X;           // [NS][2][L]
    uint8_t* slot_out;   // [NS][2][cap]
    uint64_t slot_cap;
    SideEntry* slot_side;  // [NS][2][nsub]
    uint64_t* slot_len;    // [2NS]
    double* slot_sum;      // [NS]
    uint64_t* job_stride;  // [NS]
    uint8_t* pending;      // [NS]
    uint8_t* im_zero;      // [NS] per slot: output im plane provably zero (zero-imaginary-plane mode)
    uint8_t* zero_slot;    // [NS] per slot: output stride provably all zero (zero-stride pass)
    uint8_t* redo;         // [NS] per slot: the streaming kernel left it to the legacy encoder
    uint8_t* committed;    // [NS] per slot: its encoder CTA installed it (wave layout, StreamCommit)
    int inplace;           // blocks are rewritten in place when they fit (QCS_INPLACE=0 turns it off)
    uint64_t* p_cap;       // [2NS] capacity of a block placed by the persistent kernel, valid while
    uint64_t* p_capoff;    // [2NS] ... p_off still is the offset it was placed at (qcs_stream.cuh)
    uint32_t* order;       // [NS] dense-first slot order within each wave (k_slot_order)
    int64_t* slot_of;      // [NS] generation<<32 | slot
    qcs_stride_report* reports;  // [NS]
    uint64_t* new_off;     // [2NS]
    double* partial;       // [2NS] mean pass
    // scalars
    struct Scal {
        uint64_t bump;
        int cur;
        int mode;          // 0 append, 1 compact
        int err;           // first error code (QCS_SUSPEND: wave layout arena full, resumable)
        int err_gate;
        uint64_t susp_unit;  // QCS_SUSPEND: first unit of the wave that did not fit
        uint64_t gen;
        double mean[2];
        double norm_sq;
        uint64_t compressed_bytes;
        double min_ratio;
        uint64_t gate_cin;
        // serial-chain policy (non-power-of-two bounds): on for a few gates
        // once the event rounds needed many serial repairs
        int chain_on;
        int chain_left;
        unsigned long long fb_prev;
        // wave layout, encoder-side commit (qcs_stream.cuh, StreamCommit): the wave's worst case is
        // reserved behind the bump and the CTAs take their bytes from it
        unsigned long long wave_used;
        int wave_direct;
        // persistent streaming kernel (k_stream_persist): slot queue head, strides installed so far
        unsigned long long q_head;
        unsigned long long persist_done;
        int persist_susp;  // the suspension was raised inside the persistent kernel (not by k_precheck)
    }* sc;
    qcs_gate_record* rec;  // record ring for run_program
    uint64_t rec_cap;
    unsigned long long* counters;  // [24] device diagnostics
};

// per-plane codec/delta of the chosen level, kept with the slot
struct LevelTag {
    int8_t* slot_codec;   // [NS]
    double* slot_delta;   // [NS]
};

__global__ void k_make_jobs_reset_cin(Dev d) { d.sc->gate_cin = 0; }

__device__ __forceinline__ int pool_sel(const Dev& d, uint64_t g) { return (int)((d.p_off[g] / d.slot_cap) & 1); }

// side index of plane g's live block
__device__ __forceinline__ SideEntry* side_of(const Dev& d, uint64_t g)
{
    return d.pool ? d.side + (2 * g + pool_sel(d, g)) * d.nsub : d.side + g * d.nsub;
}

__device__ __forceinline__ bool plane_is_zero(const Dev& d, uint64_t g);

// zmode (zero-stride pass): 0 off; 1 a slot's output depends only on its own
// stride (in-stride gates, flips, diagonal gates on pair units); 2 on both
// strides of its pair unit.  A stride whose two planes are the one-token zero
// encoding stays all zero under every gate but reflect_mean (apply_pair of
// zeros gives signed zeros, snap_zeros makes them +0.0), so its encoder CTA
// writes the zero encodings directly.
__device__ __forceinline__ bool stride_is_zero(const Dev& d, uint64_t j)
{
    return plane_is_zero(d, 2 * j) && plane_is_zero(d, 2 * j + 1);
}

__global__ void k_make_jobs(Dev d, Plan p, uint64_t n_slots, uint64_t gen, LevelTag lt, int codec0, double delta0,
                            int imz, int zmode, int resume)
{
    // the commits accumulate it (a gate queued behind a suspended one leaves the suspended gate's sum alone)
    if (blockIdx.x == 0 && threadIdx.x == 0 && !resume && !d.sc->err) d.sc->gate_cin = 0;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = slot_stride(p, s);
        d.job_stride[s] = j;
        d.pending[s] = 1;
        d.slot_of[j] = (int64_t)((gen << 32) | s);
        lt.slot_codec[s] = (int8_t)codec0;  // ladder level 0
        lt.slot_delta[s] = delta0;
        if (imz == 2) {  // the host knows every im plane is zero (all_im_zero)
            d.im_zero[s] = 1;
        } else if (imz) {  // zero-imaginary-plane flags: check the input planes
            bool z;
            if (p.pair)
                z = plane_is_zero(d, 2 * slot_stride(p, s & ~1ull) + 1) && plane_is_zero(d, 2 * slot_stride(p, s | 1ull) + 1);
            else
                z = plane_is_zero(d, 2 * j + 1);
            d.im_zero[s] = z ? 1 : 0;
        }
        bool zs = false;
        if (zmode == 1) zs = stride_is_zero(d, j);
        else if (zmode == 2) zs = stride_is_zero(d, slot_stride(p, s & ~1ull)) && stride_is_zero(d, slot_stride(p, s | 1ull));
        d.zero_slot[s] = zs ? 1 : 0;
    }
}

// Dense-first order of the slots of every wave [w*W, (w+1)*W): the encoder
// CTAs of all-zero strides finish at once, so putting the costly ones first
// spreads them over the SMs instead of pairing them on half of them.  One CTA,
// a stable partition per wave by a block scan of the zero flags.
constexpr int ORDER_THREADS = 1024;
__global__ void __launch_bounds__(ORDER_THREADS) k_slot_order(Dev d, uint64_t n_slots, uint64_t W)
{
    __shared__ uint32_t wsum[ORDER_THREADS / 32];
    __shared__ uint32_t carry[2];
    const int tid = threadIdx.x, wl = tid & 31, w = tid >> 5;
    for (uint64_t w0 = 0; w0 < n_slots; w0 += W) {
        const uint64_t w1 = umin64(n_slots, w0 + W);
        // dense count of the wave first
        uint32_t cnt = 0;
        for (uint64_t s = w0 + tid; s < w1; s += ORDER_THREADS) cnt += d.zero_slot[s] ? 0u : 1u;
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (wl == 0) wsum[w] = cnt;
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
            for (int i = 0; i < ORDER_THREADS / 32; ++i) t += wsum[i];
            carry[0] = 0;          // dense placed so far
            carry[1] = t;          // zero slots start after the dense ones
        }
        __syncthreads();
        for (uint64_t c0 = w0; c0 < w1; c0 += ORDER_THREADS) {
            const uint64_t s = c0 + tid;
            const bool dense = s < w1 && !d.zero_slot[s];
            const bool zero = s < w1 && d.zero_slot[s];
            const unsigned bd = __ballot_sync(0xffffffffu, dense), bz = __ballot_sync(0xffffffffu, zero);
            if (wl == 0) wsum[w] = (uint32_t)__popc(bd) | ((uint32_t)__popc(bz) << 16);
            __syncthreads();
            uint32_t pd = 0, pz = 0, td = 0, tz = 0;
            for (int i = 0; i < ORDER_THREADS / 32; ++i) {
                const uint32_t v = wsum[i];
                if (i < w) pd += v & 0xffffu, pz += v >> 16;
                td += v & 0xffffu, tz += v >> 16;
            }
            const unsigned lt = (1u << wl) - 1u;
            if (dense) d.order[w0 + carry[0] + pd + __popc(bd & lt)] = (uint32_t)s;
            if (zero) d.order[w0 + carry[1] + pz + __popc(bz & lt)] = (uint32_t)s;
            __syncthreads();
            if (tid == 0) carry[0] += td, carry[1] += tz;
            __syncthreads();
        }
    }
}

// Per-gate choice between the event rounds and the serial chain for
// non-power-of-two levels: the rounds win while the lanes'
// entry guesses hold (early, structured states); once a gate needed
// `threshold` or more in-order serial repairs, the next CHAIN_SPAN gates
// precompute every plane's chain for all levels at once, then one gate
// re-measures with the rounds.
constexpr int CHAIN_SPAN = 16;
__global__ void k_chain_policy(Dev d, unsigned long long threshold)
{
    auto* sc = d.sc;
    const unsigned long long fb = d.counters[3];
    const unsigned long long delta = fb - sc->fb_prev;
    sc->fb_prev = fb;
    if (sc->chain_on) {
        if (--sc->chain_left <= 0) sc->chain_on = 0;
    } else if (delta >= threshold) {
        sc->chain_on = 1;
        sc->chain_left = CHAIN_SPAN;
    }
}

// Zero-imaginary-plane mode: slot s gets im_zero = 1 when the
// gate is real and the im plane of every input stride of its unit is the
// one-token encoding of an all-zero plane (so the output im plane is all
// zeros too, after snap_zeros).  Pair units: both slots need both planes.
__device__ __forceinline__ bool plane_is_zero(const Dev& d, uint64_t g)
{
    const int codec = d.p_codec[g];
    const uint64_t tok = codec == 1 ? (d.L << 2) : (d.L << 1);  // run of L zeros
    const uint64_t len = d.p_len[g];
    if (len != (uint64_t)varint_len(tok)) return false;
    const uint8_t* in = d.arena[d.sc->cur] + d.p_off[g];
    uint64_t pos = 0;
    return get_varint(in, pos) == tok;
}

struct DecodeJob {
    uint64_t j0;       // first stride (stride = j0 + blockIdx)
    int apply_scale;
    double* out;       // [blocks][re|im][L]
};

__global__ void __launch_bounds__(256) k_decode(Dev d, DecodeJob dj)
{
    if (d.sc->err) return;
    const uint64_t j = dj.j0 + blockIdx.x;
    const int pl = threadIdx.x >> 7;
    const int lane = threadIdx.x & 127;
    const uint64_t g = 2 * j + pl;
    const uint8_t* in = d.arena[d.sc->cur] + d.p_off[g];
    const int codec = d.p_codec[g];
    const double td = 2.0 * d.p_delta[g];
    const double scale = dj.apply_scale ? d.scale[j] : 1.0;
    double* o = dj.out + (uint64_t)blockIdx.x * 2 * d.L + (uint64_t)pl * d.L;
    const SideEntry* side = side_of(d, g);
    for (uint64_t sc = lane; sc < d.nsub; sc += PLANE_LANES) {
        const uint64_t e0 = sc * SUB;
        const int cnt = (int)umin64(SUB, d.L - e0);
        decode_sub(in, codec, td, side[sc], cnt, o + e0, scale);
    }
}

// Decode + gate + snap for the encoder's RAW input (split path).  Fully
// parallel over (unit, chunk): each CTA decodes 256 sub-chunks (one per
// thread, via the side index), applies run_plan_unit's apply_pair
// (gate.cpp:405-454) and snap_zeros (core.cpp:39-47), and writes the planes
// uncompressed into the slot-ordered scratch X[slot][re|im][L].
//   DG_IN    partner inside the 4096-element chunk (t < 12), 2 planes x 4096
//   DG_FAR   partner 2^t >= 2048 away in the same stride, 2 x 2 planes x 2048
//   DG_PAIR  lo / hi stride of a cross-stride unit, 2 x 2 planes x 2048
enum { DG_IN = 0, DG_FAR = 1, DG_PAIR = 2 };
// R sub-chunk rows per CTA (R threads): DG_IN covers 2 planes x R/2 rows
// (IN_CH = 16 R elements, partners inside it), DG_FAR / DG_PAIR 4 planes x R/4
// rows (HALF = 8 R elements per side).
constexpr int DG_R = 128;
constexpr int DG_IN_CH = 16 * DG_R;
constexpr int DG_HALF = 8 * DG_R;
constexpr size_t DG_SMEM = sizeof(double) * DG_R * XS_STRIDE;

__global__ void __launch_bounds__(DG_R) k_decode_gate(Dev d, Plan p, GateParams gp, int mode,
                                                    uint64_t chunks, uint64_t slot_base, const uint8_t* imz,
                                                    const uint8_t* zs)
{
    if (d.sc->err) return;
    extern __shared__ __align__(16) unsigned char dg_smem[];
    double* xs = reinterpret_cast<double*>(dg_smem);
    const uint64_t u = blockIdx.x / chunks, c = blockIdx.x % chunks;
    // zero-stride pass: the encoder writes these slots without reading X
    if (zs && zs[slot_base + (mode == DG_PAIR ? 2 * u : u)]) return;
    const int tid = threadIdx.x;
    const uint64_t L = d.L;
    const uint64_t hb = 1ull << (p.pair ? 0 : p.t);
    constexpr int RQ = DG_R / 4, RH = DG_R / 2;
    // this thread's row: (stride, component, element base)
    uint64_t slot, e0;
    int comp;
    auto far_lo = [&](uint64_t e) { return ((e >> p.t) << (p.t + 1)) | (e & (hb - 1)); };
    if (mode == DG_IN) {
        slot = u;
        comp = tid / RH;
        e0 = c * DG_IN_CH + (uint64_t)(tid % RH) * SUB;
    } else {
        const int q = tid / RQ;            // 0 A.re, 1 A.im, 2 B.re, 3 B.im
        const uint64_t sub = (uint64_t)(tid % RQ) * SUB;
        comp = q & 1;
        if (mode == DG_PAIR) {
            slot = 2 * u + (q >> 1);
            e0 = c * DG_HALF + sub;
        } else {
            slot = u;
            e0 = far_lo(c * DG_HALF) + ((q >> 1) ? hb : 0) + sub;
        }
    }
    const uint64_t j = d.job_stride[slot_base + slot];
    const uint64_t g = 2 * j + comp;
    const int cnt = (int)umin64(SUB, L - umin64(e0, L));
    // zero-imaginary-plane mode: a zero im plane needs no decode (and its
    // gated values, zeros, are not written: the encoder reads only re)
    const bool zim = imz && imz[slot_base + slot];
    if (cnt > 0) {
        if (zim && comp == 1) {
            for (int i = 0; i < cnt; ++i) xs[tid * XS_STRIDE + i] = 0.0;
        } else {
            decode_sub(d.arena[d.sc->cur] + d.p_off[g], d.p_codec[g], 2.0 * d.p_delta[g],
                       side_of(d, g)[e0 / SUB], cnt, xs + tid * XS_STRIDE, d.scale[j]);
        }
    }
    __syncthreads();
    double m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = gp.u[i];
    auto at = [&](int row_base, int k) -> double& { return xs[(row_base + (k >> 5)) * XS_STRIDE + (k & 31)]; };
    if (mode == DG_IN) {
        const uint64_t lo_mask = hb - 1;
        for (int q = tid; q < DG_IN_CH / 2; q += DG_R) {
            const int i0 = (int)((((uint64_t)q & ~lo_mask) << 1) | ((uint64_t)q & lo_mask));
            const int i1 = i0 | (int)hb;
            if (p.local_ctl >= 0 && !(((c * DG_IN_CH + i0) >> p.local_ctl) & 1)) continue;
            pair_update(m, at(0, i0), at(RH, i0), at(0, i1), at(RH, i1));
        }
    } else {
        for (int i = tid; i < DG_HALF; i += DG_R) {
            const uint64_t gi = (mode == DG_PAIR ? c * DG_HALF : far_lo(c * DG_HALF)) + i;
            if (p.local_ctl >= 0 && !((gi >> p.local_ctl) & 1)) continue;
            pair_update(m, at(0, i), at(RQ, i), at(2 * RQ, i), at(3 * RQ, i));
        }
    }
    __syncthreads();
    // snap and write out: every (plane, side) segment is contiguous in X, so
    // each is one coalesced copy (pairs of doubles per thread)
    const int nseg = mode == DG_IN ? 2 : 4;
    const int seg = mode == DG_IN ? DG_IN_CH : DG_HALF;
    for (int q = 0; q < nseg; ++q) {
        uint64_t oslot, e_base;
        int ocomp;
        if (mode == DG_IN) {
            oslot = u;
            ocomp = q;
            e_base = c * DG_IN_CH;
        } else {
            ocomp = q & 1;
            if (mode == DG_PAIR) {
                oslot = 2 * u + (q >> 1);
                e_base = c * DG_HALF;
            } else {
                oslot = u;
                e_base = far_lo(c * DG_HALF) + ((q >> 1) ? hb : 0);
            }
        }
        if (ocomp == 1 && imz && imz[slot_base + oslot]) continue;
        double* dst = d.X + (2 * oslot + ocomp) * L + e_base;
        const double* rows = xs + (uint64_t)q * (seg / SUB) * XS_STRIDE;
        const int m = (int)umin64((uint64_t)seg, L - umin64(e_base, L));
        if (m == seg) {
            for (int k = 2 * tid; k < seg; k += 2 * DG_R) {
                const double v0 = snap(rows[(k >> 5) * XS_STRIDE + (k & 31)]);
                const double v1 = snap(rows[((k + 1) >> 5) * XS_STRIDE + ((k + 1) & 31)]);
                *reinterpret_cast<double2*>(dst + k) = make_double2(v0, v1);
            }
        } else {
            for (int k = tid; k < m; k += DG_R) dst[k] = snap(rows[(k >> 5) * XS_STRIDE + (k & 31)]);
        }
    }
}

// k_decode_gate for a state whose every im plane is zero (a real state: the
// host tracks it, all_im_zero) and a real gate, cross-chunk partners
// (DG_FAR / DG_PAIR): all DG_R threads decode re rows — DG_R/2 per side, so
// a CTA covers DG_RE_CH = 16 * DG_R elements per side — the gate runs on
// (re, 0) pairs with the reference's arithmetic, and only re is written (the
// encoder's zero-imaginary-plane mode writes the im plane itself).
constexpr int DG_RE_CH = 16 * DG_R;

__global__ void __launch_bounds__(DG_R) k_decode_gate_re(Dev d, Plan p, GateParams gp, int mode, uint64_t chunks,
                                                       uint64_t slot_base, const uint8_t* zs)
{
    if (d.sc->err) return;
    extern __shared__ __align__(16) unsigned char dg_smem[];
    double* xs = reinterpret_cast<double*>(dg_smem);
    const uint64_t u = blockIdx.x / chunks, c = blockIdx.x % chunks;
    if (zs && zs[slot_base + (mode == DG_PAIR ? 2 * u : u)]) return;  // zero-stride pass
    const int tid = threadIdx.x;
    const uint64_t L = d.L;
    const uint64_t hb = 1ull << (p.pair ? 0 : p.t);
    constexpr int RH = DG_R / 2;
    auto far_lo = [&](uint64_t e) { return ((e >> p.t) << (p.t + 1)) | (e & (hb - 1)); };
    const int side = tid / RH;  // 0 lo / A, 1 hi / B
    const uint64_t sub = (uint64_t)(tid % RH) * SUB;
    uint64_t slot, e0;
    if (mode == DG_PAIR) {
        slot = 2 * u + side;
        e0 = c * DG_RE_CH + sub;
    } else {
        slot = u;
        e0 = far_lo(c * DG_RE_CH) + (side ? hb : 0) + sub;
    }
    const uint64_t j = d.job_stride[slot_base + slot];
    const uint64_t g = 2 * j;  // re plane
    const int cnt = (int)umin64(SUB, L - umin64(e0, L));
    if (cnt > 0)
        decode_sub(d.arena[d.sc->cur] + d.p_off[g], d.p_codec[g], 2.0 * d.p_delta[g], side_of(d, g)[e0 / SUB], cnt,
                   xs + tid * XS_STRIDE, d.scale[j]);
    __syncthreads();
    double m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = gp.u[i];
    auto at = [&](int row_base, int k) -> double& { return xs[(row_base + (k >> 5)) * XS_STRIDE + (k & 31)]; };
    for (int i = tid; i < DG_RE_CH; i += DG_R) {
        const uint64_t gi = (mode == DG_PAIR ? c * DG_RE_CH : far_lo(c * DG_RE_CH)) + i;
        if (p.local_ctl >= 0 && !((gi >> p.local_ctl) & 1)) continue;
        double z0 = 0.0, z1 = 0.0;  // the im inputs, exactly zero
        pair_update(m, at(0, i), z0, at(RH, i), z1);
    }
    __syncthreads();
    for (int q = 0; q < 2; ++q) {
        uint64_t oslot, e_base;
        if (mode == DG_PAIR) {
            oslot = 2 * u + q;
            e_base = c * DG_RE_CH;
        } else {
            oslot = u;
            e_base = far_lo(c * DG_RE_CH) + (q ? hb : 0);
        }
        double* dst = d.X + (2 * oslot) * L + e_base;
        const double* rows = xs + (uint64_t)q * RH * XS_STRIDE;
        const int mm = (int)umin64((uint64_t)DG_RE_CH, L - umin64(e_base, L));
        if (mm == DG_RE_CH) {
            for (int k = 2 * tid; k < DG_RE_CH; k += 2 * DG_R) {
                const double v0 = snap(rows[(k >> 5) * XS_STRIDE + (k & 31)]);
                const double v1 = snap(rows[((k + 1) >> 5) * XS_STRIDE + ((k + 1) & 31)]);
                *reinterpret_cast<double2*>(dst + k) = make_double2(v0, v1);
            }
        } else {
            for (int k = tid; k < mm; k += DG_R) dst[k] = snap(rows[(k >> 5) * XS_STRIDE + (k & 31)]);
        }
    }
}

// stride_amplitude_sum (gate.cpp:303-311) of every scaled stride, straight
// from the block store: one CTA per stride decodes 4096-element chunks of both
// planes into shared memory; one thread per plane folds them serially in
// index order (the reference's FP order).
__global__ void __launch_bounds__(128) k_stride_partial(Dev d)
{
    if (d.sc->err) return;
    __shared__ double xs[128 * XS_STRIDE];
    const uint64_t j = blockIdx.x;
    const int tid = threadIdx.x, pl = tid >> 6, lane = tid & 63;
    const uint64_t g = 2 * j + pl;
    const uint8_t* in = d.arena[d.sc->cur] + d.p_off[g];
    const int codec = d.p_codec[g];
    const double td = 2.0 * d.p_delta[g];
    const double scale = d.scale[j];
    const SideEntry* side = side_of(d, g);
    double acc = 0.0;
    for (uint64_t base = 0; base < d.L; base += 2048) {
        const uint64_t e0 = base + (uint64_t)lane * SUB;
        __syncthreads();
        if (e0 < d.L) decode_sub(in, codec, td, side[e0 / SUB], (int)umin64(SUB, d.L - e0), xs + tid * XS_STRIDE, scale);
        __syncthreads();
        if (lane == 0) {
            const int m = (int)umin64(2048, d.L - base);
            for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, xs[(pl * 64 + (k >> 5)) * XS_STRIDE + (k & 31)]);
        }
    }
    if (lane == 0) d.partial[2 * j + pl] = acc;
}

__global__ void k_mean(Dev d)
{
    if (d.sc->err) return;
    double sr = 0.0, si = 0.0;
    for (uint64_t j = 0; j < d.NS; ++j) {
        sr = __dadd_rn(sr, d.partial[2 * j]);
        si = __dadd_rn(si, d.partial[2 * j + 1]);
    }
    const double na = (double)(1ull << d.n);
    d.sc->mean[0] = __ddiv_rn(sr, na);
    d.sc->mean[1] = __ddiv_rn(si, na);
}

// Ladder step for every unit: block_pair_ratio (aalc.cpp:37-42); stop at the
// first level whose ratio (pairs: min of both) reaches theta, else keep the
// last level (aalc.cpp:125-137, 346-356).
__global__ void k_ladder(Dev d, Plan p, uint64_t u0, uint64_t u1, double delta, double theta, int last_level)
{
    if (d.sc->err) return;
    const uint64_t u = u0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (u >= u1) return;
    const uint64_t s0 = p.pair ? 2 * u : u;
    if (!d.pending[s0]) return;
    const uint64_t bytes_in = d.L * 16;
    const int ns = p.pair ? 2 : 1;
    double r[2];
    uint64_t bo[2];
    for (int k = 0; k < ns; ++k) {
        const uint64_t s = s0 + k;
        bo[k] = (HEADER_BYTES + d.slot_len[2 * s]) + (HEADER_BYTES + d.slot_len[2 * s + 1]);
        r[k] = (double)bytes_in / (double)bo[k];
    }
    const double rmin = ns == 2 ? fmin(r[0], r[1]) : r[0];
    const bool done = rmin >= theta || last_level;
    if (!done) return;
    for (int k = 0; k < ns; ++k) {
        const uint64_t s = s0 + k;
        qcs_stride_report& rep = d.reports[s];
        rep.stride_index = d.job_stride[s];
        rep.bytes_in = bytes_in;
        rep.bytes_out = bo[k];
        rep.chosen_delta = delta;
        rep.ratio = r[k];
        rep.threshold_met = r[k] >= theta;
        rep.pad_ = 0;
        d.pending[s] = 0;
    }
}


__global__ void k_tag_level(Dev d, LevelTag lt, uint64_t s0, uint64_t s1, int codec, double delta)
{
    const uint64_t s = s0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s >= s1 || !d.pending[s]) return;
    lt.slot_codec[s] = (int8_t)codec;
    lt.slot_delta[s] = delta;
}

// Small layout commit (the staged commit of aalc.cpp:395-408): the encoder
// wrote every rewritten plane into its other slot; flip them and install the
// tables.  One thread per (slot, plane).
__global__ void k_pool_commit(Dev d, LevelTag lt, uint64_t n_slots)
{
    if (d.sc->err) return;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= 2 * n_slots) return;
    const uint64_t slot = i >> 1;
    const int c = (int)(i & 1);
    const uint64_t j = d.job_stride[slot];
    const uint64_t g = 2 * j + c;
    const int sel = pool_sel(d, g);
    atomicAdd((unsigned long long*)&d.sc->gate_cin, (unsigned long long)(HEADER_BYTES + d.p_len[g]));
    d.p_off[g] = (2 * g + 1 - sel) * d.slot_cap;
    d.p_len[g] = d.slot_len[i];
    d.p_codec[g] = lt.slot_codec[slot];
    d.p_delta[g] = lt.slot_delta[slot];
    if (c == 0) {
        d.sum_sq[j] = d.slot_sum[slot];
        d.scale[j] = 1.0;
    }
}

// The last ladder level (as k_ladder with last_level) fused with the small
// layout's commit (as k_pool_commit) for every slot of the unit.
__global__ void k_ladder_commit(Dev d, LevelTag lt, Plan p, double delta, double theta)
{
    if (d.sc->err) return;
    const uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (u >= p.n_units) return;
    const uint64_t s0 = p.pair ? 2 * u : u;
    const int ns = p.pair ? 2 : 1;
    const uint64_t bytes_in = d.L * 16;
    if (d.pending[s0]) {
        double r[2];
        uint64_t bo[2];
        for (int k = 0; k < ns; ++k) {
            const uint64_t s = s0 + k;
            bo[k] = (HEADER_BYTES + d.slot_len[2 * s]) + (HEADER_BYTES + d.slot_len[2 * s + 1]);
            r[k] = (double)bytes_in / (double)bo[k];
        }
        for (int k = 0; k < ns; ++k) {
            const uint64_t s = s0 + k;
            qcs_stride_report& rep = d.reports[s];
            rep.stride_index = d.job_stride[s];
            rep.bytes_in = bytes_in;
            rep.bytes_out = bo[k];
            rep.chosen_delta = delta;
            rep.ratio = r[k];
            rep.threshold_met = r[k] >= theta;
            rep.pad_ = 0;
            d.pending[s] = 0;
        }
    }
    unsigned long long cin = 0;
    for (int k = 0; k < ns; ++k) {
        const uint64_t s = s0 + k;
        const uint64_t j = d.job_stride[s];
        for (int c = 0; c < 2; ++c) {
            const uint64_t g = 2 * j + c;
            const int sel = pool_sel(d, g);
            cin += HEADER_BYTES + d.p_len[g];
            d.p_off[g] = (2 * g + 1 - sel) * d.slot_cap;
            d.p_len[g] = d.slot_len[2 * s + c];
            d.p_codec[g] = lt.slot_codec[s];
            d.p_delta[g] = lt.slot_delta[s];
        }
        d.sum_sq[j] = d.slot_sum[s];
        d.scale[j] = 1.0;
    }
    atomicAdd((unsigned long long*)&d.sc->gate_cin, cin);
}

// Small layout basis state (aalc.cpp:140-174): every plane's slot 0 holds the
// lossless all-zero block, the hot stride's re plane the hot block.
__global__ void k_init_pool(Dev d, uint64_t hot_g, uint4 zero, uint32_t zero_len, uint4 hot0, uint4 hot1,
                            uint32_t hot_len)
{
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= 2 * d.NS) return;
    uint4* dst = reinterpret_cast<uint4*>(d.arena[0] + 2 * g * d.slot_cap);
    if (g == hot_g) {
        dst[0] = hot0;
        dst[1] = hot1;
        d.p_len[g] = hot_len;
    } else {
        dst[0] = zero;
        d.p_len[g] = zero_len;
    }
    d.p_off[g] = 2 * g * d.slot_cap;
}

// Lazy renormalisation (aalc.cpp:410-419) and the GateRecord fold
// (aalc.cpp:612-631), serial in stride / report order like the reference.
// The tables are staged through shared memory by all threads; thread 0 folds
// serially (the FP order is the reference's), so the chain never waits on HBM.
constexpr int NORM_THREADS = 256;
constexpr int NORM_CHUNK = 2048;

__device__ double norm_fold(const Dev& d, double f, bool scale_by_f, double* sh_a, double* sh_b)
{
    double total = 0.0;
    for (uint64_t c0 = 0; c0 < d.NS; c0 += NORM_CHUNK) {
        const int m = (int)umin64(NORM_CHUNK, d.NS - c0);
        __syncthreads();
        // the terms in parallel (the same products as before), then the
        // reference's serial left-to-right sum on one thread
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double sc = d.scale[c0 + i];
            const double a = scale_by_f ? __dmul_rn(sc, f) : sc;
            sh_a[i] = __dmul_rn(__dmul_rn(a, a), d.sum_sq[c0 + i]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll 8
            for (int i = 0; i < m; ++i) total = __dadd_rn(total, sh_a[i]);
        }
    }
    return total;
}

__global__ void __launch_bounds__(NORM_THREADS) k_norm(Dev d, uint64_t n_slots, uint64_t rec_index,
                                                      uint64_t gate_index, int renorm)
{
    __shared__ double sh_a[NORM_CHUNK], sh_b[NORM_CHUNK];
    __shared__ double sh_f;
    __shared__ int sh_do;
    if (d.sc->err) {
        if (threadIdx.x == 0 && d.sc->err_gate < 0) d.sc->err_gate = (int)gate_index;
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0 && d.sc->mode == 1) d.sc->cur = 1 - d.sc->cur;
    const double total = renorm ? norm_fold(d, 1.0, false, sh_a, sh_b) : 0.0;
    if (threadIdx.x == 0) {
        sh_do = renorm && total > 0.0;
        sh_f = sh_do ? __ddiv_rn(1.0, __dsqrt_rn(total)) : 1.0;
    }
    __syncthreads();
    const bool do_scale = sh_do;
    const double f = sh_f;
    // norm_sq_tracked after scaling: same products as the reference's
    // scale *= f followed by the serial re-measure
    const double nsq = norm_fold(d, f, do_scale, sh_a, sh_b);
    __syncthreads();
    if (do_scale)
        for (uint64_t j = threadIdx.x; j < d.NS; j += blockDim.x) d.scale[j] = __dmul_rn(d.scale[j], f);
    if (threadIdx.x == 0) d.sc->norm_sq = nsq;
    if (!d.rec) return;
    // GateRecord fold in report order: min / max / sums are order-free, the
    // ratio sum is serial
    double* rr = sh_a;
    qcs_gate_record r;
    r.min_ratio = INFINITY;
    r.max_chosen_delta = 0.0;
    double rs = 0.0;
    uint64_t b_in = 0, b_out = 0, viol = 0;
    for (uint64_t c0 = 0; c0 < n_slots; c0 += NORM_CHUNK) {
        const int m = (int)umin64(NORM_CHUNK, n_slots - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const qcs_stride_report& rep = d.reports[c0 + i];
            rr[i] = rep.ratio;
            r.min_ratio = fmin(r.min_ratio, rep.ratio);
            r.max_chosen_delta = fmax(r.max_chosen_delta, rep.chosen_delta);
            b_in += rep.bytes_in;
            b_out += rep.bytes_out;
            viol += rep.threshold_met ? 0 : 1;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int i = 0; i < m; ++i) rs = __dadd_rn(rs, rr[i]);
    }
    // block reductions of the order-free parts
    __shared__ double red_min[NORM_THREADS / 32], red_max[NORM_THREADS / 32];
    __shared__ uint64_t red_in[NORM_THREADS / 32], red_out[NORM_THREADS / 32], red_v[NORM_THREADS / 32];
    for (int o = 16; o; o >>= 1) {
        r.min_ratio = fmin(r.min_ratio, __shfl_xor_sync(0xffffffffu, r.min_ratio, o));
        r.max_chosen_delta = fmax(r.max_chosen_delta, __shfl_xor_sync(0xffffffffu, r.max_chosen_delta, o));
        b_in += __shfl_xor_sync(0xffffffffu, b_in, o);
        b_out += __shfl_xor_sync(0xffffffffu, b_out, o);
        viol += __shfl_xor_sync(0xffffffffu, viol, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red_min[w] = r.min_ratio;
        red_max[w] = r.max_chosen_delta;
        red_in[w] = b_in;
        red_out[w] = b_out;
        red_v[w] = viol;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    r.min_ratio = INFINITY;
    r.max_chosen_delta = 0.0;
    r.bytes_before = r.bytes_after = r.threshold_violations = 0;
    for (int i = 0; i < NORM_THREADS / 32; ++i) {
        r.min_ratio = fmin(r.min_ratio, red_min[i]);
        r.max_chosen_delta = fmax(r.max_chosen_delta, red_max[i]);
        r.bytes_before += red_in[i];
        r.bytes_after += red_out[i];
        r.threshold_violations += red_v[i];
    }
    r.gate_index = gate_index;
    r.stride_count = n_slots;
    r.mean_ratio = n_slots ? __ddiv_rn(rs, (double)n_slots) : 0.0;
    r.elapsed_ns = 0;
    r.norm_after = __dsqrt_rn(nsq);
    r.compressed_in = d.sc->gate_cin;
    d.rec[rec_index] = r;
}

__global__ void k_index_planes(Dev d, uint64_t g0, uint64_t count)
{
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint64_t g = g0 + i;
    const int rc = index_plane(d.arena[d.sc->cur] + d.p_off[g], d.p_len[g], d.p_codec[g],
                               d.p_delta[g], d.L, side_of(d, g), nullptr);
    if (rc) atomicCAS(&d.sc->err, 0, rc);
}

__global__ void k_stats(Dev d)
{
    if (threadIdx.x != 0) return;
    uint64_t tot = 0;
    double m = INFINITY, nsq = 0.0;
    const uint64_t bytes_in = d.L * 16;
    for (uint64_t j = 0; j < d.NS; ++j) {
        const uint64_t b = (HEADER_BYTES + d.p_len[2 * j]) + (HEADER_BYTES + d.p_len[2 * j + 1]);
        tot += b;
        m = fmin(m, (double)bytes_in / (double)b);
        nsq = __dadd_rn(nsq, __dmul_rn(__dmul_rn(d.scale[j], d.scale[j]), d.sum_sq[j]));
    }
    d.sc->compressed_bytes = tot;
    d.sc->min_ratio = m;
    d.sc->norm_sq = nsq;
}

// codec API: standalone validation + decode of one payload
__global__ void k_decode_payload(const uint8_t* in, uint64_t len, int codec, double delta,
                                 uint64_t n, double* out, int* err)
{
    *err = index_plane(in, len, codec, delta, n, nullptr, out);
}

uint64_t payload_cap(uint64_t n) { return ((9 * n + 64) + 15) & ~uint64_t(15); }

bool is_pow2(double x)
{
    int e;
    const double m = std::frexp(x, &e);
    return x > 0 && std::isfinite(x) && m == 0.5;
}

CodecParams make_params(double delta)
{
    CodecParams cp{};
    cp.delta = delta;
    cp.lossy = delta != 0.0;
    cp.td = 2.0 * delta;
    cp.lim = cp.td * 32768.0;
    cp.pow2 = cp.lossy && is_pow2(cp.td) && std::isfinite(1.0 / cp.td);
    cp.inv_td = cp.pow2 ? 1.0 / cp.td : 0.0;
    return cp;
}

// cudaFuncSetAttribute is per device context: remember each (kernel,
// device) pair once, thread-safely (states on several devices, rank threads).
int set_smem_attr(const void* fn, int bytes)
{
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    int dev = 0;
    CU(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : done)
        if (e.first == fn && e.second == dev) return 0;
    CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.emplace_back(fn, dev);
    return 0;
}

template <bool L, int NPL, int LPL, int MODE>
int launch_fused_t(const FusedArgs& a, uint64_t grid, cudaStream_t s)
{
    if (const int rc = set_smem_attr(reinterpret_cast<const void*>(k_fused<L, NPL, LPL, MODE>),
                                     (int)FusedLayout<NPL * LPL>::SMEM))
        return rc;
    if (grid == 0) return 0;
    k_fused<L, NPL, LPL, MODE><<<(unsigned)grid, NPL * LPL, FusedLayout<NPL * LPL>::SMEM, s>>>(a);
    CU(cudaGetLastError());
    return 0;
}

template <int LANES, bool RAW>
int launch_stream_t(const FusedArgs& a, uint8_t* redo, const StreamCommit& dc, uint64_t grid, cudaStream_t s)
{
    if (const int rc = set_smem_attr(reinterpret_cast<const void*>(k_stream<LANES, RAW>), (int)sizeof(StreamSharedT<LANES>)))
        return rc;
    if (grid == 0) return 0;
    k_stream<LANES, RAW><<<(unsigned)grid, LANES, sizeof(StreamSharedT<LANES>), s>>>(a, redo, dc);
    CU(cudaGetLastError());
    return 0;
}

// streaming kernel (qcs_stream.cuh): CTA width by the slots per SM of the launch
template <bool RAW>
int launch_stream(const FusedArgs& a, uint8_t* redo, const StreamCommit& dc, uint64_t grid, cudaStream_t s)
{
    static const int force_t = getenv("QCS_STREAM_LANES") ? atoi(getenv("QCS_STREAM_LANES")) : 0;  // experiments
    if (force_t == 128) return launch_stream_t<128, RAW>(a, redo, dc, grid, s);
    if (force_t == 256) return launch_stream_t<256, RAW>(a, redo, dc, grid, s);
    if (force_t == 512) return launch_stream_t<512, RAW>(a, redo, dc, grid, s);
    if (grid >= 8 * 148) return launch_stream_t<128, RAW>(a, redo, dc, grid, s);
    if (grid >= 4 * 148) return launch_stream_t<256, RAW>(a, redo, dc, grid, s);
    return launch_stream_t<512, RAW>(a, redo, dc, grid, s);
}

template <int LANES>
int launch_stream_persist_t(const FusedArgs& a, uint8_t* redo, const StreamCommit& dc, uint64_t n_slots,
                            unsigned long long* q_head, uint64_t grid, cudaStream_t s)
{
    if (const int rc = set_smem_attr(reinterpret_cast<const void*>(k_stream_persist<LANES>), (int)sizeof(StreamSharedT<LANES>)))
        return rc;
    if (grid == 0) return 0;
    k_stream_persist<LANES><<<(unsigned)grid, LANES, sizeof(StreamSharedT<LANES>), s>>>(a, redo, dc, n_slots, q_head);
    CU(cudaGetLastError());
    return 0;
}

// persistent streaming kernel: one CTA per staging slot, width by the CTAs per SM
int launch_stream_persist(const FusedArgs& a, uint8_t* redo, const StreamCommit& dc, uint64_t n_slots,
                          unsigned long long* q_head, uint64_t grid, cudaStream_t s)
{
    static const int force_t = getenv("QCS_STREAM_LANES") ? atoi(getenv("QCS_STREAM_LANES")) : 0;  // experiments
    const int lanes = force_t ? force_t : (grid >= 4 * 148 ? 128 : (grid >= 2 * 148 ? 256 : 512));
    if (lanes == 128) return launch_stream_persist_t<128>(a, redo, dc, n_slots, q_head, grid, s);
    if (lanes == 256) return launch_stream_persist_t<256>(a, redo, dc, n_slots, q_head, grid, s);
    return launch_stream_persist_t<512>(a, redo, dc, n_slots, q_head, grid, s);
}

// FM_*_W: 2 planes x 256 lanes (one CTA per SM), for gates with fewer units
// than SMs, where per-stride parallelism is all there is
enum { FM_LOCAL = 0, FM_LOCAL_W = 1, FM_RAW2_W = 2, FM_RAW1 = 3, FM_RAW2 = 4 };

int codec_max_rounds()
{
    const char* e = getenv("QCS_MAX_ROUNDS");
    return e ? std::max(1, atoi(e)) : 6;
}

// elements per plane per iteration of the usual encoder CTA: in-stride
// partners closer than this are gated inside it (MODE_LOCAL)
constexpr uint64_t FUSED_SPAN = 4096;

int launch_fused(const FusedArgs& a, int fm, uint64_t grid, cudaStream_t s)
{
    const bool L = a.cp.lossy != 0;
    switch (fm) {
        case FM_LOCAL: return L ? launch_fused_t<true, 2, 128, MODE_LOCAL>(a, grid, s) : launch_fused_t<false, 2, 128, MODE_LOCAL>(a, grid, s);
        case FM_LOCAL_W: return L ? launch_fused_t<true, 2, 256, MODE_LOCAL>(a, grid, s) : launch_fused_t<false, 2, 256, MODE_LOCAL>(a, grid, s);
        case FM_RAW2_W: return L ? launch_fused_t<true, 2, 256, MODE_RAW>(a, grid, s) : launch_fused_t<false, 2, 256, MODE_RAW>(a, grid, s);
        case FM_RAW1: return L ? launch_fused_t<true, 1, 256, MODE_RAW>(a, grid, s) : launch_fused_t<false, 1, 256, MODE_RAW>(a, grid, s);
        default: return L ? launch_fused_t<true, 2, 128, MODE_RAW>(a, grid, s) : launch_fused_t<false, 2, 128, MODE_RAW>(a, grid, s);
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// host state
// ---------------------------------------------------------------------------
struct qcs_dev_state {
    Dev d{};
    int device = 0;
    cudaStream_t stream = nullptr;
    LevelTag lt{};
    uint64_t gen = 0;
    uint64_t launches = 0;
    int split_local = 0;  // QCS_SPLIT_LOCAL=1: in-chunk gates also take the split path
    int max_rounds = 6;  // QCS_MAX_ROUNDS (tests force the neighbour-exit repair)
    // serial-chain mode for non-power-of-two bounds (QCS_SERIAL_CHAIN=0 turns
    // it off): codes/predictor scratch for `chain_levels` ladder levels
    int serial_chain = 1;
    int imz = 1;  // zero-imaginary-plane mode (QCS_IMZ=0 turns it off)
    int stream_commit = 1;   // wave layout: the streaming kernel's CTAs install their strides (QCS_STREAM_COMMIT=0: staged)
    int stream_persist = 1;  // ... from one persistent launch per gate (QCS_STREAM_PERSIST=0: a launch per wave)
    int stream_mode = 1;  // streaming kernel for element-wise gates (QCS_STREAM=0 turns it off; bit 2: also as the split path's encoder)
    int diag_local = 1;  // diagonal far/pair gates in the fused kernel (QCS_DIAG_LOCAL=0: split path)
    int zero_pass = 1;   // zero strides skip the codec (QCS_ZERO_PASS=0 turns it off)
    int ladder_exit = 1; // ladder levels give up at the byte budget (QCS_LADDER_EXIT=0 turns it off)
    int force_wide = 0;  // QCS_WIDE=1: 2 x 256-lane encoder CTAs for every gate (experiments)
    int debug_sync = 0;  // QCS_DEBUG_SYNC=1: synchronise and log after every kernel of a gate (debugging)
    bool all_im_zero = true;  // every im plane is zero (real state): real gates keep it
    int chain_levels = 0;
    int16_t* chain_codes = nullptr;
    double* chain_preds = nullptr;
    unsigned long long* cta_trace = nullptr;  // QCS_CTA_TRACE=1: per-slot phase cycles
    // Large states ("wave mode"): one arena, per-wave staging
    // buffers (slots, side, X) for `wave` slots, per-wave commit placed by the
    // host, in-place compaction through the X buffer.
    int big = 0;
    bool poisoned = false;       // a wave-layout gate failed after committing some waves
    uint64_t wave = 0;           // slots per wave (== NS in the small layout)
    uint64_t bump = 0;           // wave mode: arena fill (host-authoritative)
    uint64_t compactions = 0;
    double compact_ns = 0.0;     // host wall time spent compacting (diagnostics)
    uint64_t* mv_src = nullptr;  // [2NS] compaction work lists
    uint64_t* mv_dst = nullptr;
    uint64_t* mv_len = nullptr;
    Dev::Scal* h_sc = nullptr;   // pinned mirror
    qcs_stride_report* h_rep = nullptr;
    std::vector<void*> allocs;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    // per-kernel-class profiling (qcs_state_profile)
    int prof = 0;            // 0 off, 1 every kernel class, 2 the encoder (class 2) only
    bool prof_open = false;  // the last prof_start recorded a mark
    struct Mark {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> pool;
    double cls_ns[6] = {0, 0, 0, 0, 0, 0};
    uint64_t cls_n[6] = {0, 0, 0, 0, 0, 0};
};

namespace {

cudaEvent_t pool_event(qcs_dev_state* st)
{
    if (!st->pool.empty()) {
        cudaEvent_t e = st->pool.back();
        st->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void dbg_sync(qcs_dev_state* st, const char* what)
{
    if (!st->debug_sync) return;
    const cudaError_t e = cudaStreamSynchronize(st->stream);
    fprintf(stderr, "[qcs] %s: %s\n", what, cudaGetErrorString(e));
}

void prof_start(qcs_dev_state* st, int cls)
{
    st->prof_open = false;
    if (!st->prof || (st->prof == 2 && cls != 2)) return;
    qcs_dev_state::Mark m{cls, pool_event(st), pool_event(st)};
    cudaEventRecord(m.a, st->stream);
    st->marks.push_back(m);
    st->prof_open = true;
}

void prof_stop(qcs_dev_state* st)
{
    if (!st->prof_open || st->marks.empty()) return;
    cudaEventRecord(st->marks.back().b, st->stream);
    st->prof_open = false;
}

void prof_collect(qcs_dev_state* st)
{
    for (auto& m : st->marks) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) {
            st->cls_ns[m.cls] += (double)ms * 1e6;
            st->cls_n[m.cls] += 1;
        }
        st->pool.push_back(m.a);
        st->pool.push_back(m.b);
    }
    st->marks.clear();
    cudaGetLastError();
}

template <typename T>
int dalloc(qcs_dev_state* s, T** p, size_t count)
{
    void* q = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(QCS_E_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
    s->allocs.push_back(q);
    *p = static_cast<T*>(q);
    return 0;
}

int validate_gate(const qcs_dev_state* st, const qcs_gate_desc* g)
{
    const int n = st->d.n;
    switch (g->kind) {  // GateOp::validate, gate.cpp:109-137
        case 0:
        case 1:
            if (g->target < 0 || g->target >= n) return set_err(QCS_E_RANGE, "target qubit out of range");
            if (g->kind == 1) {
                if (g->control < 0 || g->control >= n) return set_err(QCS_E_RANGE, "control qubit out of range");
                if (g->control == g->target) return set_err(QCS_E_INVALID, "control qubit equals target qubit");
            }
            return 0;
        case 2:
            if (g->flip_index >= (1ull << n)) return set_err(QCS_E_RANGE, "flip index out of range");
            return 0;
        case 3:
            return 0;
        default:
            return set_err(QCS_E_INVALID, "unknown gate kind %d", g->kind);
    }
}

int validate_ladder(const double* lad, int nl, double theta)
{
    if (nl <= 0 || !lad) return set_err(QCS_E_INVALID, "error-bound ladder must not be empty");
    for (int i = 0; i < nl; ++i) {
        if (!(lad[i] >= 0.0) || !std::isfinite(lad[i]))
            return set_err(QCS_E_INVALID, "error bounds must be finite and >= 0");
        if (i > 0 && !(lad[i] > lad[i - 1])) return set_err(QCS_E_INVALID, "error bounds must be strictly increasing");
    }
    if (!(theta >= 1.0)) return set_err(QCS_E_INVALID, "ratio threshold must be >= 1");
    return 0;
}

// make_stride_plan (gate.cpp:313-403) in closed form.
Plan make_plan(const qcs_dev_state* st, const qcs_gate_desc* g)
{
    const int s = st->d.s;
    const uint64_t NS = st->d.NS;
    Plan p{};
    p.fixed = -1;
    p.kind = g->kind;
    p.t = g->target;
    p.c = g->kind == 1 ? g->control : -1;
    p.local_ctl = -1;
    p.pb = 0;
    auto add_fixed = [&](int pos, int v) {
        p.pos[p.npos] = pos;
        p.val[p.npos] = v;
        ++p.npos;
        if (p.npos == 2 && p.pos[0] > p.pos[1]) {
            std::swap(p.pos[0], p.pos[1]);
            std::swap(p.val[0], p.val[1]);
        }
    };
    if (g->kind == 0 || g->kind == 1) {
        const int t = g->target, c = p.c;
        if (c >= 0 && c < s) p.local_ctl = c;
        if (t < s) {
            p.pair = 0;
            if (c >= s) add_fixed(c - s, 1);
        } else {
            p.pair = 1;
            p.pb = t - s;
            add_fixed(t - s, 0);
            if (c >= s) add_fixed(c - s, 1);
        }
        p.n_units = NS >> p.npos;
    } else if (g->kind == 2) {
        p.fixed = (int64_t)(g->flip_index >> s);
        p.flip_off = g->flip_index & (st->d.L - 1);
        p.n_units = 1;
    } else {
        p.reflect = 1;
        p.n_units = NS;
    }
    return p;
}

uint64_t grid_for(uint64_t work, uint64_t block = 256)
{
    return umin64((work + block - 1) / block, 148ull * 32);
}
__global__ void k_set_mean(Dev d, double mr, double mi)
{
    d.sc->mean[0] = mr;
    d.sc->mean[1] = mi;
}

// CTA-wide copy of n16 16-byte words, four independent loads in flight per
// thread (the plain one-load loop left the copy kernels at ~2 TB/s)
__device__ __forceinline__ void cta_copy16(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t n16)
{
    const uint64_t T = blockDim.x;
    uint64_t i = threadIdx.x;
    for (; i + 3 * T < n16; i += 4 * T) {
        const uint4 a = __ldcs(src + i), b = __ldcs(src + i + T), c = __ldcs(src + i + 2 * T), e = __ldcs(src + i + 3 * T);
        dst[i] = a;
        dst[i + T] = b;
        dst[i + 2 * T] = c;
        dst[i + 3 * T] = e;
    }
    for (; i < n16; i += T) dst[i] = __ldcs(src + i);
}

// Wave mode: install the wave's new blocks at host-chosen arena offsets
// (new_off), replace the side index, tables, scale and sum (the staged commit
// of aalc.cpp:395-408, one wave at a time).
constexpr int COPY_THREADS = 256;
// slack: the offsets are k_wave_alloc's (new blocks carry slack16); 0: host-placed, exact size
__global__ void __launch_bounds__(COPY_THREADS) k_wave_commit(Dev d, LevelTag lt, uint64_t s0, const uint8_t* committed,
                                                             int slack)
{
    if (d.sc->err) return;
    const uint64_t loc = blockIdx.x >> 1;
    const int c = (int)(blockIdx.x & 1);
    const uint64_t slot = s0 + loc;
    if (committed && committed[slot]) return;  // installed by its encoder CTA
    const uint64_t j = d.job_stride[slot];
    const uint64_t g = 2 * j + c;
    const uint64_t len = d.slot_len[2 * slot + c];
    const uint64_t dst_off = d.new_off[2 * slot + c];
    const uint4* s4 = reinterpret_cast<const uint4*>(d.slot_out + (2 * loc + c) * d.slot_cap);
    uint4* d4 = reinterpret_cast<uint4*>(d.arena[0] + dst_off);
    cta_copy16(d4, s4, (len + 15) / 16);
    const SideEntry* ss = d.slot_side + (2 * loc + c) * d.nsub;
    SideEntry* ds = d.side + g * d.nsub;
    static_assert(sizeof(SideEntry) == 16, "side entries copy as 16-byte words");
    cta_copy16(reinterpret_cast<uint4*>(ds), reinterpret_cast<const uint4*>(ss), d.nsub);
    if (threadIdx.x == 0) {
        atomicAdd((unsigned long long*)&d.sc->gate_cin, (unsigned long long)(HEADER_BYTES + d.p_len[g]));
        if (dst_off != d.p_off[g]) {  // a new block (in place: offset and capacity stay)
            d.p_cap[g] = slack ? slack16(round16d(len)) : round16d(len);
            d.p_capoff[g] = dst_off;
        }
        d.p_off[g] = dst_off;
        d.p_len[g] = len;
        d.p_codec[g] = lt.slot_codec[slot];
        d.p_delta[g] = lt.slot_delta[slot];
        if (c == 0) {
            d.sum_sq[j] = d.slot_sum[slot];
            d.scale[j] = 1.0;
        }
    }
}

// Wave layout, device-side placement of a wave's new blocks (no host round
// trip): an exclusive scan of the 16-byte-rounded payload lengths of the wave's
// 2*(s1-s0) planes, one bump of the arena for the whole wave, new_off for
// k_wave_commit.  A wave that does not fit suspends the gate (QCS_SUSPEND,
// the wave's first unit in susp_unit): its blocks stay where they are, every
// later kernel is a no-op, and the host compacts the arena and resumes.
constexpr int ALLOC_THREADS = 1024;
// committed (null: none): slots their encoder CTAs installed already, inside the
// block k_wave_reserve set aside — the bump first moves past what they took.
__global__ void __launch_bounds__(ALLOC_THREADS) k_wave_alloc(Dev d, uint64_t s0, uint64_t m2, uint64_t unit0,
                                                              const uint8_t* committed)
{
    __shared__ uint64_t wsum[ALLOC_THREADS / 32];
    __shared__ uint64_t base_sh;
    __shared__ int ok_sh;
    if (d.sc->err) return;
    const int tid = threadIdx.x, wl = tid & 31, w = tid >> 5;
    // a plane whose new block fits the capacity of its current one (a block placed with slack,
    // p_cap / p_capoff, qcs_stream.cuh) is rewritten in place: by the commit every read of this
    // wave's inputs is over; any other gets a new block with slack
    auto plane_of = [&](uint64_t i) -> uint64_t { return 2 * d.job_stride[s0 + i / 2] + (i & 1); };
    auto in_place = [&](uint64_t i) -> bool {
        const uint64_t g = plane_of(i);
        return d.inplace && d.p_capoff[g] == d.p_off[g] && round16d(d.slot_len[2 * s0 + i]) <= d.p_cap[g];
    };
    auto need_of = [&](uint64_t i) -> uint64_t {
        if (i >= m2 || (committed && committed[s0 + i / 2]) || in_place(i)) return 0;
        return slack16(round16d(d.slot_len[2 * s0 + i]));
    };
    if (committed && tid == 0 && d.sc->wave_direct) {
        d.sc->bump += d.sc->wave_used;
        d.sc->wave_used = 0;
        d.sc->wave_direct = 0;
    }
    __syncthreads();
    uint64_t total = 0;
    for (uint64_t c0 = 0; c0 < m2; c0 += ALLOC_THREADS) total += need_of(c0 + tid);
    for (int o = 16; o; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    if (wl == 0) wsum[w] = total;
    __syncthreads();
    if (tid == 0) {
        uint64_t t = 0;
        for (int i = 0; i < ALLOC_THREADS / 32; ++i) t += wsum[i];
        const uint64_t b = d.sc->bump;
        ok_sh = b + t <= d.arena_cap;
        base_sh = b;
        if (ok_sh) {
            d.sc->bump = b + t;
        } else {
            d.sc->err = QCS_SUSPEND;
            d.sc->susp_unit = unit0;
        }
    }
    __syncthreads();
    if (!ok_sh) return;
    uint64_t carry = base_sh;
    for (uint64_t c0 = 0; c0 < m2; c0 += ALLOC_THREADS) {
        const uint64_t i = c0 + tid;
        const uint64_t v = need_of(i);
        uint64_t inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (wl >= o) inc += u;
        }
        __syncthreads();
        if (wl == 31) wsum[w] = inc;
        __syncthreads();
        uint64_t pre = 0, tot = 0;
        for (int k = 0; k < ALLOC_THREADS / 32; ++k) {
            if (k < w) pre += wsum[k];
            tot += wsum[k];
        }
        if (i < m2) d.new_off[2 * s0 + i] = (v == 0 && !(committed && committed[s0 + i / 2]) && in_place(i))
                                                ? d.p_off[plane_of(i)]
                                                : carry + pre + inc - v;
        carry += tot;
    }
}

// Wave layout, encoder-side commit: set the wave's worst case (every plane at
// its slot capacity) aside behind the bump when it fits — the CTAs then install
// their strides themselves (StreamCommit); otherwise the staged path.
__global__ void k_wave_reserve(Dev d, uint64_t m2)
{
    if (d.sc->err) return;
    d.sc->wave_used = 0;
    d.sc->wave_direct = (d.sc->bump + m2 * round16d(d.slot_cap) <= d.arena_cap) ? 1 : 0;
}

// Persistent streaming kernel, around its launch: reset the slot queue (and, for a gate's first
// attempt, the installed flags and their count); afterwards a suspension inside it is tagged for
// the host (SUSP_PERSIST + progress).
__global__ void k_persist_begin(Dev d, uint64_t n_slots, int resume)
{
    // (a gate queued behind a suspended one must not touch the suspended gate's flags)
    if (d.sc->err) return;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i == 0) {
        d.sc->q_head = 0;
        d.sc->persist_susp = 0;
        if (!resume) d.sc->persist_done = 0;
    }
    if (!resume && i < n_slots) {
        d.committed[i] = 0;
        d.redo[i] = 0;
    }
}
__global__ void k_persist_end(Dev d, int64_t gate_index)
{
    if (d.sc->err == QCS_SUSPEND && d.sc->persist_susp && d.sc->err_gate < 0) {
        d.sc->err_gate = (int)gate_index;
        d.sc->susp_unit = SUSP_PERSIST | d.sc->persist_done;
    }
}

// Wave layout, before a gate's first wave: when its new blocks (estimated as
// 5/4 of the blocks it rewrites) would not fit behind the bump but would after
// a compaction, suspend the gate at unit 0 -- the host compacts before any of
// its waves is encoded (a wave that still does not fit suspends in k_wave_alloc).
__global__ void __launch_bounds__(ALLOC_THREADS) k_precheck(Dev d, uint64_t n_slots)
{
    __shared__ unsigned long long need_sh, live_sh;
    if (d.sc->err) return;
    if (threadIdx.x == 0) need_sh = live_sh = 0;
    __syncthreads();
    unsigned long long need = 0, live = 0;
    for (uint64_t s = threadIdx.x; s < n_slots; s += ALLOC_THREADS) {
        const uint64_t j = d.job_stride[s];
        need += round16d(d.p_len[2 * j]) + round16d(d.p_len[2 * j + 1]);
    }
    for (uint64_t g = threadIdx.x; g < 2 * d.NS; g += ALLOC_THREADS) live += round16d(d.p_len[g]);
    atomicAdd(&need_sh, need);
    atomicAdd(&live_sh, live);
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint64_t est = need_sh + need_sh / 4 + (1ull << 20);
    if (d.sc->bump + est > d.arena_cap && live_sh + est <= d.arena_cap) {
        d.sc->err = QCS_SUSPEND;
        d.sc->susp_unit = 0;
    }
}

// Byte moves for compaction: item i copies len[i] bytes from src+so[i] to
// dst+do[i] (16-byte aligned; one CTA per item).
__global__ void __launch_bounds__(COPY_THREADS) k_move(const uint8_t* src, uint8_t* dst, const uint64_t* so,
                                              const uint64_t* dof, const uint64_t* len)
{
    const uint64_t i = blockIdx.x;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + so[i]);
    uint4* d4 = reinterpret_cast<uint4*>(dst + dof[i]);
    cta_copy16(d4, s4, (len[i] + 15) / 16);
}

inline uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// In-place compaction of the single arena: live blocks slide down in offset
// order.  Batches go arena -> X -> arena; a block's destination never reaches
// past its own source end, so it can only overlap sources of blocks already
// moved (earlier batches) or of its own batch (bounced).  Blocks shared by
// several planes (basis-state zero block) move once.
int compact_arena_impl(qcs_dev_state* st);
int compact_arena(qcs_dev_state* st)
{
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = compact_arena_impl(st);
    st->compact_ns += (double)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

int compact_arena_impl(qcs_dev_state* st)
{
    Dev& d = st->d;
    cudaStream_t s = st->stream;
    const uint64_t np = 2 * d.NS;
    CU(cudaStreamSynchronize(s));
    std::vector<uint64_t> off(np), len(np), nof(np);
    CU(cudaMemcpy(off.data(), d.p_off, 8 * np, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(len.data(), d.p_len, 8 * np, cudaMemcpyDeviceToHost));
    std::vector<uint64_t> ord(np);
    for (uint64_t i = 0; i < np; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](uint64_t a, uint64_t b) { return off[a] < off[b]; });
    const uint64_t bounce = 16 * st->wave * d.L;
    uint8_t* X = reinterpret_cast<uint8_t*>(d.X);
    std::vector<uint64_t> bs, bt, bd, bl;  // batch: src, bounce offset, dst, len
    uint64_t at = 0, bfill = 0;
    auto flush = [&]() -> int {
        if (bs.empty()) return 0;
        const uint64_t m = bs.size();
        // sources ascend and every later block lies above them: when the batch's destinations end
        // at or below its first source, no destination byte is a source still to be read — one
        // pass inside the arena instead of the bounce through X (the usual case after a few gates:
        // the live blocks are the newest, at the top)
        bool direct = true;
        for (uint64_t i = 0; i < m && direct; ++i) direct = bd[i] + round16(bl[i]) <= bs[0];
        CU(cudaMemcpyAsync(st->mv_src, bs.data(), 8 * m, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(st->mv_dst, (direct ? bd : bt).data(), 8 * m, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(st->mv_len, bl.data(), 8 * m, cudaMemcpyHostToDevice, s));
        if (direct) {
            k_move<<<(unsigned)m, COPY_THREADS, 0, s>>>(d.arena[0], d.arena[0], st->mv_src, st->mv_dst, st->mv_len);
            st->launches += 1;
        } else {
            k_move<<<(unsigned)m, COPY_THREADS, 0, s>>>(d.arena[0], X, st->mv_src, st->mv_dst, st->mv_len);
            CU(cudaMemcpyAsync(st->mv_src, bd.data(), 8 * m, cudaMemcpyHostToDevice, s));
            k_move<<<(unsigned)m, COPY_THREADS, 0, s>>>(X, d.arena[0], st->mv_dst, st->mv_src, st->mv_len);
            st->launches += 2;
        }
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(s));  // the host vectors are reused
        bs.clear(), bt.clear(), bd.clear(), bl.clear();
        bfill = 0;
        return 0;
    };
    for (uint64_t k = 0; k < np;) {
        const uint64_t g0 = ord[k];
        uint64_t k2 = k + 1;
        while (k2 < np && off[ord[k2]] == off[g0]) ++k2;
        const uint64_t l16 = round16(len[g0]);
        if (bfill + l16 > bounce) {
            const int rc = flush();
            if (rc) return rc;
        }
        if (at != off[g0] && l16) {
            bs.push_back(off[g0]);
            bt.push_back(bfill);
            bd.push_back(at);
            bl.push_back(len[g0]);
            bfill += l16;
        }
        for (uint64_t q = k; q < k2; ++q) nof[ord[q]] = at;
        at += l16;
        k = k2;
    }
    int rc = flush();
    if (rc) return rc;
    CU(cudaMemcpy(d.p_off, nof.data(), 8 * np, cudaMemcpyHostToDevice));
    CU(cudaMemset(d.p_capoff, 0xff, 8 * np));  // packed by length: no block keeps its slack
    st->bump = at;
    CU(cudaMemcpy(&d.sc->bump, &st->bump, 8, cudaMemcpyHostToDevice));
    ++st->compactions;
    return 0;
}

// Reserve `need` arena bytes in wave mode (compacting when full).
int big_reserve(qcs_dev_state* st, uint64_t need, uint64_t* at)
{
    st->bump = st->h_sc->bump;  // the device's bump is authoritative (k_wave_alloc); h_sc is fresh
    if (st->bump + need > st->d.arena_cap) {
        const int rc = compact_arena(st);
        if (rc) return rc;
    }
    if (st->bump + need > st->d.arena_cap) return QCS_E_NOMEM;
    *at = st->bump;
    st->bump += need;
    return 0;
}

// Wave mode: place and install the wave [s0, s1) after its encode.
int big_commit_wave(qcs_dev_state* st, uint64_t s0, uint64_t s1, uint64_t gate_index, uint64_t units_done)
{
    Dev& d = st->d;
    cudaStream_t s = st->stream;
    const uint64_t m = 2 * (s1 - s0);
    std::vector<uint64_t> len(m), nof(m);
    CU(cudaMemcpyAsync(len.data(), d.slot_len + 2 * s0, 8 * m, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(st->h_sc, d.sc, sizeof(Dev::Scal), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (st->h_sc->err) return -1;  // device error: the caller reports it
    uint64_t need = 0;
    for (uint64_t i = 0; i < m; ++i) need += round16(len[i]);
    uint64_t at = 0;
    const int rc = big_reserve(st, need, &at);
    if (rc == QCS_E_NOMEM)
        return set_err(QCS_E_NOMEM, units_done == 0 ? "gate %llu failed: block arena exhausted"
                                                    : "gate %llu failed: block arena exhausted after %llu of its units were committed",
                       (unsigned long long)gate_index, (unsigned long long)units_done);
    if (rc) return rc;
    for (uint64_t i = 0; i < m; ++i) {
        nof[i] = at;
        at += round16(len[i]);
    }
    CU(cudaMemcpyAsync(d.new_off + 2 * s0, nof.data(), 8 * m, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(&d.sc->bump, &st->bump, 8, cudaMemcpyHostToDevice, s));
    k_wave_commit<<<(unsigned)m, COPY_THREADS, 0, s>>>(d, st->lt, s0, nullptr, 0);
    ++st->launches;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s));  // nof / bump are host locals
    return 0;
}

// Scratch for the serial-chain mode: codes and sub-chunk predictors of
// `levels` ladder levels for one wave.  Grows once; false (and the event-
// round path) when it would take more than a quarter of the free memory.
bool ensure_chain_scratch(qcs_dev_state* st, int levels)
{
    if (st->chain_levels >= levels) return true;
    const Dev& d = st->d;
    const size_t rows = 2 * st->wave;
    const size_t cb = (size_t)levels * rows * d.L * sizeof(int16_t);
    const size_t pb = (size_t)levels * rows * d.nsub * sizeof(double);
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess || cb + pb > fr / 4) {
        cudaGetLastError();
        return false;
    }
    if (st->chain_codes) cudaFree(st->chain_codes), cudaFree(st->chain_preds);
    auto drop = [&](void* q) { st->allocs.erase(std::remove(st->allocs.begin(), st->allocs.end(), q), st->allocs.end()); };
    drop(st->chain_codes);
    drop(st->chain_preds);
    st->chain_codes = nullptr;
    st->chain_preds = nullptr;
    st->chain_levels = 0;
    if (dalloc(st, &st->chain_codes, cb / sizeof(int16_t)) || dalloc(st, &st->chain_preds, pb / sizeof(double))) {
        g_err.clear();
        return false;
    }
    st->chain_levels = levels;
    return true;
}

// One gate, fully stream-ordered.  rec_index < 0: no record.
// given_mean == kMeanPreset: reflect_mean uses the mean already stored on the
// device (the cluster driver folds it across shards, qcs_cluster.cuh)
const double kMeanPreset[2] = {0.0, 0.0};

// load (x_ext != null): the strides [load_first, load_first + load_count)
// are compressed from the caller's raw device planes x_ext (g unused).
int enqueue_gate(qcs_dev_state* st, const qcs_gate_desc* g, const double* lad, int nl,
                 double theta, int64_t rec_index, uint64_t gate_index, uint64_t* n_slots_out,
                 int renorm = 1, const double* given_mean = nullptr, const double* x_ext = nullptr,
                 uint64_t load_first = 0, uint64_t load_count = 0, uint64_t first_unit = 0,
                 bool precheck_done = false)
{
    // wave layout: the gate's waves before first_unit are committed; a gate suspended inside the
    // persistent streaming kernel resumes with every slot not installed yet (SUSP_PERSIST)
    const bool resume = first_unit > 0;
    if (first_unit & SUSP_PERSIST) first_unit = 0;  // (the low bits count installed strides: progress only)
    Dev& d = st->d;
    cudaStream_t s = st->stream;
    static const qcs_gate_desc k_load_desc{KIND_LOAD, 0, -1, 0, 0, {1, 0, 0, 0, 0, 0, 1, 0}};
    if (x_ext) g = &k_load_desc;
    Plan p = x_ext ? Plan{} : make_plan(st, g);
    if (x_ext) {
        p.fixed = -1;
        p.kind = KIND_LOAD;
        p.c = -1;
        p.local_ctl = -1;
        p.n_units = load_count;
        p.first = load_first;
    }
    const uint64_t n_slots = p.pair ? 2 * p.n_units : p.n_units;
    *n_slots_out = n_slots;
    const uint64_t gen = ++st->gen;

    prof_start(st, 5);
    // zero-imaginary-plane mode: real gates (single / controlled with a real
    // unitary, phase flips) on strides whose im planes are all zero
    const bool real_gate = p.kind == 2 || (p.kind <= 1 && g->u[1] == 0.0 && g->u[3] == 0.0 && g->u[5] == 0.0 &&
                                           g->u[7] == 0.0);
    const bool imz = real_gate && st->imz;
    // a complex gate (or reflect_mean, or a load) may fill im planes: cleared
    // before the first wave commits, so a gate that fails part-way never
    // leaves the flag claiming a real state
    if (!real_gate) st->all_im_zero = false;
    const bool diag_gate = p.kind <= 1 && g->u[2] == 0.0 && g->u[3] == 0.0 && g->u[4] == 0.0 && g->u[5] == 0.0;
    // diagonal gates (u12 = u21 = 0: CP, CZ, Z, T, phase): every element is
    // gated on its own (qcs_fused.cuh, FusedArgs::diag), so far partners and
    // pair units need no partner data and stay in the fused in-chunk kernel;
    // the plan, the joint pair ladder and the reports are unchanged.  (With
    // fewer slots than SMs the split path's chunk-parallel decode keeps every
    // SM busy, which the per-stride fused kernel cannot: C1.)
    const bool diag = !x_ext && diag_gate && st->diag_local && (p.pair || (1ull << p.t) >= FUSED_SPAN) &&
                      n_slots >= 148;
    // zero-stride pass: a slot's output depends on its own stride alone, or
    // (pair units on the split path) on both strides of its unit
    const int zmode = !st->zero_pass || p.kind == KIND_LOAD || p.reflect ? 0 : (p.pair && !diag ? 2 : 1);
    k_make_jobs<<<(unsigned)grid_for(n_slots), 256, 0, s>>>(d, p, n_slots, gen, st->lt, lad[0] > 0.0 ? 1 : 0, lad[0],
                                                            imz ? (st->all_im_zero ? 2 : 1) : 0, zmode, resume ? 1 : 0);
    ++st->launches;
    if (st->big && !resume && !precheck_done) {
        k_precheck<<<1, ALLOC_THREADS, 0, s>>>(d, n_slots);
        ++st->launches;
    }
    if (zmode && n_slots > 148) {  // (up to one CTA per SM the order is moot)
        const uint64_t wslots = std::max<uint64_t>(1, st->wave / (p.pair ? 2 : 1)) * (p.pair ? 2 : 1);
        k_slot_order<<<1, ORDER_THREADS, 0, s>>>(d, n_slots, wslots);
        ++st->launches;
    }
    prof_stop(st);
    dbg_sync(st, "k_make_jobs");
    if (resume) {
        // the mean of reflect_mean was taken before the first wave (aalc.cpp:270-295)
    } else if (p.reflect && given_mean == kMeanPreset) {
        // sharded run (qcs_cluster): the global mean is already in d.sc->mean
    } else if (p.reflect && given_mean) {  // sharded run: mean combined across ranks
        k_set_mean<<<1, 1, 0, s>>>(d, given_mean[0], given_mean[1]);
        ++st->launches;
    } else if (p.reflect) {  // mean pass (aalc.cpp:270-295) needs every stride first
        prof_start(st, 4);
        k_stride_partial<<<(unsigned)d.NS, 128, 0, s>>>(d);
        k_mean<<<1, 1, 0, s>>>(d);
        prof_stop(st);
        st->launches += 2;
    }
    // cross-chunk partners (pair units, in-stride targets >= 2^12): decode +
    // gate fully parallel into X, then the encoder reads X (split path)
    int dg = -1;
    if (diag) dg = -1;
    else if (p.pair) dg = DG_PAIR;
    else if (p.kind <= 1 && (1ull << p.t) >= FUSED_SPAN) dg = DG_FAR;
    // in-chunk partners take the split path too when asked (QCS_SPLIT_LOCAL)
    else if (p.kind <= 1 && st->split_local && (1ull << p.t) >= DG_HALF) dg = DG_FAR;
    else if (p.kind <= 1 && st->split_local && d.L >= DG_IN_CH) dg = DG_IN;
    // gates with fewer units than SMs: one 512-thread CTA per stride
    // 2 x 256-lane CTAs (16 warps, one per SM) when the usual 2 x 128-lane CTAs
    // would leave SMs at 8 warps: fewer units than SMs, or up to two per SM of
    // which some may be all-zero strides (zero-stride pass) -- the encoder is
    // latency-bound and its throughput per SM follows the resident warps.
    // Real states (zero-imaginary-plane mode) keep the narrow CTAs (measured).
    const bool wide = (n_slots < 148 || (n_slots <= 296 && !imz) || st->force_wide) && d.L >= 2 * FUSED_SPAN;
    const int fm = dg >= 0 ? (wide ? FM_RAW2_W : FM_RAW2) : (wide ? FM_LOCAL_W : FM_LOCAL);  // pairs always split
    if (dg >= 0) {
        if (const int rc = set_smem_attr(reinterpret_cast<const void*>(k_decode_gate), (int)DG_SMEM)) return rc;
        if (const int rc = set_smem_attr(reinterpret_cast<const void*>(k_decode_gate_re), (int)DG_SMEM)) return rc;
    }
    if (x_ext) dg = -1;
    GateParams gp;
    for (int i = 0; i < 8; ++i) gp.u[i] = g->u[i];
    // Serial-chain mode: lossy levels whose 2*delta is not a
    // power of two have no lattice to verify lanes against, so their
    // reference chains are computed up front, serially per plane but for all
    // planes and all such levels at once (k_serial_chain); the encoder then
    // only tokenizes.  Needs the gated planes in X: the split path provides
    // them, in-chunk gates get a decode+gate+snap pass that only writes X.
    ChainLevels chl{};
    int lev_of[64];
    for (int k = 0; k < nl && k < 64; ++k) {
        lev_of[k] = -1;
        const CodecParams cpk = make_params(lad[k]);
        if (cpk.lossy && !cpk.pow2 && chl.n < 8) {
            lev_of[k] = chl.n;
            chl.delta[chl.n] = lad[k];
            chl.td[chl.n] = cpk.td;
            chl.inv[chl.n] = 1.0 / cpk.td;
            chl.lim[chl.n] = cpk.lim;
            ++chl.n;
        }
    }
    bool chain = chl.n > 0 && st->serial_chain && nl <= 64;
    for (int k = 0; chain && k < nl; ++k)
        if (make_params(lad[k]).lossy && !make_params(lad[k]).pow2 && lev_of[k] < 0) chain = false;
    if (chain) chain = ensure_chain_scratch(st, chl.n);
    // QCS_SERIAL_CHAIN=1: policy (default); 2: always the serial chain
    const int* chain_flag = nullptr;
    if (chain && st->serial_chain == 1) {
        if (!resume) {  // a resumed gate keeps the choice it started with
            const unsigned long long thr = std::max<unsigned long long>(1, 2 * d.NS * d.nsub / 16);
            k_chain_policy<<<1, 1, 0, s>>>(d, thr);
            ++st->launches;
        }
        chain_flag = &d.sc->chain_on;
    }
    const int fm_lvl = (chain || x_ext) ? (wide ? FM_RAW2_W : FM_RAW2) : fm;
    auto fused_args = [&](double delta, uint64_t s0) {
        FusedArgs a{};
        a.arena0 = d.arena[0];
        a.arena1 = d.arena[1];
        a.arena_cur = &d.sc->cur;
        a.p_off = d.p_off;
        a.p_len = d.p_len;
        a.p_codec = d.p_codec;
        a.p_delta = d.p_delta;
        a.side_in = d.side;
        a.scale = d.scale;
        a.job_stride = d.job_stride;
        for (int i = 0; i < 8; ++i) a.u[i] = g->u[i];
        a.kind = p.kind;
        a.diag = diag ? (p.pair ? 2 : 1) : 0;
        a.t = p.t;
        a.local_ctl = p.local_ctl;
        a.flip_off = p.flip_off;
        a.mean = d.sc->mean;
        a.n = d.L;
        a.pending = d.pending;
        a.slot_base = s0;
        a.max_rounds = st->max_rounds;
        a.cta_trace = st->cta_trace;
        a.snap = 1;
        a.pool = d.pool;
        a.out = d.pool ? d.arena[0] : d.slot_out;
        a.cap = d.slot_cap;
        a.side = d.pool ? d.side : d.slot_side;
        a.nsub = d.nsub;
        a.out_len = d.slot_len;
        a.sumsq = d.slot_sum;
        a.cp = make_params(delta);
        a.counters = d.counters;
        a.im_zero = imz ? d.im_zero : nullptr;
        a.err = &d.sc->err;
        a.zero_slot = zmode ? d.zero_slot : nullptr;
        a.order = (zmode && n_slots > 148) ? d.order : nullptr;
        return a;
    };
    // wave layout, single-level ladder, streaming kernel: the encoder CTAs install their strides
    // (QCS_STREAM_COMMIT=0: always the staged commit)
    const bool wave_direct = st->stream_commit && st->big && nl == 1 && !x_ext && !chain && st->stream_mode &&
                             ((p.kind <= 1 && diag_gate) || p.kind == 2 || p.kind == 3) &&
                             (fm_lvl == FM_LOCAL || fm_lvl == FM_LOCAL_W) && make_params(lad[0]).lossy &&
                             make_params(lad[0]).pow2 && d.L >= SUB && d.L <= (1ull << 31);
    // ... and from one persistent kernel over the whole gate instead of a launch per wave
    // (QCS_STREAM_PERSIST=0: waves)
    const bool persist = wave_direct && st->stream_persist;
    if (persist) {
        FusedArgs as = fused_args(lad[0], 0);
        as.diag = p.kind <= 1 ? (p.pair ? 2 : 1) : 0;
        as.X = d.X;  // (scratch of the sum's serial head: min(512, L) doubles per staging slot)
        as.x_plane_stride = d.L;
        as.ladder_theta = 0.0;
        StreamCommit dc{};
        dc.bump_rw = (unsigned long long*)&d.sc->bump;
        dc.arena_cap = d.arena_cap;
        dc.err_rw = &d.sc->err;
        dc.persist_done = &d.sc->persist_done;
        dc.persist_susp = &d.sc->persist_susp;
        dc.p_cap = d.inplace ? d.p_cap : nullptr;
        dc.p_capoff = d.p_capoff;
        dc.arena = d.arena[0];
        dc.side = d.side;
        dc.p_off = d.p_off;
        dc.p_len = d.p_len;
        dc.p_codec = d.p_codec;
        dc.p_delta = d.p_delta;
        dc.scale = d.scale;
        dc.sum_sq = d.sum_sq;
        dc.gate_cin = (unsigned long long*)&d.sc->gate_cin;
        dc.committed = d.committed;
        const uint64_t grid = std::min<uint64_t>(n_slots, st->wave);
        prof_start(st, 2);
        k_persist_begin<<<(unsigned)grid_for(std::max<uint64_t>(n_slots, 1)), 256, 0, s>>>(d, n_slots, resume ? 1 : 0);
        const int rc = launch_stream_persist(as, d.redo, dc, n_slots, &d.sc->q_head, grid, s);
        if (rc) return rc;
        k_persist_end<<<1, 1, 0, s>>>(d, (int64_t)gate_index);
        prof_stop(st);
        st->launches += 3;
        dbg_sync(st, "k_stream_persist");
    }
    const uint64_t spu = p.pair ? 2 : 1;                        // slots per unit
    const uint64_t wave_units = std::max<uint64_t>(1, st->wave / spu);
    for (uint64_t u0 = first_unit; u0 < p.n_units; u0 += wave_units) {
        const uint64_t u1 = std::min<uint64_t>(p.n_units, u0 + wave_units);
        const uint64_t s0 = u0 * spu, s1 = u1 * spu, nw = s1 - s0;
        if (dg >= 0) {
            const uint64_t chunks = dg == DG_PAIR ? (d.L + DG_HALF - 1) / DG_HALF
                                                  : (dg == DG_FAR ? d.L / (2 * DG_HALF) : d.L / DG_IN_CH);
            const uint64_t units = dg == DG_PAIR ? (u1 - u0) : nw;
            prof_start(st, 0);
            const bool re_only = imz && st->all_im_zero && dg != DG_IN && d.L >= DG_RE_CH &&
                                 (dg == DG_PAIR || (1ull << p.t) >= (uint64_t)DG_RE_CH);
            if (re_only) {
                const uint64_t chunks_re = dg == DG_PAIR ? (d.L + DG_RE_CH - 1) / DG_RE_CH : d.L / (2 * DG_RE_CH);
                k_decode_gate_re<<<(unsigned)(units * chunks_re), DG_R, DG_SMEM, s>>>(d, p, gp, dg, chunks_re, s0,
                                                                                      zmode ? d.zero_slot : nullptr);
            } else {
                k_decode_gate<<<(unsigned)(units * chunks), DG_R, DG_SMEM, s>>>(d, p, gp, dg, chunks, s0,
                                                                              imz ? d.im_zero : nullptr,
                                                                              zmode ? d.zero_slot : nullptr);
            }
            prof_stop(st);
            ++st->launches;
            dbg_sync(st, "k_decode_gate");
        }
        // the wave's raw input planes: the caller's (load) or the scratch X
        const double* xw = x_ext ? x_ext + s0 * 2 * d.L : d.X;
        if (chain) {
            if (dg < 0 && !x_ext) {  // in-chunk gate: decode + gate + snap into X only
                FusedArgs a = fused_args(lad[0], s0);
                a.dump_x = d.X;
                prof_start(st, 0);
                const int rc = launch_fused(a, fm, nw, s);
                prof_stop(st);
                if (rc) return rc;
                ++st->launches;
            }
            const uint64_t chains = 2 * nw * (uint64_t)chl.n;
            prof_start(st, 1);
            k_serial_chain<<<(unsigned)((chains + 127) / 128), 128, 0, s>>>(xw, 2 * nw, d.L, d.nsub, chl,
                                                                           st->chain_codes, st->chain_preds,
                                                                           d.pending, s0, chain_flag, &d.sc->err);
            prof_stop(st);
            ++st->launches;
        }
        for (int k = 0; k < nl; ++k) {
            FusedArgs a = fused_args(lad[k], s0);
            if (fm_lvl == FM_RAW2 || fm_lvl == FM_RAW2_W) {  // split path: gated, snapped planes in X
                a.X = xw;
                a.x_plane_stride = d.L;
                a.snap = 0;  // gated planes were snapped; a load's, in place by k_snap
            }
            if (chain && lev_of[k] >= 0) {
                a.pre_codes = st->chain_codes + (uint64_t)lev_of[k] * 2 * nw * d.L;
                a.pre_pred = st->chain_preds + (uint64_t)lev_of[k] * 2 * nw * d.nsub;
                a.chain_on = chain_flag;
            }
            // early exit of levels that cannot reach theta (all but the last)
            a.ladder_theta = (k < nl - 1 && st->ladder_exit) ? theta : 0.0;
            if (k > 0) {  // level 0 was tagged by k_make_jobs
                prof_start(st, 5);
                k_tag_level<<<(unsigned)grid_for(nw), 256, 0, s>>>(d, st->lt, s0, s1, a.cp.lossy ? 1 : 0, lad[k]);
                prof_stop(st);
                ++st->launches;
            }
            prof_start(st, 2);
            int rc = 0;
            // element-wise gates at a power-of-two lossy level: the streaming
            // kernel first; the legacy encoder then only re-encodes the slots
            // it left (escapes, off-lattice predictors: d.redo)
            const bool elementwise = (p.kind <= 1 && diag_gate) || p.kind == 2 || p.kind == 3;
            const bool stream_level = st->stream_mode && a.cp.lossy && a.cp.pow2 && d.L >= SUB && d.L <= (1ull << 31);
            if (persist) {
                // the persistent kernel encoded and installed the slots; what it left (d.redo) is
                // re-encoded here and goes through the staged commit
                a.redo_only = d.redo;
            } else if (stream_level && elementwise && (fm_lvl == FM_LOCAL || fm_lvl == FM_LOCAL_W) && !a.dump_x) {
                FusedArgs as = a;
                if (p.kind <= 1) as.diag = p.pair ? 2 : 1;
                as.X = d.X;  // (scratch of the sum's serial head: min(512, L) doubles per slot)
                as.x_plane_stride = d.L;
                StreamCommit dc{};
                if (wave_direct) {
                    k_wave_reserve<<<1, 1, 0, s>>>(d, 2 * nw);
                    ++st->launches;
                    dc.direct = &d.sc->wave_direct;
                    dc.wave_used = &d.sc->wave_used;
                    dc.bump = &d.sc->bump;
                    dc.arena = d.arena[0];
                    dc.side = d.side;
                    dc.p_off = d.p_off;
                    dc.p_len = d.p_len;
                    dc.p_codec = d.p_codec;
                    dc.p_delta = d.p_delta;
                    dc.scale = d.scale;
                    dc.sum_sq = d.sum_sq;
                    dc.gate_cin = (unsigned long long*)&d.sc->gate_cin;
                    dc.committed = d.committed;
                }
                rc = launch_stream<false>(as, d.redo, dc, nw, s);
                if (rc) return rc;
                ++st->launches;
                a.redo_only = d.redo;
            } else if (stream_level && (fm_lvl == FM_RAW2 || fm_lvl == FM_RAW2_W) && !a.pre_codes && (st->stream_mode & 4)) {
                // split path (or a load): the planes are in X, the streaming walk only encodes them.
                // Experimental (QCS_STREAM=5): measured slower than the legacy encoder there (C2 2.3e10
                // against 3.5e10: lane-strided reads of X without a shared-memory transpose, and no
                // zero-imaginary-plane shortcut)
                rc = launch_stream<true>(a, d.redo, StreamCommit{}, nw, s);
                if (rc) return rc;
                ++st->launches;
                a.redo_only = d.redo;
            }
            rc = launch_fused(a, fm_lvl, nw, s);
            prof_stop(st);
            if (rc) return rc;
            ++st->launches;
            dbg_sync(st, "k_fused");
            if (!st->big && k == nl - 1) {  // last level + commit in one kernel
                prof_start(st, 3);
                k_ladder_commit<<<(unsigned)((p.n_units + 127) / 128), 128, 0, s>>>(d, st->lt, p, lad[k], theta);
                prof_stop(st);
            } else {
                prof_start(st, 5);
                k_ladder<<<(unsigned)((u1 - u0 + 127) / 128), 128, 0, s>>>(d, p, u0, u1, lad[k], theta, k == nl - 1);
                prof_stop(st);
            }
            ++st->launches;
        }
        if (st->big) {  // place (device bump) and install the wave: no host round trip
            prof_start(st, 3);
            k_wave_alloc<<<1, ALLOC_THREADS, 0, s>>>(d, s0, 2 * nw, u0, wave_direct ? d.committed : nullptr);
            k_wave_commit<<<(unsigned)(2 * nw), COPY_THREADS, 0, s>>>(d, st->lt, s0, wave_direct ? d.committed : nullptr, 1);
            prof_stop(st);
            st->launches += 2;
        }
    }
    prof_start(st, 3);
    k_norm<<<1, NORM_THREADS, 0, s>>>(d, n_slots, rec_index < 0 ? 0 : (uint64_t)rec_index, gate_index, renorm);
    prof_stop(st);
    ++st->launches;
    dbg_sync(st, "k_norm");
    CU(cudaGetLastError());
    return 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* qcs_last_error(void) { return g_err.c_str(); }
int qcs_version(void) { return 1; }

void qcs_state_destroy(qcs_dev_state_t st)
{
    if (!st) return;
    cudaSetDevice(st->device);
    if (st->stream) cudaStreamSynchronize(st->stream);
    for (void* p : st->allocs) cudaFree(p);
    if (st->h_sc) cudaFreeHost(st->h_sc);
    if (st->h_rep) cudaFreeHost(st->h_rep);
    for (auto& m : st->marks) {
        cudaEventDestroy(m.a);
        cudaEventDestroy(m.b);
    }
    for (auto e : st->pool) cudaEventDestroy(e);
    if (st->ev_a) cudaEventDestroy(st->ev_a);
    if (st->ev_b) cudaEventDestroy(st->ev_b);
    if (st->stream) cudaStreamDestroy(st->stream);
    delete st;
}

int qcs_state_create(int n, int s, uint64_t basis, int device, qcs_dev_state_t* out)
{
    if (n < 1 || n > 59) return set_err(QCS_E_INVALID, "n_qubits must be in [1, 59], got %d", n);
    if (s < 0 || s > n) return set_err(QCS_E_INVALID, "stride_bits must be in [0, n_qubits], got %d", s);
    const bool zero_state = basis == ~0ull;  // shard that holds no amplitude
    if (!zero_state && basis >= (1ull << n)) return set_err(QCS_E_RANGE, "basis index out of range");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(QCS_E_CUDA, "no CUDA device available (the engine has no CPU path)");
    }
    if (device < 0 || device >= ndev) return set_err(QCS_E_INVALID, "bad device %d", device);
    qcs_dev_state* st = new qcs_dev_state();
    st->device = device;
    if (const char* e = getenv("QCS_SPLIT_LOCAL")) st->split_local = atoi(e);
    if (const char* e = getenv("QCS_SERIAL_CHAIN")) st->serial_chain = atoi(e);
    if (const char* e = getenv("QCS_IMZ")) st->imz = atoi(e);
    if (const char* e = getenv("QCS_STREAM")) st->stream_mode = atoi(e);
    if (const char* e = getenv("QCS_STREAM_COMMIT")) st->stream_commit = atoi(e);
    if (const char* e = getenv("QCS_STREAM_PERSIST")) st->stream_persist = atoi(e);
    if (const char* e = getenv("QCS_DIAG_LOCAL")) st->diag_local = atoi(e);
    if (const char* e = getenv("QCS_ZERO_PASS")) st->zero_pass = atoi(e);
    if (const char* e = getenv("QCS_LADDER_EXIT")) st->ladder_exit = atoi(e);
    if (const char* e = getenv("QCS_WIDE")) st->force_wide = atoi(e);
    if (const char* e = getenv("QCS_DEBUG_SYNC")) st->debug_sync = atoi(e);
    if (const char* e = getenv("QCS_MAX_ROUNDS")) st->max_rounds = std::max(1, atoi(e));
    cudaSetDevice(device);
    int rc = 0;
#define TRY(x)                    \
    do {                          \
        rc = (x);                 \
        if (rc) {                 \
            qcs_state_destroy(st); \
            return rc;            \
        }                         \
    } while (0)
    Dev& d = st->d;
    d.n = n;
    d.s = s;
    d.L = 1ull << s;
    d.NS = 1ull << (n - s);
    d.nsub = (d.L + SUB - 1) / SUB;
    const uint64_t raw = (16ull << n);
    if (cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking) != cudaSuccess) {
        qcs_state_destroy(st);
        return set_err(QCS_E_CUDA, "stream creation failed");
    }
    d.slot_cap = payload_cap(d.L);
    // layout: small (two arenas, whole-gate staging, device-side commit) when
    // it fits comfortably, else wave mode
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const uint64_t side_b = 2 * d.NS * d.nsub * sizeof(SideEntry);
    const uint64_t small_arena = std::max<uint64_t>(raw + raw / 8 + 4096 * d.NS, 1ull << 24);
    const uint64_t pool_b = 4 * d.NS * d.slot_cap;  // two slots per plane
    const uint64_t small_need = pool_b + 2 * side_b + raw;
    const char* fb = getenv("QCS_FORCE_BIG");
    st->big = (fb && atoi(fb)) || (double)small_need > 0.7 * (double)free_b;
    if (!st->big) {
        d.pool = 1;
        st->wave = d.NS;
        d.arena_cap = pool_b;
        TRY(dalloc(st, &d.arena[0], d.arena_cap + 64));  // +64: word-window reads past a last block
        d.arena[1] = d.arena[0];
    } else {
        const uint64_t per_slot = 16 * d.L + 2 * d.slot_cap + 2 * d.nsub * sizeof(SideEntry);
        // up to four encoder slots per SM per wave: the hardware backfills
        // the SMs of all-zero strides (zero-stride pass) with the next
        // costly ones; at most an eighth of the free memory (C3: 592 slots)
        uint64_t w = d.NS < 2 ? 1 : std::min<uint64_t>(d.NS, 592);
        if (const char* e = getenv("QCS_WAVE_SLOTS")) w = std::max<uint64_t>(1, std::min<uint64_t>(d.NS, strtoull(e, nullptr, 10)));
        while (w > 2 && w * per_slot > std::max<uint64_t>(12ull << 30, free_b / 8)) w /= 2;
        w = std::max<uint64_t>(w, std::min<uint64_t>(d.NS, 2));  // a pair unit needs 2 slots
        if (w > 1 && (w & 1)) --w;  // whole pair units per wave
        st->wave = w;
        const uint64_t tables = 2 * d.NS * 64 + d.NS * 64;
        uint64_t reserve = 1ull << 30;  // left to the caller (QCS_RESERVE_BYTES)
        if (const char* e = getenv("QCS_RESERVE_BYTES")) reserve = strtoull(e, nullptr, 10);
        uint64_t cap = 0, min_cap = 1ull << 20;
        if (const char* e = getenv("QCS_ARENA_BYTES")) cap = strtoull(e, nullptr, 10), min_cap = 64;
        else if (free_b > side_b + w * per_slot + tables + reserve)
            // never more than a live state plus a full rewrite can use
            cap = std::min<uint64_t>(free_b - side_b - w * per_slot - tables - reserve, 2 * small_arena + (64ull << 20));
        cap &= ~uint64_t(15);
        if (cap < min_cap) {
            qcs_state_destroy(st);
            return set_err(QCS_E_NOMEM, "not enough device memory for a %d-qubit state with %d stride bits", n, s);
        }
        d.arena_cap = cap;
        TRY(dalloc(st, &d.arena[0], d.arena_cap + 64));  // +64: word-window reads past a last block
        d.arena[1] = nullptr;
        TRY(dalloc(st, &st->mv_src, 2 * d.NS));
        TRY(dalloc(st, &st->mv_dst, 2 * d.NS));
        TRY(dalloc(st, &st->mv_len, 2 * d.NS));
    }
    TRY(dalloc(st, &d.p_off, 2 * d.NS));
    TRY(dalloc(st, &d.p_len, 2 * d.NS));
    TRY(dalloc(st, &d.p_codec, 2 * d.NS));
    TRY(dalloc(st, &d.p_delta, 2 * d.NS));
    TRY(dalloc(st, &d.side, (d.pool ? 4 : 2) * d.NS * d.nsub));
    TRY(dalloc(st, &d.scale, d.NS));
    TRY(dalloc(st, &d.sum_sq, d.NS));
    TRY(dalloc(st, &d.X, 2 * st->wave * d.L));
    TRY(dalloc(st, &d.slot_out, d.pool ? 16 : 2 * st->wave * d.slot_cap));   // pool: unused
    TRY(dalloc(st, &d.slot_side, d.pool ? 1 : 2 * st->wave * d.nsub));
    TRY(dalloc(st, &d.slot_len, 2 * d.NS));
    TRY(dalloc(st, &d.slot_sum, d.NS));
    TRY(dalloc(st, &d.job_stride, d.NS));
    TRY(dalloc(st, &d.pending, d.NS));
    TRY(dalloc(st, &d.im_zero, d.NS));
    TRY(dalloc(st, &d.zero_slot, d.NS));
    TRY(dalloc(st, &d.redo, d.NS));
    TRY(dalloc(st, &d.committed, d.NS));
    TRY(dalloc(st, &d.p_cap, 2 * d.NS));
    TRY(dalloc(st, &d.p_capoff, 2 * d.NS));
    CU(cudaMemset(d.p_capoff, 0xff, 16 * d.NS));
    d.inplace = 1;
    if (const char* e = getenv("QCS_INPLACE")) d.inplace = atoi(e);
    TRY(dalloc(st, &d.order, d.NS));
    TRY(dalloc(st, &d.slot_of, d.NS));
    TRY(dalloc(st, &d.reports, d.NS));
    TRY(dalloc(st, &d.new_off, 2 * d.NS));
    TRY(dalloc(st, &d.partial, 2 * d.NS));
    TRY(dalloc(st, &d.sc, 1));
    TRY(dalloc(st, &d.counters, 24));
    if (const char* e = getenv("QCS_CTA_TRACE"))
        if (atoi(e)) TRY(dalloc(st, &st->cta_trace, 8 * d.NS));
    CU(cudaMemset(d.counters, 0, 192));
    TRY(dalloc(st, &st->lt.slot_codec, d.NS));
    TRY(dalloc(st, &st->lt.slot_delta, d.NS));
    if (cudaMallocHost(&st->h_sc, sizeof(Dev::Scal)) != cudaSuccess ||
        cudaMallocHost(&st->h_rep, sizeof(qcs_stride_report) * d.NS) != cudaSuccess) {
        qcs_state_destroy(st);
        return set_err(QCS_E_NOMEM, "pinned allocation failed");
    }
    cudaEventCreate(&st->ev_a);
    cudaEventCreate(&st->ev_b);
    // basis_state (aalc.cpp:140-174): one shared lossless all-zero block, plus
    // the hot stride's re block.  Payloads are tiny; build them here.
    auto varint = [](std::vector<uint8_t>& o, uint64_t v) {
        while (v >= 0x80) {
            o.push_back((uint8_t)v | 0x80);
            v >>= 7;
        }
        o.push_back((uint8_t)v);
    };
    std::vector<uint8_t> zero, hot;
    varint(zero, d.L << 1);
    const uint64_t off = basis & (d.L - 1);
    if (off) varint(hot, off << 1);
    varint(hot, (1ull << 1) | 1u);
    const double one = 1.0;
    uint64_t w;
    memcpy(&w, &one, 8);
    for (int i = 0; i < 8; ++i) hot.push_back((uint8_t)(w >> (8 * i)));
    if (d.L - off - 1) varint(hot, (d.L - off - 1) << 1);
    // arena image: the zero block at 0, the hot block at 16 (up to 27 bytes:
    // two varints of up to 9 bytes around the tag and the word), the bump
    // after it, 16-byte rounded
    const uint64_t img_bytes = 16 + round16(hot.size());
    std::vector<uint8_t> img(std::max<uint64_t>(img_bytes, 48), 0);
    memcpy(img.data(), zero.data(), zero.size());
    memcpy(img.data() + 16, hot.data(), hot.size());
    if (!d.pool) CU(cudaMemcpy(d.arena[0], img.data(), img_bytes, cudaMemcpyHostToDevice));
    std::vector<uint64_t> h_off(2 * d.NS, 0), h_len(2 * d.NS, zero.size());
    std::vector<int8_t> h_codec(2 * d.NS, 0);
    std::vector<double> h_delta(2 * d.NS, 0.0), h_scale(d.NS, 1.0), h_sum(d.NS, 0.0);
    if (!zero_state) {
        const uint64_t hj = basis >> s;
        h_off[2 * hj] = 16;
        h_len[2 * hj] = hot.size();
        h_sum[hj] = 1.0;
    }
    CU(cudaMemcpy(d.p_off, h_off.data(), 8 * h_off.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.p_len, h_len.data(), 8 * h_len.size(), cudaMemcpyHostToDevice));
    if (d.pool) {  // every plane owns its blocks: zero block, or the hot block
        uint4 z, h0, h1;
        memcpy(&z, img.data(), 16);
        memcpy(&h0, img.data() + 16, 16);
        memcpy(&h1, img.data() + 32, 16);
        const uint64_t hot_g = zero_state ? ~0ull : 2 * (basis >> s);
        k_init_pool<<<(unsigned)((2 * d.NS + 255) / 256), 256, 0, st->stream>>>(d, hot_g, z, (uint32_t)zero.size(), h0, h1,
                                                                               (uint32_t)hot.size());
        ++st->launches;
        CU(cudaGetLastError());
    }
    CU(cudaMemcpy(d.p_codec, h_codec.data(), h_codec.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.p_delta, h_delta.data(), 8 * h_delta.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.scale, h_scale.data(), 8 * h_scale.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.sum_sq, h_sum.data(), 8 * h_sum.size(), cudaMemcpyHostToDevice));
    Dev::Scal sc{};
    sc.bump = img_bytes;
    st->bump = img_bytes;
    sc.cur = 0;
    sc.err_gate = -1;
    sc.norm_sq = zero_state ? 0.0 : 1.0;
    CU(cudaMemcpy(d.sc, &sc, sizeof sc, cudaMemcpyHostToDevice));
    CU(cudaMemset(d.slot_of, 0xff, 8 * d.NS));
    k_index_planes<<<(unsigned)((2 * d.NS + 127) / 128), 128, 0, st->stream>>>(d, 0, 2 * d.NS);
    st->launches += 1;
    CU(cudaStreamSynchronize(st->stream));
    CU(cudaMemcpy(st->h_sc, d.sc, sizeof(Dev::Scal), cudaMemcpyDeviceToHost));
    if (st->h_sc->err) {
        const int e = st->h_sc->err;
        qcs_state_destroy(st);
        return set_err(e, "basis state indexing failed");
    }
    *out = st;
    return 0;
#undef TRY
}

static int sync_and_check(qcs_dev_state* st)
{
    CU(cudaStreamSynchronize(st->stream));
    prof_collect(st);
    CU(cudaMemcpy(st->h_sc, st->d.sc, sizeof(Dev::Scal), cudaMemcpyDeviceToHost));
    return 0;
}

static int report_device_error(qcs_dev_state* st)
{
    const int e = st->h_sc->err;
    const int gi = st->h_sc->err_gate;
    // clear so the (unchanged) state stays usable
    Dev::Scal sc = *st->h_sc;
    sc.err = 0;
    sc.err_gate = -1;
    cudaMemcpy(st->d.sc, &sc, sizeof sc, cudaMemcpyHostToDevice);
    if (e == QCS_E_NOMEM) return set_err(QCS_E_NOMEM, "gate %d failed: block arena exhausted", gi);
    return set_err(QCS_E_RUNTIME, "gate %d failed: device codec error %d", gi, e);
}

// Wave layout: a synchronisation found QCS_SUSPEND (the wave starting at
// *unit of gate *gate did not fit in the arena).  Compact the arena and clear
// the error word so the gate can be re-enqueued from that wave.  `prev_*` is
// the previous suspension point: suspending at the same point again right
// after a compaction means the live state itself does not fit — a true
// out-of-memory (the gate is part-applied if its first wave was committed).
static int handle_suspend(qcs_dev_state* st, int64_t* gate, uint64_t* unit, int64_t prev_gate, uint64_t prev_unit)
{
    *gate = st->h_sc->err_gate;
    *unit = st->h_sc->susp_unit;
    Dev::Scal sc = *st->h_sc;
    sc.err = 0;
    sc.err_gate = -1;
    sc.susp_unit = 0;
    sc.persist_susp = 0;
    CU(cudaMemcpy(st->d.sc, &sc, sizeof sc, cudaMemcpyHostToDevice));
    *st->h_sc = sc;
    if (*gate == prev_gate && *unit == prev_unit) {
        const uint64_t done = *unit & ~SUSP_PERSIST;  // waves' units, or strides of the persistent kernel
        if (done > 0) st->poisoned = true;
        return set_err(QCS_E_NOMEM, done ? "gate %lld failed: block arena exhausted after %llu of its units were committed"
                                         : "gate %lld failed: block arena exhausted",
                       (long long)*gate, (unsigned long long)done);
    }
    return compact_arena(st);
}

int qcs_apply_gate(qcs_dev_state_t st, const qcs_gate_desc* g, const double* lad, int nl,
                   double theta, qcs_stride_report* reports, uint64_t* n_reports,
                   double* norm_after)
{
    return qcs_apply_gate_ex(st, g, lad, nl, theta, 0, nullptr, reports, n_reports, norm_after);
}

int qcs_apply_gate_ex(qcs_dev_state_t st, const qcs_gate_desc* g, const double* lad, int nl,
                      double theta, int flags, const double* mean, qcs_stride_report* reports,
                      uint64_t* n_reports, double* norm_after)
{
    if (!st || !g) return set_err(QCS_E_INVALID, "null argument");
    if ((flags & QCS_GIVEN_MEAN) && !mean) return set_err(QCS_E_INVALID, "null mean");
    if (st->poisoned) return set_err(QCS_E_RUNTIME, "state unusable: an earlier gate failed part-way (wave layout)");
    int rc = validate_gate(st, g);
    if (rc) return rc;
    rc = validate_ladder(lad, nl, theta);
    if (rc) return rc;
    cudaSetDevice(st->device);
    uint64_t ns = 0;
    st->d.rec = nullptr;
    int64_t pg = -2;
    uint64_t pu = 0, unit = 0;
    for (;;) {
        rc = enqueue_gate(st, g, lad, nl, theta, -1, 0, &ns, (flags & QCS_NO_RENORM) ? 0 : 1,
                          (flags & QCS_GIVEN_MEAN) ? mean : nullptr, nullptr, 0, 0, unit, pg != -2);
        if (rc) return rc;
        rc = sync_and_check(st);
        if (rc) return rc;
        if (st->h_sc->err != QCS_SUSPEND) break;
        int64_t gi;
        rc = handle_suspend(st, &gi, &unit, pg, pu);
        if (rc) return rc;
        pg = gi, pu = unit;
    }
    if (st->h_sc->err) return report_device_error(st);
    if (reports && ns) {
        CU(cudaMemcpy(reports, st->d.reports, ns * sizeof(qcs_stride_report), cudaMemcpyDeviceToHost));
    }
    if (n_reports) *n_reports = ns;
    if (norm_after) *norm_after = std::sqrt(st->h_sc->norm_sq);
    return 0;
}

int qcs_run_program(qcs_dev_state_t st, const qcs_gate_desc* gates, uint64_t n_gates,
                    uint64_t first_index, const double* lad, int nl, double theta,
                    qcs_gate_record* records, uint64_t* n_done)
{
    if (!st || (!gates && n_gates)) return set_err(QCS_E_INVALID, "null argument");
    if (n_done) *n_done = 0;
    if (st->poisoned) return set_err(QCS_E_RUNTIME, "state unusable: an earlier gate failed part-way (wave layout)");
    int rc = validate_ladder(lad, nl, theta);
    if (rc) return rc;
    for (uint64_t i = 0; i < n_gates; ++i) {
        rc = validate_gate(st, &gates[i]);
        if (rc) {
            const std::string m = g_err;
            // the reference validates inside apply_gate, after earlier gates ran
            uint64_t done = 0;
            if (i) {
                int r2 = qcs_run_program(st, gates, i, first_index, lad, nl, theta, records, &done);
                if (r2) return r2;
            }
            if (n_done) *n_done = i;
            return set_err(rc, "gate %llu failed: %s", (unsigned long long)(first_index + i), m.c_str());
        }
    }
    cudaSetDevice(st->device);
    Dev& d = st->d;
    if (d.rec_cap < n_gates) {
        qcs_gate_record* r = nullptr;
        rc = dalloc(st, &r, std::max<uint64_t>(n_gates, 1));
        if (rc) return rc;
        d.rec = r;
        d.rec_cap = n_gates;
    }
    qcs_gate_record* rec = d.rec;
    std::vector<cudaEvent_t> ev(n_gates + 1);
    for (auto& e : ev) cudaEventCreate(&e);
    std::vector<double> el_ns(n_gates, 0.0);
    // Passes: gates [i0, n) are queued back to back with one synchronisation
    // at the end.  In the wave layout a pass can suspend inside gate k when the
    // arena is full (QCS_SUSPEND): the arena is compacted and the next pass
    // resumes gate k from the wave that did not fit (no host round trip per
    // wave otherwise).
    uint64_t i0 = 0, unit0 = 0, done = 0;
    int64_t pg = -2;
    uint64_t pu = 0;
    int rc2 = 0;
    std::string enq_err;
    for (;;) {
        uint64_t enq = i0;  // gates fully enqueued
        cudaEventRecord(ev[i0], st->stream);
        for (uint64_t i = i0; i < n_gates; ++i) {
            uint64_t ns;
            d.rec = rec;
            rc = enqueue_gate(st, &gates[i], lad, nl, theta, (int64_t)i, first_index + i, &ns, 1, nullptr, nullptr, 0, 0,
                              i == i0 ? unit0 : 0, i == i0 && pg >= 0);
            if (rc) break;
            cudaEventRecord(ev[i + 1], st->stream);
            enq = i + 1;
        }
        if (rc) enq_err = g_err;
        rc2 = sync_and_check(st);
        if (rc2) break;
        uint64_t ran = enq;  // gates whose kernels did their work in this pass
        const bool susp = st->h_sc->err == QCS_SUSPEND;
        if (st->h_sc->err) ran = std::min<uint64_t>(ran, (uint64_t)std::max<int64_t>(0, (int64_t)st->h_sc->err_gate - (int64_t)first_index) + (susp ? 1 : 0));
        for (uint64_t i = i0; i < ran; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            el_ns[i] += (double)ms * 1e6;
        }
        if (!susp || rc) {
            done = susp ? ran - 1 : ran;
            if (susp) {  // an enqueue error after a suspension: no resume
                if ((st->h_sc->susp_unit & ~SUSP_PERSIST) > 0) st->poisoned = true;
                Dev::Scal sc = *st->h_sc;
                sc.err = 0;
                sc.err_gate = -1;
                CU(cudaMemcpy(d.sc, &sc, sizeof sc, cudaMemcpyHostToDevice));
                *st->h_sc = sc;
            }
            break;
        }
        int64_t gk;
        uint64_t uk;
        // the compaction is part of the suspended gate's device time
        cudaEventRecord(ev[n_gates], st->stream);
        const auto h0 = std::chrono::steady_clock::now();
        rc2 = handle_suspend(st, &gk, &uk, pg, pu);
        const double comp_ns = (double)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - h0).count();
        if (rc2) {
            done = (uint64_t)(gk - (int64_t)first_index);
            break;
        }
        el_ns[(uint64_t)(gk - (int64_t)first_index)] += comp_ns;
        pg = gk, pu = uk;
        i0 = (uint64_t)(gk - (int64_t)first_index);
        unit0 = uk;
    }
    if (done) {
        std::vector<qcs_gate_record> h(done);
        cudaMemcpy(h.data(), rec, done * sizeof(qcs_gate_record), cudaMemcpyDeviceToHost);
        for (uint64_t i = 0; i < done; ++i) {
            h[i].elapsed_ns = (uint64_t)el_ns[i];
            if (records) records[i] = h[i];
        }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (n_done) *n_done = done;
    if (rc2) return rc2;
    if (st->h_sc->err) return report_device_error(st);
    if (rc) {
        g_err = enq_err;
        return rc;
    }
    return 0;
}

// compress_stride_adaptive (aalc.cpp:117-138) of caller-provided device planes
__global__ void k_snap_planes(double* x, uint64_t n)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        x[i] = snap(x[i]);
}

int qcs_load_strides_device(qcs_dev_state_t st, uint64_t first, uint64_t count, double* dev_planes,
                            const double* lad, int nl, double theta)
{
    if (!st || (!dev_planes && count)) return set_err(QCS_E_INVALID, "null argument");
    if (st->poisoned) return set_err(QCS_E_RUNTIME, "state unusable: an earlier gate failed part-way (wave layout)");
    if (first > st->d.NS || count > st->d.NS - first) return set_err(QCS_E_RANGE, "stride range out of range");
    int rc = validate_ladder(lad, nl, theta);
    if (rc) return rc;
    if (!count) return 0;
    cudaSetDevice(st->device);
    const uint64_t nel = count * 2 * st->d.L;
    k_snap_planes<<<(unsigned)grid_for(nel), 256, 0, st->stream>>>(dev_planes, nel);
    ++st->launches;
    uint64_t ns = 0;
    st->d.rec = nullptr;
    int64_t pg = -2;
    uint64_t pu = 0, unit = 0;
    for (;;) {
        rc = enqueue_gate(st, nullptr, lad, nl, theta, -1, 0, &ns, 0, nullptr, dev_planes, first, count, unit, pg != -2);
        if (rc) return rc;
        rc = sync_and_check(st);
        if (rc) return rc;
        if (st->h_sc->err != QCS_SUSPEND) break;
        int64_t gi;
        rc = handle_suspend(st, &gi, &unit, pg, pu);
        if (rc) return rc;
        pg = gi, pu = unit;
    }
    if (st->h_sc->err) return report_device_error(st);
    return 0;
}

int qcs_read_stride(qcs_dev_state_t st, uint64_t j, int apply_scale, double* re, double* im)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    if (j >= st->d.NS) return set_err(QCS_E_RANGE, "stride index out of range");
    cudaSetDevice(st->device);
    k_decode<<<1, 256, 0, st->stream>>>(st->d, DecodeJob{j, apply_scale, st->d.X});
    ++st->launches;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st->stream));
    const uint64_t L = st->d.L;
    if (re) CU(cudaMemcpy(re, st->d.X, L * 8, cudaMemcpyDeviceToHost));
    if (im) CU(cudaMemcpy(im, st->d.X + L, L * 8, cudaMemcpyDeviceToHost));
    return 0;
}

int qcs_read_strides_device(qcs_dev_state_t st, uint64_t first, uint64_t count, int apply_scale,
                            double* dev_out)
{
    if (!st || !dev_out) return set_err(QCS_E_INVALID, "null argument");
    if (first > st->d.NS || count > st->d.NS - first) return set_err(QCS_E_RANGE, "stride range out of range");
    cudaSetDevice(st->device);
    for (uint64_t j0 = first; j0 < first + count; j0 += 65535) {
        const uint64_t m = std::min<uint64_t>(65535, first + count - j0);
        k_decode<<<(unsigned)m, 256, 0, st->stream>>>(st->d, DecodeJob{j0, apply_scale, dev_out + (j0 - first) * 2 * st->d.L});
        ++st->launches;
    }
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st->stream));
    return 0;
}

int qcs_to_amplitudes(qcs_dev_state_t st, double* amps)
{
    if (!st || !amps) return set_err(QCS_E_INVALID, "null argument");
    cudaSetDevice(st->device);
    const uint64_t L = st->d.L, NS = st->d.NS;
    std::vector<double> buf(2 * L * st->wave);
    for (uint64_t j0 = 0; j0 < NS; j0 += st->wave) {
        const uint64_t m = std::min<uint64_t>(st->wave, NS - j0);
        k_decode<<<(unsigned)m, 256, 0, st->stream>>>(st->d, DecodeJob{j0, 1, st->d.X});
        ++st->launches;
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(buf.data(), st->d.X, 16 * L * m, cudaMemcpyDeviceToHost, st->stream));
        CU(cudaStreamSynchronize(st->stream));
        for (uint64_t q = 0; q < m; ++q) {
            const uint64_t j = j0 + q;
            for (uint64_t i = 0; i < L; ++i) {
                amps[2 * (j * L + i)] = buf[2 * L * q + i];
                amps[2 * (j * L + i) + 1] = buf[2 * L * q + L + i];
            }
        }
    }
    return 0;
}

int qcs_state_stats(qcs_dev_state_t st, uint64_t* bytes, double* min_ratio, double* norm_sq)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    cudaSetDevice(st->device);
    k_stats<<<1, 32, 0, st->stream>>>(st->d);
    ++st->launches;
    int rc = sync_and_check(st);
    if (rc) return rc;
    if (bytes) *bytes = st->h_sc->compressed_bytes;
    if (min_ratio) *min_ratio = st->h_sc->min_ratio;
    if (norm_sq) *norm_sq = st->h_sc->norm_sq;
    return 0;
}

int qcs_stride_info(qcs_dev_state_t st, uint64_t j, double* scale, double* ssq, uint64_t* rl,
                    uint64_t* il)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    if (j >= st->d.NS) return set_err(QCS_E_RANGE, "stride index out of range");
    cudaSetDevice(st->device);
    CU(cudaStreamSynchronize(st->stream));
    double a = 0, b = 0;
    uint64_t l[2];
    CU(cudaMemcpy(&a, st->d.scale + j, 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&b, st->d.sum_sq + j, 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(l, st->d.p_len + 2 * j, 16, cudaMemcpyDeviceToHost));
    if (scale) *scale = a;
    if (ssq) *ssq = b;
    if (rl) *rl = l[0];
    if (il) *il = l[1];
    return 0;
}

static void put_header(uint8_t* p, int codec, double delta, uint64_t count, uint64_t plen)
{
    p[0] = 'Q';
    p[1] = 'C';
    p[2] = 'S';
    p[3] = '1';
    p[4] = (uint8_t)codec;
    uint64_t w;
    memcpy(&w, &delta, 8);
    for (int i = 0; i < 8; ++i) p[5 + i] = (uint8_t)(w >> (8 * i));
    for (int i = 0; i < 8; ++i) p[13 + i] = (uint8_t)(count >> (8 * i));
    for (int i = 0; i < 8; ++i) p[21 + i] = (uint8_t)(plen >> (8 * i));
}

static uint64_t rd64(const uint8_t* p)
{
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

int qcs_export_blocks(qcs_dev_state_t st, uint64_t j, uint8_t* buf, uint64_t cap, uint64_t* len,
                      double* scale, double* ssq)
{
    if (!st || !len) return set_err(QCS_E_INVALID, "null argument");
    if (j >= st->d.NS) return set_err(QCS_E_RANGE, "stride index out of range");
    cudaSetDevice(st->device);
    CU(cudaStreamSynchronize(st->stream));
    uint64_t off[2], pl[2];
    int8_t codec[2];
    double delta[2];
    int cur = 0;
    CU(cudaMemcpy(off, st->d.p_off + 2 * j, 16, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(pl, st->d.p_len + 2 * j, 16, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(codec, st->d.p_codec + 2 * j, 2, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(delta, st->d.p_delta + 2 * j, 16, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&cur, &st->d.sc->cur, sizeof(int), cudaMemcpyDeviceToHost));
    *len = 2 * HEADER_BYTES + pl[0] + pl[1];
    if (scale) CU(cudaMemcpy(scale, st->d.scale + j, 8, cudaMemcpyDeviceToHost));
    if (ssq) CU(cudaMemcpy(ssq, st->d.sum_sq + j, 8, cudaMemcpyDeviceToHost));
    if (!buf) return 0;
    if (*len > cap) return set_err(QCS_E_CAPACITY, "output buffer too small");
    uint64_t o = 0;
    for (int c = 0; c < 2; ++c) {
        put_header(buf + o, codec[c], delta[c], st->d.L, pl[c]);
        o += HEADER_BYTES;
        if (pl[c]) CU(cudaMemcpy(buf + o, st->d.arena[cur] + off[c], pl[c], cudaMemcpyDeviceToHost));
        o += pl[c];
    }
    return 0;
}

int qcs_import_blocks(qcs_dev_state_t st, uint64_t j, const uint8_t* buf, uint64_t len,
                      double scale, double ssq)
{
    if (st) st->all_im_zero = false;  // arbitrary blocks: no longer known real
    if (!st || !buf) return set_err(QCS_E_INVALID, "null argument");
    if (j >= st->d.NS) return set_err(QCS_E_RANGE, "stride index out of range");
    cudaSetDevice(st->device);
    Dev& d = st->d;
    // parse_block (codec.cpp:391-420) for both planes
    uint64_t o = 0, poff[2], plen[2];
    int codec[2];
    double delta[2];
    for (int c = 0; c < 2; ++c) {
        if (o + HEADER_BYTES > len) return set_err(QCS_E_TRUNCATED, "block header extends past end of data");
        const uint8_t* p = buf + o;
        if (p[0] != 'Q' || p[1] != 'C' || p[2] != 'S' || p[3] != '1') return set_err(QCS_E_BAD_MAGIC, "bad block magic");
        codec[c] = p[4];
        if (codec[c] != 0 && codec[c] != 1) return set_err(QCS_E_UNKNOWN_CODEC, "unknown codec id %d", codec[c]);
        uint64_t w = rd64(p + 5);
        memcpy(&delta[c], &w, 8);
        const uint64_t count = rd64(p + 13);
        plen[c] = rd64(p + 21);
        o += HEADER_BYTES;
        if (o + plen[c] > len) return set_err(QCS_E_TRUNCATED, "block payload extends past end of data");
        if (count != d.L) return set_err(QCS_E_INVALID, "block length disagrees with geometry");
        poff[c] = o;
        o += plen[c];
    }
    CU(cudaStreamSynchronize(st->stream));
    CU(cudaMemcpy(st->h_sc, d.sc, sizeof(Dev::Scal), cudaMemcpyDeviceToHost));
    const uint64_t need = ((plen[0] + 15) & ~15ull) + ((plen[1] + 15) & ~15ull);
    uint64_t at = st->h_sc->bump;
    uint64_t pool_old[2] = {0, 0};
    if (d.pool) {
        CU(cudaMemcpy(pool_old, d.p_off + 2 * j, 16, cudaMemcpyDeviceToHost));
    } else if (st->big) {
        const int r = big_reserve(st, need, &at);
        if (r == QCS_E_NOMEM) return set_err(QCS_E_NOMEM, "block arena exhausted");
        if (r) return r;
    } else if (st->h_sc->bump + need > d.arena_cap) {
        return set_err(QCS_E_NOMEM, "block arena exhausted");
    }
    const int cur = st->h_sc->cur;
    uint64_t new_off[2];
    for (int c = 0; c < 2; ++c) {
        if (d.pool) {
            if (plen[c] > d.slot_cap) return set_err(QCS_E_BAD_VALUE, "block payload larger than any valid block");
            const uint64_t g = 2 * j + c;
            new_off[c] = (2 * g + 1 - ((pool_old[c] / d.slot_cap) & 1)) * d.slot_cap;
        } else {
            new_off[c] = at;
            at += (plen[c] + 15) & ~15ull;
        }
        if (plen[c]) CU(cudaMemcpy(d.arena[cur] + new_off[c], buf + poff[c], plen[c], cudaMemcpyHostToDevice));
    }
    // validate into a scratch side table first so a bad block leaves the state intact
    uint64_t old_off[2], old_len[2];
    int8_t old_codec[2];
    double old_delta[2];
    CU(cudaMemcpy(old_off, d.p_off + 2 * j, 16, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(old_len, d.p_len + 2 * j, 16, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(old_codec, d.p_codec + 2 * j, 2, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(old_delta, d.p_delta + 2 * j, 16, cudaMemcpyDeviceToHost));
    int8_t c8[2] = {(int8_t)codec[0], (int8_t)codec[1]};
    CU(cudaMemcpy(d.p_off + 2 * j, new_off, 16, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.p_len + 2 * j, plen, 16, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.p_codec + 2 * j, c8, 2, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.p_delta + 2 * j, delta, 16, cudaMemcpyHostToDevice));
    k_index_planes<<<1, 2, 0, st->stream>>>(d, 2 * j, 2);
    ++st->launches;
    int rc = sync_and_check(st);
    if (rc) return rc;
    if (st->h_sc->err) {
        const int e = st->h_sc->err;
        CU(cudaMemcpy(d.p_off + 2 * j, old_off, 16, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(d.p_len + 2 * j, old_len, 16, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(d.p_codec + 2 * j, old_codec, 2, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(d.p_delta + 2 * j, old_delta, 16, cudaMemcpyHostToDevice));
        k_index_planes<<<1, 2, 0, st->stream>>>(d, 2 * j, 2);
        Dev::Scal sc = *st->h_sc;
        sc.err = 0;
        CU(cudaMemcpy(d.sc, &sc, sizeof sc, cudaMemcpyHostToDevice));
        CU(cudaStreamSynchronize(st->stream));
        return set_err(e, "corrupt block for stride %llu", (unsigned long long)j);
    }
    Dev::Scal sc = *st->h_sc;
    sc.bump = st->big ? st->bump : at;
    CU(cudaMemcpy(d.sc, &sc, sizeof sc, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.scale + j, &scale, 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d.sum_sq + j, &ssq, 8, cudaMemcpyHostToDevice));
    return 0;
}

// ---------------------------------------------------------------------------
// stride images for sharded runs
// ---------------------------------------------------------------------------
struct PackEntry {
    uint64_t j;
    double scale, sum_sq;
    uint64_t len[2];
    uint64_t codec[2];
    double delta[2];
    uint64_t off[2];   // payload offsets in the image
    uint64_t soff;     // side index offset in the image (plane 0, then plane 1)
};
constexpr uint64_t PACK_MAGIC = 0x31504b5053434351ull;  // "QCSPKP1"
constexpr uint64_t PACK_HDR = 32;                      // magic, count, L, total

__global__ void __launch_bounds__(128) k_pack_copy(Dev d, uint8_t* img, const PackEntry* ent)
{
    const PackEntry& e = ent[blockIdx.x >> 1];
    const int c = (int)(blockIdx.x & 1);
    const uint64_t g = 2 * e.j + c;
    const uint4* s4 = reinterpret_cast<const uint4*>(d.arena[d.sc->cur] + d.p_off[g]);
    uint4* d4 = reinterpret_cast<uint4*>(img + e.off[c]);
    for (uint64_t i = threadIdx.x; i < (e.len[c] + 15) / 16; i += blockDim.x) d4[i] = s4[i];
    const SideEntry* ss = side_of(d, g);
    SideEntry* ds = reinterpret_cast<SideEntry*>(img + e.soff) + (uint64_t)c * d.nsub;
    for (uint64_t i = threadIdx.x; i < d.nsub; i += blockDim.x) ds[i] = ss[i];
}

// Stage image entries [i0, i0 + gridDim/2) into slots 0.. as if a gate had
// produced them, so the ordinary commit path installs them.
__global__ void __launch_bounds__(128) k_unpack_stage(Dev d, LevelTag lt, const uint8_t* img, const PackEntry* ent,
                                                      uint64_t i0, uint64_t xr, uint64_t gen)
{
    const uint64_t loc = blockIdx.x >> 1;
    const int c = (int)(blockIdx.x & 1);
    const PackEntry& e = ent[i0 + loc];
    const uint4* s4 = reinterpret_cast<const uint4*>(img + e.off[c]);
    uint8_t* dpay;
    SideEntry* ds;
    if (d.pool) {  // straight into the plane's other slot; k_pool_commit flips
        const uint64_t g = 2 * (e.j ^ xr) + c;
        const int other = 1 - pool_sel(d, g);
        dpay = d.arena[0] + (2 * g + other) * d.slot_cap;
        ds = d.side + (2 * g + other) * d.nsub;
    } else {
        dpay = d.slot_out + (2 * loc + c) * d.slot_cap;
        ds = d.slot_side + (2 * loc + c) * d.nsub;
    }
    uint4* d4 = reinterpret_cast<uint4*>(dpay);
    for (uint64_t i = threadIdx.x; i < (e.len[c] + 15) / 16; i += blockDim.x) d4[i] = s4[i];
    const SideEntry* ss = reinterpret_cast<const SideEntry*>(img + e.soff) + (uint64_t)c * d.nsub;
    for (uint64_t i = threadIdx.x; i < d.nsub; i += blockDim.x) ds[i] = ss[i];
    if (threadIdx.x == 0) {
        const uint64_t j = e.j ^ xr;
        d.slot_len[2 * loc + c] = e.len[c];
        if (c == 0) {
            d.job_stride[loc] = j;
            d.slot_sum[loc] = e.sum_sq;
            lt.slot_codec[loc] = (int8_t)e.codec[0];
            lt.slot_delta[loc] = e.delta[0];
            d.slot_of[j] = (int64_t)((gen << 32) | loc);
        }
    }
}

__global__ void k_unpack_finish(Dev d, const PackEntry* ent, uint64_t i0, uint64_t m, uint64_t xr)
{
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i == 0 && d.sc->mode == 1) {  // the small layout compacted into the other arena
        d.sc->cur = 1 - d.sc->cur;
        d.sc->mode = 0;
    }
    if (i >= m) return;
    const PackEntry& e = ent[i0 + i];
    const uint64_t j = e.j ^ xr;
    d.scale[j] = e.scale;
    // the im plane may use another codec than re (k_unpack_stage tagged re's)
    d.p_codec[2 * j + 1] = (int8_t)e.codec[1];
    d.p_delta[2 * j + 1] = e.delta[1];
}

int qcs_pack_strides(qcs_dev_state_t st, int bit, int value, void* dev_buf, uint64_t cap, uint64_t* len)
{
    return qcs_pack_strides_range(st, bit, value, 0, UINT64_MAX, dev_buf, cap, len);
}

int qcs_pack_strides_range(qcs_dev_state_t st, int bit, int value, uint64_t first, uint64_t count, void* dev_buf,
                           uint64_t cap, uint64_t* len)
{
    if (!st || !len) return set_err(QCS_E_INVALID, "null argument");
    Dev& d = st->d;
    if (bit < 0 || (bit < 63 && (1ull << bit) >= d.NS)) return set_err(QCS_E_RANGE, "stride bit out of range");
    cudaSetDevice(st->device);
    int rc = sync_and_check(st);
    if (rc) return rc;
    const uint64_t np = 2 * d.NS;
    std::vector<uint64_t> plen(np);
    std::vector<int8_t> pc(np);
    std::vector<double> pd(np), sc(d.NS), ss(d.NS);
    CU(cudaMemcpy(plen.data(), d.p_len, 8 * np, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(pc.data(), d.p_codec, np, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(pd.data(), d.p_delta, 8 * np, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(sc.data(), d.scale, 8 * d.NS, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(ss.data(), d.sum_sq, 8 * d.NS, cudaMemcpyDeviceToHost));
    std::vector<PackEntry> ent;
    uint64_t rank_in_set = 0;  // position among the strides with bit == value
    for (uint64_t j = 0; j < d.NS; ++j)
        if ((int)((j >> bit) & 1) == (value ? 1 : 0)) {
            const uint64_t r = rank_in_set++;
            if (r < first || r - first >= count) continue;
            PackEntry e{};
            e.j = j;
            e.scale = sc[j];
            e.sum_sq = ss[j];
            for (int c = 0; c < 2; ++c) {
                e.len[c] = plen[2 * j + c];
                e.codec[c] = (uint64_t)pc[2 * j + c];
                e.delta[c] = pd[2 * j + c];
            }
            ent.push_back(e);
        }
    uint64_t at = round16(PACK_HDR + sizeof(PackEntry) * ent.size());
    const uint64_t side_b = 2 * d.nsub * sizeof(SideEntry);
    for (auto& e : ent) {
        e.off[0] = at;
        at += round16(e.len[0]);
        e.off[1] = at;
        at += round16(e.len[1]);
        e.soff = at;
        at += side_b;
    }
    *len = at;
    if (!dev_buf) return 0;
    if (at > cap) return set_err(QCS_E_CAPACITY, "image buffer too small");
    std::vector<uint8_t> hdr(PACK_HDR + sizeof(PackEntry) * ent.size());
    const uint64_t h4[4] = {PACK_MAGIC, (uint64_t)ent.size(), d.L, at};
    memcpy(hdr.data(), h4, PACK_HDR);
    if (!ent.empty()) memcpy(hdr.data() + PACK_HDR, ent.data(), sizeof(PackEntry) * ent.size());
    uint8_t* img = static_cast<uint8_t*>(dev_buf);
    CU(cudaMemcpyAsync(img, hdr.data(), hdr.size(), cudaMemcpyHostToDevice, st->stream));
    if (!ent.empty()) {
        k_pack_copy<<<(unsigned)(2 * ent.size()), 128, 0, st->stream>>>(d, img, reinterpret_cast<const PackEntry*>(img + PACK_HDR));
        ++st->launches;
    }
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st->stream));
    return 0;
}

int qcs_unpack_strides(qcs_dev_state_t st, const void* dev_buf, uint64_t len, uint64_t xor_mask)
{
    if (st) st->all_im_zero = false;  // images from another shard: no longer known real
    if (!st || !dev_buf) return set_err(QCS_E_INVALID, "null argument");
    Dev& d = st->d;
    cudaSetDevice(st->device);
    int rc = sync_and_check(st);
    if (rc) return rc;
    if (len < PACK_HDR) return set_err(QCS_E_TRUNCATED, "stride image truncated");
    const uint8_t* img = static_cast<const uint8_t*>(dev_buf);
    uint64_t h4[4];
    CU(cudaMemcpy(h4, img, PACK_HDR, cudaMemcpyDeviceToHost));
    if (h4[0] != PACK_MAGIC) return set_err(QCS_E_BAD_MAGIC, "bad stride image magic");
    if (h4[2] != d.L) return set_err(QCS_E_INVALID, "stride image length disagrees with geometry");
    const uint64_t count = h4[1];
    if (count > d.NS || h4[3] > len || PACK_HDR + sizeof(PackEntry) * count > len)
        return set_err(QCS_E_TRUNCATED, "stride image truncated");
    std::vector<PackEntry> ent(count);
    if (count) CU(cudaMemcpy(ent.data(), img + PACK_HDR, sizeof(PackEntry) * count, cudaMemcpyDeviceToHost));
    for (const auto& e : ent) {
        if ((e.j ^ xor_mask) >= d.NS) return set_err(QCS_E_RANGE, "stride index out of range");
        for (int c = 0; c < 2; ++c)
            if (e.len[c] > d.slot_cap || e.off[c] + e.len[c] > len || e.codec[c] > 1)
                return set_err(QCS_E_BAD_VALUE, "corrupt stride image entry");
    }
    const PackEntry* dent = reinterpret_cast<const PackEntry*>(img + PACK_HDR);
    for (uint64_t i0 = 0; i0 < count; i0 += st->wave) {
        const uint64_t m = std::min<uint64_t>(st->wave, count - i0);
        const uint64_t gen = ++st->gen;
        k_unpack_stage<<<(unsigned)(2 * m), 128, 0, st->stream>>>(d, st->lt, img, dent, i0, xor_mask, gen);
        ++st->launches;
        if (st->big) {
            rc = big_commit_wave(st, 0, m, 0, i0);
            if (rc < 0) return report_device_error(st);
            if (rc) return rc;
        } else {
            k_make_jobs_reset_cin<<<1, 1, 0, st->stream>>>(d);
            k_pool_commit<<<(unsigned)((2 * m + 255) / 256), 256, 0, st->stream>>>(d, st->lt, m);
            st->launches += 2;
        }
        k_unpack_finish<<<(unsigned)((m + 127) / 128), 128, 0, st->stream>>>(d, dent, i0, m, xor_mask);
        ++st->launches;
        CU(cudaGetLastError());
        rc = sync_and_check(st);
        if (rc) return rc;
        if (st->h_sc->err) return report_device_error(st);
    }
    return 0;
}

__global__ void k_scale_all(double* scale, uint64_t ns, double f)
{
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j < ns) scale[j] = __dmul_rn(scale[j], f);
}

int qcs_stride_norms(qcs_dev_state_t st, double* scales, double* sums)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    cudaSetDevice(st->device);
    CU(cudaStreamSynchronize(st->stream));
    if (scales) CU(cudaMemcpy(scales, st->d.scale, 8 * st->d.NS, cudaMemcpyDeviceToHost));
    if (sums) CU(cudaMemcpy(sums, st->d.sum_sq, 8 * st->d.NS, cudaMemcpyDeviceToHost));
    return 0;
}

int qcs_stride_sums(qcs_dev_state_t st, double* partial)
{
    if (!st || !partial) return set_err(QCS_E_INVALID, "null argument");
    cudaSetDevice(st->device);
    int rc = sync_and_check(st);
    if (rc) return rc;
    Dev& d = st->d;
    k_stride_partial<<<(unsigned)d.NS, 128, 0, st->stream>>>(d);
    st->launches += 1;
    CU(cudaGetLastError());
    rc = sync_and_check(st);
    if (rc) return rc;
    if (st->h_sc->err) return report_device_error(st);
    CU(cudaMemcpy(partial, d.partial, 16 * d.NS, cudaMemcpyDeviceToHost));
    return 0;
}

int qcs_scale_all(qcs_dev_state_t st, double f)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    cudaSetDevice(st->device);
    k_scale_all<<<(unsigned)((st->d.NS + 255) / 256), 256, 0, st->stream>>>(st->d.scale, st->d.NS, f);
    ++st->launches;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st->stream));
    return 0;
}

int qcs_state_memory(qcs_dev_state_t st, uint64_t* arena, uint64_t* side, uint64_t* scratch)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    int rc = sync_and_check(st);
    if (rc) return rc;
    const Dev& d = st->d;
    if (arena) *arena = st->h_sc->bump;
    if (side) *side = 2 * d.NS * d.nsub * sizeof(SideEntry);
    if (scratch) *scratch = 16 * st->wave * d.L + 2 * st->wave * d.slot_cap + 2 * st->wave * d.nsub * sizeof(SideEntry);
    return 0;
}

uint64_t qcs_state_launches(qcs_dev_state_t st) { return st ? st->launches : 0; }

int qcs_state_profile(qcs_dev_state_t st, int enable)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    int rc = sync_and_check(st);
    if (rc) return rc;
    st->prof = enable == 2 ? 2 : (enable != 0 ? 1 : 0);
    st->prof_open = false;
    for (int i = 0; i < 6; ++i) {
        st->cls_ns[i] = 0;
        st->cls_n[i] = 0;
    }
    return 0;
}

int qcs_state_counters(qcs_dev_state_t st, uint64_t* out, int n)
{
    if (!st || !out || n < 0 || n > 24) return set_err(QCS_E_INVALID, "bad argument");
    int rc = sync_and_check(st);
    if (rc) return rc;
    CU(cudaMemcpy(out, st->d.counters, 8 * n, cudaMemcpyDeviceToHost));
    if (n > 4) out[4] = st->compactions;  // host-side: in-place arena compactions
    if (n > 5) out[5] = st->big ? st->wave : 0;
    if (n > 14) out[14] = (uint64_t)st->compact_ns;  // (replaces the unused 'tail' phase slot)
    return 0;
}

int qcs_state_kernel_time(qcs_dev_state_t st, int cls, double* total_ns, uint64_t* launches)
{
    if (!st) return set_err(QCS_E_INVALID, "null state");
    if (cls < 0 || cls >= 6) return set_err(QCS_E_RANGE, "kernel class out of range");
    int rc = sync_and_check(st);
    if (rc) return rc;
    if (total_ns) *total_ns = st->cls_ns[cls];
    if (launches) *launches = st->cls_n[cls];
    return 0;
}

namespace {
int codec_serial_chain()
{
    const char* e = getenv("QCS_SERIAL_CHAIN");
    return e ? atoi(e) : 1;
}
}  // namespace

int qcs_codec_compress(const double* x, uint64_t n, double delta, uint8_t* out, uint64_t cap,
                       uint64_t* len)
{
    if (!len || (!x && n)) return set_err(QCS_E_INVALID, "null argument");
    if (!(delta >= 0.0) || !std::isfinite(delta)) return set_err(QCS_E_INVALID, "error bound must be finite and >= 0");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(QCS_E_CUDA, "no CUDA device available (the codec has no CPU path)");
    }
    for (uint64_t i = 0; i < n; ++i)  // require_finite (codec.cpp:83-91): input argument check
        if (!std::isfinite(x[i])) return set_err(QCS_E_BAD_VALUE, "NaN/Inf cannot be compressed");
    const uint64_t nsub = (n + SUB - 1) / SUB;
    const uint64_t pcap = payload_cap(n);
    double* dx = nullptr;
    uint8_t* dout = nullptr;
    SideEntry* dside = nullptr;
    uint64_t* dlen = nullptr;
    cudaStream_t s = nullptr;
    auto cleanup = [&]() {
        cudaFree(dx);
        cudaFree(dout);
        cudaFree(dside);
        cudaFree(dlen);
        if (s) cudaStreamDestroy(s);
    };
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&dx, std::max<uint64_t>(8 * n, 16)) != cudaSuccess ||
        cudaMalloc(&dout, 2 * pcap) != cudaSuccess ||
        cudaMalloc(&dside, std::max<uint64_t>(2 * nsub, 1) * sizeof(SideEntry)) != cudaSuccess ||
        cudaMalloc(&dlen, 16) != cudaSuccess) {
        cleanup();
        return set_err(QCS_E_NOMEM, "device allocation failed");
    }
    cudaMemcpyAsync(dx, x, 8 * n, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(dlen, 0, 16, s);
    FusedArgs a{};
    a.max_rounds = codec_max_rounds();
    a.X = dx;
    a.x_plane_stride = n;
    a.n = n;
    a.pending = nullptr;
    a.snap = 0;
    a.out = dout;
    a.cap = pcap;
    a.side = dside;
    a.nsub = nsub;
    a.out_len = dlen;
    a.sumsq = nullptr;
    a.cp = make_params(delta);
    int16_t* dcodes = nullptr;
    double* dpreds = nullptr;
    int rc = 0;
    if (n && a.cp.lossy && !a.cp.pow2 && codec_serial_chain()) {  // serial-chain mode
        if (cudaMalloc(&dcodes, 2 * n + 16) != cudaSuccess || cudaMalloc(&dpreds, 8 * nsub + 16) != cudaSuccess) {
            cudaGetLastError();
            rc = set_err(QCS_E_NOMEM, "device allocation failed");
        } else {
            ChainLevels chl{};
            chl.n = 1;
            chl.delta[0] = delta;
            chl.td[0] = a.cp.td;
            chl.inv[0] = 1.0 / a.cp.td;
            chl.lim[0] = a.cp.lim;
            k_serial_chain<<<1, 128, 0, s>>>(dx, 1, n, nsub, chl, dcodes, dpreds, nullptr, 0, nullptr, nullptr);
            a.pre_codes = dcodes;
            a.pre_pred = dpreds;
        }
    }
    if (!rc && n) rc = launch_fused(a, FM_RAW1, 1, s);
    uint64_t plen = 0;
    if (!rc) {
        cudaMemcpyAsync(&plen, dlen, 8, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) rc = set_err(QCS_E_CUDA, "codec kernel failed");
    }
    if (!rc) {
        *len = HEADER_BYTES + plen;
        if (out) {
            if (*len > cap) {
                rc = set_err(QCS_E_CAPACITY, "output buffer too small");
            } else {
                put_header(out, a.cp.lossy ? 1 : 0, delta, n, plen);
                if (plen && cudaMemcpy(out + HEADER_BYTES, dout, plen, cudaMemcpyDeviceToHost) != cudaSuccess)
                    rc = set_err(QCS_E_CUDA, "copy failed");
            }
        }
    }
    cudaFree(dcodes);
    cudaFree(dpreds);
    cleanup();
    return rc;
}

int qcs_codec_decompress(const uint8_t* blk, uint64_t len, double* out, uint64_t n)
{
    if (!blk || (!out && n)) return set_err(QCS_E_INVALID, "null argument");
    // parse_block (codec.cpp:391-420)
    if (len < HEADER_BYTES) return set_err(QCS_E_TRUNCATED, "block header extends past end of data");
    if (blk[0] != 'Q' || blk[1] != 'C' || blk[2] != 'S' || blk[3] != '1') return set_err(QCS_E_BAD_MAGIC, "bad block magic");
    const int codec = blk[4];
    if (codec != 0 && codec != 1) return set_err(QCS_E_UNKNOWN_CODEC, "unknown codec id %d", codec);
    double delta;
    uint64_t w = rd64(blk + 5);
    memcpy(&delta, &w, 8);
    const uint64_t count = rd64(blk + 13), plen = rd64(blk + 21);
    if (HEADER_BYTES + plen > len) return set_err(QCS_E_TRUNCATED, "block payload extends past end of data");
    if (count != n) return set_err(QCS_E_INVALID, "output span does not match scalar count");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(QCS_E_CUDA, "no CUDA device available (the codec has no CPU path)");
    }
    uint8_t* din = nullptr;
    double* dout = nullptr;
    int* derr = nullptr;
    auto cleanup = [&]() {
        cudaFree(din);
        cudaFree(dout);
        cudaFree(derr);
    };
    if (cudaMalloc(&din, std::max<uint64_t>(plen, 16)) != cudaSuccess ||
        cudaMalloc(&dout, std::max<uint64_t>(8 * n, 16)) != cudaSuccess || cudaMalloc(&derr, 4) != cudaSuccess) {
        cleanup();
        return set_err(QCS_E_NOMEM, "device allocation failed");
    }
    int herr = 0;
    if (plen) cudaMemcpy(din, blk + HEADER_BYTES, plen, cudaMemcpyHostToDevice);
    k_decode_payload<<<1, 1>>>(din, plen, codec, delta, n, dout, derr);
    cudaError_t e = cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        cleanup();
        return set_err(QCS_E_CUDA, "decode kernel failed: %s", cudaGetErrorString(e));
    }
    if (herr) {
        cleanup();
        return set_err(herr, herr == QCS_E_TRUNCATED ? "payload truncated" : "malformed payload");
    }
    if (n) cudaMemcpy(out, dout, 8 * n, cudaMemcpyDeviceToHost);
    cleanup();
    return 0;
}


// Test hook: lossless-encode a (re, im) stride pair and return the stored
// sum of squares the engine would record (StrideBuffer::sum_sq, core.cpp:30-37).
// Test/diagnostic hook (not in the public header): per-slot phase cycles of
// the last encoder launch when QCS_CTA_TRACE=1.
int qcs_debug_cta_trace(qcs_dev_state_t st, uint64_t* out, uint64_t n_slots)
{
    if (!st || !st->cta_trace) return set_err(QCS_E_INVALID, "trace off");
    CU(cudaStreamSynchronize(st->stream));
    CU(cudaMemcpy(out, st->cta_trace, 8 * 8 * std::min<uint64_t>(n_slots, st->d.NS), cudaMemcpyDeviceToHost));
    return 0;
}

// Diagnostic hook: the split path's uncompressed encoder input of a slot.
int qcs_debug_read_x(qcs_dev_state_t st, uint64_t slot, double* out)
{
    if (!st || slot >= st->wave) return set_err(QCS_E_INVALID, "bad slot");
    CU(cudaStreamSynchronize(st->stream));
    CU(cudaMemcpy(out, st->d.X + 2 * slot * st->d.L, 16 * st->d.L, cudaMemcpyDeviceToHost));
    return 0;
}

int qcs_debug_stride_sumsq(const double* re, const double* im, uint64_t n, double* out)
{
    const uint64_t nsub = (n + SUB - 1) / SUB, pcap = payload_cap(n);
    double *dx = nullptr, *dsum = nullptr;
    uint8_t* dout = nullptr;
    SideEntry* dside = nullptr;
    uint64_t* dlen = nullptr;
    int rc = 0;
    if (cudaMalloc(&dx, 16 * n + 16) != cudaSuccess || cudaMalloc(&dsum, 8) != cudaSuccess ||
        cudaMalloc(&dout, 2 * pcap) != cudaSuccess || cudaMalloc(&dside, 2 * nsub * sizeof(SideEntry) + 16) != cudaSuccess ||
        cudaMalloc(&dlen, 16) != cudaSuccess) {
        rc = set_err(QCS_E_NOMEM, "device allocation failed");
    } else {
        cudaMemcpy(dx, re, 8 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dx + n, im, 8 * n, cudaMemcpyHostToDevice);
        FusedArgs a{};
        a.max_rounds = codec_max_rounds();
        a.X = dx; a.x_plane_stride = n; a.n = n; a.snap = 0; a.out = dout; a.cap = pcap;
        a.side = dside; a.nsub = nsub; a.out_len = dlen; a.sumsq = dsum; a.cp = make_params(0.0);
        rc = launch_fused(a, FM_RAW2, 1, 0);
        if (!rc && cudaMemcpy(out, dsum, 8, cudaMemcpyDeviceToHost) != cudaSuccess) rc = set_err(QCS_E_CUDA, "copy failed");
    }
    cudaFree(dx); cudaFree(dsum); cudaFree(dout); cudaFree(dside); cudaFree(dlen);
    return rc;
}

}  // extern "C"

#include "qcs_cluster.cuh"
