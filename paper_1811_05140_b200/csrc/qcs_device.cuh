// Device-side building blocks shared by the codec and gate kernels.
//
// Arithmetic contract: every parity-relevant FP64 operation is written with
// the explicit round-to-nearest intrinsics in the reference's left-to-right
// order and the whole library is compiled with -fmad=false, so no DFMA is
// ever formed (checked with cuobjdump -sass in DESIGN.md §6).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace qcs {

constexpr int SUB = 32;                         // elements per lane sub-chunk
constexpr int PLANE_LANES = 128;                // lanes per plane in the codec CTA
constexpr int ITER = PLANE_LANES * SUB;         // elements per plane per CTA iteration
constexpr int CODEC_THREADS = 2 * PLANE_LANES;  // one CTA = one stride (re + im planes)
constexpr int XS_STRIDE = SUB + 1;              // padded lane pitch in shared memory
constexpr int QRADIUS = 32768;                  // codec.cpp:11
constexpr int32_t WCODE = INT32_MIN;            // element stored as a raw word
constexpr double ZERO_SNAP = 1e-300;            // core.hpp:22
constexpr uint32_t HEADER_BYTES = 29;           // codec.hpp:54

enum : int { TY_NONE = 0, TY_Z = 1, TY_C = 2, TY_W = 3 };

// Side index entry: one per SUB-element sub-chunk of a plane.  Lets any
// sub-chunk be decoded on its own, bit-exactly: byte offset (within the
// payload) of the token covering the sub-chunk's first element, how many of
// that token's elements precede the sub-chunk, and the exact predictor value
// entering it (the reference decoder's `pred`, codec.cpp:296).
struct SideEntry {
    uint32_t off;
    uint32_t skip;
    double pred;
};

// Parameters of one error-bound level (ErrorBound, codec.hpp:24-32).
struct CodecParams {
    double delta;    // absolute bound; 0 = lossless
    double td;       // 2*delta (codec.cpp:219)
    double inv_td;   // 1/td, used only when td is a power of two (exact)
    double lim;      // td * 32768 (codec.cpp:220)
    int lossy;
    int pow2;
};

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) with mbarrier completion ----
// One thread arms the CTA-local mbarrier with the byte count and issues the
// copy; every consumer waits on the barrier's phase parity.  Sizes and both
// addresses must be multiples of 16 bytes.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// global -> shared bulk copy of `bytes` (issuing thread only).  The fence
// orders this thread's (and, after a barrier, the CTA's) earlier generic
// accesses to dst before the async-proxy write.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}

#ifdef QCS_WATCHDOG
#include <cstdio>
#define QCS_WD(cond, what)                                                                                  \
    do {                                                                                                    \
        if (cond) {                                                                                         \
            printf("[qcs watchdog] %s block %d thread %d\n", what, (int)blockIdx.x, (int)threadIdx.x);     \
            __trap();                                                                                       \
        }                                                                                                   \
    } while (0)
#else
#define QCS_WD(cond, what) \
    do {                   \
    } while (0)
#endif

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
#ifdef QCS_WATCHDOG
    unsigned long long spins = 0;
#endif
    while (!done) {
#ifdef QCS_WATCHDOG
        QCS_WD(++spins > (1ull << 28), "mbar_wait");
#endif
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(b), "r"(parity)
            : "memory");
    }
}

__host__ __device__ inline uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__host__ __device__ inline int type_of(int32_t c)
{
    return c == 0 ? TY_Z : (c == WCODE ? TY_W : TY_C);
}

__device__ __forceinline__ int varint_len(uint64_t v)
{
    const int bits = 64 - __clzll(v | 1ull);
    return (bits + 6) / 7;
}

__device__ __forceinline__ uint64_t zigzag(int64_t q)
{
    return (static_cast<uint64_t>(q) << 1) ^ static_cast<uint64_t>(q >> 63);
}

__device__ __forceinline__ int64_t unzigzag(uint64_t z)
{
    return static_cast<int64_t>(z >> 1) ^ -static_cast<int64_t>(z & 1);
}

// Token value of a run of `len` elements of type ty (Z or W) for the codec.
// Lossless: len<<1 | (W ? 1 : 0)  (codec.cpp:13-15).
// Lossy:    len<<2 | (W ? 2 : 0)  (codec.cpp:17-20).
__device__ __forceinline__ uint64_t run_token(int lossy, int ty, uint64_t len)
{
    if (lossy) return (len << 2) | (ty == TY_W ? 2u : 0u);
    return (len << 1) | (ty == TY_W ? 1u : 0u);
}

__device__ __forceinline__ uint64_t code_token(int32_t q)
{
    return (zigzag(q) << 2) | 1u;
}

__device__ __forceinline__ void put_varint(uint8_t* p, uint64_t v)
{
    while (v >= 0x80) {
        *p++ = static_cast<uint8_t>(v) | 0x80;
        v >>= 7;
    }
    *p = static_cast<uint8_t>(v);
}

__device__ __forceinline__ void put_word(uint8_t* p, uint64_t w)
{
    if ((reinterpret_cast<uintptr_t>(p) & 7u) == 0) {  // aligned: one 8-byte store
        *reinterpret_cast<uint64_t*>(p) = w;
        return;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = static_cast<uint8_t>(w >> (8 * i));
}

__device__ __forceinline__ uint64_t get_word(const uint8_t* p)
{
    uint64_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= static_cast<uint64_t>(p[i]) << (8 * i);
    return w;
}

// Trusted varint read (internal blocks, already validated).
__device__ __forceinline__ uint64_t get_varint(const uint8_t* in, uint64_t& pos)
{
    uint64_t v = 0;
    int shift = 0;
    for (;;) {
        const uint8_t b = in[pos++];
        v |= static_cast<uint64_t>(b & 0x7f) << (shift & 63);
        if (!(b & 0x80)) return v;
        shift += 7;
    }
}

__device__ __forceinline__ double snap(double x)
{
    return fabs(x) < ZERO_SNAP ? 0.0 : x;  // StrideBuffer::snap_zeros, core.cpp:39-47
}

// One step of the reference lossy encoder (compress_lossy, codec.cpp:224-247)
// from predictor P on input x.  Returns the code (0 = zero code, WCODE =
// escape) and advances P exactly as the reference does.
__device__ __forceinline__ int32_t ref_step(const CodecParams& cp, double& P, double x)
{
    const double diff = __dsub_rn(x, P);
    if (fabs(diff) < cp.lim) {
        const double qd = cp.pow2 ? __dmul_rn(diff, cp.inv_td) : __ddiv_rn(diff, cp.td);
        // llround: nearest, halfway away from zero.  trunc/sub are exact.
        double t = trunc(qd);
        if (fabs(__dsub_rn(qd, t)) >= 0.5) t = __dadd_rn(t, copysign(1.0, qd));
        if (t > -32768.0 && t < 32768.0) {
            const double recon = __dadd_rn(P, __dmul_rn(cp.td, t));
            if (fabs(__dsub_rn(x, recon)) <= cp.delta) {
                P = recon;
                return static_cast<int32_t>(t);
            }
        }
    }
    P = x;
    return WCODE;
}

// The predictor value the reference would hold after coding x when the chain
// sits on the 2*delta lattice anchored at 0: used only as a *guess* for a
// lane's entry predictor; every guess is verified.
__device__ __forceinline__ double lattice_guess(const CodecParams& cp, double xprev2, double xprev1)
{
    double t = cp.pow2 ? __dmul_rn(xprev2, cp.inv_td) : __ddiv_rn(xprev2, cp.td);
    t = rint(t);
    double P = __dmul_rn(cp.td, t);
    ref_step(cp, P, xprev1);
    return P;
}

// Guess for the predictor entering a lane when the chain is anchored at `a`
// (the last escape before the lane, or any exact predictor on the same
// lattice): the lattice point a + 2*delta*M nearest to x2, then one exact
// reference step onto x1.  Only a guess; verified bit-for-bit.
__device__ __forceinline__ double anchored_guess(const CodecParams& cp, double a, double x2, double x1)
{
    const double d = __dsub_rn(x2, a);
    const double M = rint(cp.pow2 ? __dmul_rn(d, cp.inv_td) : __ddiv_rn(d, cp.td));
    double P = __dadd_rn(a, __dmul_rn(cp.td, M));
    ref_step(cp, P, x1);
    return P;
}

// Point of the lattice a + 2*delta*Z nearest x (power-of-two delta).
__device__ __forceinline__ double lattice_point(const CodecParams& cp, double a, double x)
{
    const double M = rint(__dmul_rn(__dsub_rn(x, a), cp.inv_td));
    return __dadd_rn(a, __dmul_rn(cp.td, M));
}

// lattice_point with rounding emulation: if a + 2*delta*M is not exact the
// reference chain rounds right here, and the rounded value anchors what
// follows (a heuristic for the speculation; verification decides).
// v = fl(a + y) is exact iff fl(v - a) == y and fl(v - y) == a: if the add
// rounded, its error e is a non-zero multiple of u = min(ulp a, ulp y) (the
// result then has ulp >= u), so |e| >= u and e cannot vanish in both
// re-subtractions, each of which would need |e| <= ulp/2.  Branch-free, and
// the two subtractions are independent.
__device__ __forceinline__ bool add_exact(double a, double y, double v)
{
    return (__dsub_rn(v, a) == y) & (__dsub_rn(v, y) == a);
}

__device__ __forceinline__ double lattice_step(const CodecParams& cp, double& a, double x)
{
    const double M = rint(__dmul_rn(__dsub_rn(x, a), cp.inv_td));
    const double y = __dmul_rn(cp.td, M);
    const double v = __dadd_rn(a, y);
    // the chain rounds here exactly when a + y is inexact
    if (!add_exact(a, y, v)) a = v;
    return v;
}

// Escape prediction from the previous input (exact whenever the previous
// element escaped, since the predictor then IS that input): the reference
// escapes when llround((x - P)/2delta) leaves (-32768, 32768).
__device__ __forceinline__ bool predict_escape(const CodecParams& cp, double x, double xprev)
{
    return fabs(__dmul_rn(__dsub_rn(x, xprev), cp.inv_td)) >= 32767.5;
}

// lattice_step that also returns M (relative to the anchor it used) and
// whether the reference step is provably equal to the lattice step:
//   with P_prev = a + 2d*M_prev exactly, y = fl(x-a)/2d, |y| < 2^30 and y at
//   least 2^-19 away from a half-integer, the reference's
//   llround(fl(x-P_prev)/2d) equals rint(y) - M_prev (both subtractions err by
//   < 2^-21 in units of 2d), its recon fl(P_prev + 2d*q) rounds the same real
//   a + 2d*M as we do, and its bound check |x-recon| <= delta holds.
__device__ __forceinline__ double lattice_step_m(const CodecParams& cp, double& a, double x, double& M,
                                                 bool& safe)
{
    const double y = __dmul_rn(__dsub_rn(x, a), cp.inv_td);
    M = rint(y);
    const double fr = fabs(__dsub_rn(y, M));
    safe = fabs(y) < 1073741824.0 && fr < 0.5 - 1.9073486328125e-06;  // 2^30, 0.5 - 2^-19
    const double yv = __dmul_rn(cp.td, M);
    const double v = __dadd_rn(a, yv);
    if (!add_exact(a, yv, v)) a = v;  // the chain rounds here: re-anchor (M relative to v is 0)
    return v;
}

// lattice_step_m without moving the anchor: sets rnd when the chain would
// round (re-anchor) here, so a group of steps can run independently.
__device__ __forceinline__ double lattice_try(const CodecParams& cp, double a, double x, double& M,
                                              bool& safe, bool& rnd)
{
    const double y = __dmul_rn(__dsub_rn(x, a), cp.inv_td);
    M = rint(y);
    const double fr = fabs(__dsub_rn(y, M));
    safe = fabs(y) < 1073741824.0 && fr < 0.5 - 1.9073486328125e-06;
    const double yv = __dmul_rn(cp.td, M);
    const double v = __dadd_rn(a, yv);
    rnd |= !add_exact(a, yv, v);
    return v;
}

__device__ __forceinline__ bool same_bits(double a, double b)
{
    return __double_as_longlong(a) == __double_as_longlong(b);
}

// apply_pair arithmetic (gate.cpp:153-162), left to right, no FMA.
__device__ __forceinline__ void pair_update(const double* m, double& r0, double& i0, double& r1,
                                            double& i1)
{
    const double t0r = r0, t0i = i0, t1r = r1, t1i = i1;
    r0 = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(m[0], t0r), __dmul_rn(m[1], t0i)), __dmul_rn(m[2], t1r)),
                   __dmul_rn(m[3], t1i));
    i0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[0], t0i), __dmul_rn(m[1], t0r)), __dmul_rn(m[2], t1i)),
                   __dmul_rn(m[3], t1r));
    r1 = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(m[4], t0r), __dmul_rn(m[5], t0i)), __dmul_rn(m[6], t1r)),
                   __dmul_rn(m[7], t1i));
    i1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[4], t0i), __dmul_rn(m[5], t0r)), __dmul_rn(m[6], t1i)),
                   __dmul_rn(m[7], t1r));
}

// Row halves of apply_pair: the lo output from (t0, t1) and the hi output.
__device__ __forceinline__ void pair_lo(const double* m, double t0r, double t0i, double t1r, double t1i,
                                        double& r, double& i)
{
    r = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(m[0], t0r), __dmul_rn(m[1], t0i)), __dmul_rn(m[2], t1r)),
                  __dmul_rn(m[3], t1i));
    i = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[0], t0i), __dmul_rn(m[1], t0r)), __dmul_rn(m[2], t1i)),
                  __dmul_rn(m[3], t1r));
}

__device__ __forceinline__ void pair_hi(const double* m, double t0r, double t0i, double t1r, double t1i,
                                        double& r, double& i)
{
    r = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(m[4], t0r), __dmul_rn(m[5], t0i)), __dmul_rn(m[6], t1r)),
                  __dmul_rn(m[7], t1i));
    i = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[4], t0i), __dmul_rn(m[5], t0r)), __dmul_rn(m[6], t1i)),
                  __dmul_rn(m[7], t1r));
}

}  // namespace qcs
