// Streaming fused kernel for ELEMENT-WISE gates: decompress -> scale -> gate
// -> snap -> recompress (+ stored sum of squares, side index) with no
// uncompressed plane anywhere — not even in shared memory.
//
// Same contract and buffers as k_fused MODE_LOCAL (qcs_fused.cuh), i.e. the
// body of CompressedState::apply_gate's worker loop (aalc.cpp:315-382) for
// gates whose run_plan_unit (gate.cpp:405-454) touches every amplitude on its
// own: diagonal single / controlled gates on any target (a diagonal
// apply_pair, gate.cpp:153-162, adds the partner multiplied by exact zeros;
// DESIGN.md §4), phase flips, reflect_mean.  Output level: lossy with 2*delta a
// power of two.
//
// One CTA per stride, ST_LANES lanes; a lane owns one 32-element sub-chunk of
// BOTH planes per iteration and walks it once, element by element:
//   re/im token streams (side-index entry, staged payload bytes) -> predictor
//   values -> * scale -> gate -> snap -> quantize -> code tokens into the
//   lane's staging row, units of the exact sum of squares.
// Quantization uses the fact the legacy encoder's event rounds establish for
// such states (qcs_fused.cuh, lane_chain): while no step of a plane's chain
// is an escape, the reference predictor (codec.cpp:224-247) stays on the
// lattice 2*delta*Z anchored at the plane's initial predictor 0, so
//   M_k = rint(x_k / 2d),  code_k = M_k - M_{k-1},  recon_k = 2d * M_k
// whenever the step is PROVEN equal to the reference's (|y| < 2^30, y at least
// 2^-19 from a half-integer, |code| <= 32766); any other step is the
// reference step itself (ref_step) from the exact predictor 2d*M_{k-1}, and
// must land on the lattice again.  An escape, an off-lattice predictor or any
// state this kernel does not cover sets redo[slot]: the legacy kernel then
// re-encodes that slot from scratch (the outputs written here are dead).
// Without escapes the only runs are zero runs, which carry no reserved bytes,
// so a run token sits where the run closes and a sub-chunk starting inside a
// run has its side offset at the lane's own first byte.
//
// Stored sum of squares (aalc.cpp:46-52, core.cpp:30-37): the integer-units
// argument of fused_sumsq without stored values — every lane accumulates its
// units under the binade of the running sum and under the next one while it
// walks; an iteration without event is one CTA reduction; at a binade crossing
// or tie the lane whose prefix reaches the binade's end replays its sub-chunk
// (decode + gate + quantize again) up to the event, adds it exactly, and the
// lanes after it switch to their next-binade units.
//
// Iteration = steps A (TMA staging of both planes' payload bytes), B (the
// walk), C (first elements, runs across lanes, lead tokens, byte scan, side
// index), D (stored sum), E (rows packed into the plane's contiguous image in
// the dead staging buffer, 16-byte stores).  In the wave layout with a
// single-level ladder the CTA finally installs its own stride (StreamCommit).
#pragma once

#include "qcs_fused.cuh"

namespace qcs {

// CTA shapes: ST_LANES lanes (one complex sub-chunk each per iteration) —
// 128 (four CTAs per SM), 256 (two) or 512 (one), chosen by the slots per SM
// of the launch: shared memory per lane is constant (~432 bytes)
constexpr int ST_LEAD = 12;               // bytes reserved in front of a row's body for the lead tokens
constexpr int ST_ROW = 116;               // row pitch: 12 lead + 93 body + 5 tail, rounded to an odd word count
constexpr int ST_STAGE_PER_LANE = 96;     // staged payload bytes per plane, lane and iteration (3 B per element)
constexpr int ST_SERIAL = 512;            // first terms of a stride's sum, added one by one (fused_sumsq)

template <int ST_LANES>
struct StreamSharedT {
    static constexpr int ST_WARPS = ST_LANES / 32;
    static constexpr int ST_STAGE = ST_STAGE_PER_LANE * ST_LANES;
    alignas(16) uint8_t in[2][ST_STAGE];
    alignas(16) uint8_t rows[2 * ST_LANES * ST_ROW];
    int mlast[2][ST_LANES];
    uint32_t wmax[2][ST_WARPS];
    uint32_t wbytes[2][ST_WARPS];
    uint64_t wunits[ST_WARPS];
    uint64_t bar[2];
    // carried per plane
    uint64_t out_pos[2];
    uint32_t run_start[2];  // first element of the zero run open at the iteration's start (== base: none)
    int m_carry[2];         // M of the plane's last element so far
    // sum of squares
    double s;
    double ev_s;
    uint64_t ev_part;
    uint32_t ev_k;
    int ev_any;
    int ev_owner;
};
static_assert(sizeof(StreamSharedT<128>) <= 55 * 1024 + 768, "four 128-lane streaming CTAs per SM");
static_assert(sizeof(StreamSharedT<256>) <= 112 * 1024, "two 256-lane streaming CTAs per SM");
static_assert(sizeof(StreamSharedT<512>) <= 226 * 1024, "one 512-lane streaming CTA per SM");

// Sequential reader of one plane's token stream from a side-index entry
// (decode_sub's walk, one element per call).  `in` is 4-byte aligned; reads
// up to 7 bytes past a token's first byte.
struct TokReader {
    const uint8_t* in;  // generic pointer to the staged bytes (slow paths)
    uint32_t sa;        // the same as a shared-window address
    uint32_t pos;
    uint32_t skip;
    uint32_t zleft, wleft;
    int codec;
    double td, P;

    __device__ __forceinline__ void init(const uint8_t* in_, int codec_, double td_, SideEntry se)
    {
        in = in_;
        sa = (uint32_t)__cvta_generic_to_shared(in_);
        pos = se.off;
        codec = codec_;
        skip = se.skip;
        zleft = wleft = 0;
        td = td_;
        P = se.pred;
    }
    __device__ __forceinline__ uint32_t fetch4(uint32_t at) const
    {
        uint32_t lo, hi;
        const uint32_t ad = sa + (at & ~3u);
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(ad));
        asm volatile("ld.shared.u32 %0, [%1+4];" : "=r"(hi) : "r"(ad));
        return __funnelshift_r(lo, hi, (at & 3u) << 3);
    }
    __device__ __forceinline__ double word()
    {
        const uint64_t w = (uint64_t)fetch4(pos) | ((uint64_t)fetch4(pos + 4) << 32);
        pos += 8;
        return __longlong_as_double((long long)w);
    }
    // a run token (value v): zero run or raw words, lossy or lossless
    __device__ __forceinline__ double run_token(uint64_t v)
    {
        const bool words = codec == 1 ? (v & 3u) == 2u : (v & 1u) != 0u;
        const uint32_t left = (uint32_t)((codec == 1 ? v >> 2 : v >> 1) - skip) - 1u;
        if (!words) {
            zleft = left;
            skip = 0;
            return codec == 1 ? P : 0.0;
        }
        pos += 8u * skip;
        skip = 0;
        wleft = left;
        const double x = word();
        if (codec == 1) P = x;
        return x;
    }
    // the next element's decoded value (before the stride scale)
    __device__ __forceinline__ double next()
    {
        // (the window is read speculatively: inside a run it is not a token)
        const uint32_t w = fetch4(pos);
        const uint32_t m = ~w & 0x80808080u;
        const uint32_t tm = m ^ (m - 1u);  // the token's bits (m != 0)
        const uint32_t x = w & tm;
        // lossy code token (tag 1 in the first byte) of up to 4 bytes, no run pending
        if (((zleft | wleft) | (uint32_t)(codec ^ 1) | ((w & 3u) ^ 1u)) == 0u && m != 0u) {
            pos += (uint32_t)__popc(tm & 0x01010101u);
            const uint32_t z = ((x >> 2) & 0x1fu) | ((x >> 3) & 0xfe0u) | ((x >> 4) & 0x7f000u) | ((x >> 5) & 0x3f80000u);
            P = __dadd_rn(P, __dmul_rn(td, (double)((int)(z >> 1) ^ -(int)(z & 1u))));
            return P;
        }
        const uint32_t v = (x & 0x7fu) | ((x >> 1) & 0x3f80u) | ((x >> 2) & 0x1fc000u) | ((x >> 3) & 0xfe00000u);
        if ((zleft | wleft) == 0u) {
            if (m != 0u) {  // a run token of up to 4 bytes
                pos += (uint32_t)__ffs((int)m) >> 3;
                return run_token(v);
            }
            uint64_t p64 = pos;
            const uint64_t v = get_varint(in, p64);
            pos = (uint32_t)p64;
            if (codec == 1 && (v & 3u) == 1u) {  // (not a valid code: too large; keep the walk defined)
                P = __dadd_rn(P, __dmul_rn(td, (double)unzigzag(v >> 2)));
                return P;
            }
            return run_token(v);
        }
        if (zleft) {
            --zleft;
            return codec == 1 ? P : 0.0;
        }
        --wleft;
        const double xw = word();
        if (codec == 1) P = xw;
        return xw;
    }
};

// Wave layout, single-level ladder: the encoder CTA installs its own stride
// (the staged commit of aalc.cpp:395-408 for that stride) instead of leaving it
// to k_wave_commit — its copy from the staging slot into the arena then runs
// under the other CTAs' encoding.  The host reserved the wave's worst case
// behind the bump (k_wave_reserve sets *direct); a CTA takes its 16-byte-rounded
// bytes from that block with one atomic, copies payloads and side entries,
// installs the tables and marks the slot committed.  Slots left to the legacy
// encoder, and every slot when *direct is 0, keep the staged path.
struct StreamCommit {
    const int* direct;             // null: never
    unsigned long long* wave_used; // bytes taken from the wave's block
    const uint64_t* bump;          // arena fill before the wave
    // persistent kernel (k_stream_persist): no wave, every stride takes its bytes from the
    // arena's bump itself; a stride that does not fit suspends the gate (the slots installed
    // so far stay, `committed`; the host compacts and the gate resumes with the others)
    unsigned long long* bump_rw;   // non-null: persistent mode
    uint64_t arena_cap;
    int* err_rw;
    int* persist_susp;             // set with the error word: the suspension is this kernel's
    unsigned long long* persist_done;
    // block capacities: a block this kernel places gets a little slack (1/256 + 64 bytes); the
    // stride's next encoding goes over it in place when both planes fit — by then the CTA has read
    // the old blocks to their end and nobody else reads them — so a state whose strides keep
    // their size needs no new arena bytes and no compaction.  p_capoff[g] is the offset p_cap[g]
    // belongs to: any other installer (staged commit, import, compaction) moves p_off and so
    // invalidates the capacity.
    uint64_t* p_cap;
    uint64_t* p_capoff;
    uint8_t* arena;
    SideEntry* side;               // the block store's side index [2NS][nsub]
    uint64_t* p_off;
    uint64_t* p_len;
    int8_t* p_codec;
    double* p_delta;
    double* scale;
    double* sum_sq;
    unsigned long long* gate_cin;
    uint8_t* committed;            // [slot]
};

__device__ __forceinline__ void stream_copy16(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t n16, int tid,
                                              int nt)
{
    uint64_t i = (uint64_t)tid;
    const uint64_t T = (uint64_t)nt;
    for (; i + 3 * T < n16; i += 4 * T) {
        const uint4 a = __ldcs(src + i), b = __ldcs(src + i + T), c = __ldcs(src + i + 2 * T), e = __ldcs(src + i + 3 * T);
        __stcs(dst + i, a);
        __stcs(dst + i + T, b);
        __stcs(dst + i + 2 * T, c);
        __stcs(dst + i + 3 * T, e);
    }
    for (; i < n16; i += T) __stcs(dst + i, __ldcs(src + i));
}

// install slot `gslot` (stride j) from its staging slot; lens: the planes' payload bytes
__device__ __forceinline__ void stream_commit(const FusedArgs& a, const StreamCommit& dc, uint64_t slot, uint64_t gslot,
                                              uint64_t j, uint64_t len0, uint64_t len1, double sumsq, uint64_t* sh_off,
                                              int tid, int nt)
{
    const uint64_t r0 = (len0 + 15) & ~uint64_t(15), r1 = (len1 + 15) & ~uint64_t(15);
    uint64_t at, at1;
    bool fresh = true;
    uint64_t c0 = r0, c1 = r1;  // capacities of freshly placed blocks
    if (dc.bump_rw) {
        __shared__ uint64_t sh_at1;
        __shared__ int sh_fresh;
        c0 = (r0 + (r0 >> 8) + 64 + 15) & ~uint64_t(15);  // (slack16 of qcs_engine.cu)
        c1 = (r1 + (r1 >> 8) + 64 + 15) & ~uint64_t(15);
        if (tid == 0) {
            const uint64_t g0 = 2 * j, g1 = 2 * j + 1;
            const bool reuse = dc.p_cap && dc.p_capoff[g0] == dc.p_off[g0] && dc.p_capoff[g1] == dc.p_off[g1] &&
                               r0 <= dc.p_cap[g0] && r1 <= dc.p_cap[g1];
            sh_fresh = reuse ? 0 : 1;
            if (reuse) {
                *sh_off = dc.p_off[g0];
                sh_at1 = dc.p_off[g1];
            }
        }
        __syncthreads();
        fresh = sh_fresh != 0;
        if (tid == 0 && fresh) {
            const unsigned long long need = (unsigned long long)(c0 + c1);
            unsigned long long off = atomicAdd(dc.bump_rw, need);
            if (off + need > dc.arena_cap) {
                // arena full: suspend the gate.  (The bump stays where it is — taking the bytes back
                // could pull it under a block another CTA placed meanwhile; the compaction that
                // follows recomputes it from the live blocks.)
                *dc.persist_susp = 1;
                __threadfence();
                atomicCAS(dc.err_rw, 0, 99 /* QCS_SUSPEND */);
                off = ~0ull;
                dc.committed[gslot] = 0;
            }
            *sh_off = (uint64_t)off;
            sh_at1 = (uint64_t)off + c0;
        }
        __syncthreads();
        if (*sh_off == ~uint64_t(0)) return;
        at = *sh_off;
        at1 = sh_at1;
    } else {
        if (tid == 0) *sh_off = (uint64_t)atomicAdd(dc.wave_used, (unsigned long long)(r0 + r1));
        __syncthreads();
        at = *dc.bump + *sh_off;
        at1 = at + r0;
    }
    stream_copy16(reinterpret_cast<uint4*>(dc.arena + at), reinterpret_cast<const uint4*>(a.out + (2 * slot) * a.cap), r0 / 16, tid, nt);
    stream_copy16(reinterpret_cast<uint4*>(dc.arena + at1), reinterpret_cast<const uint4*>(a.out + (2 * slot + 1) * a.cap),
                  r1 / 16, tid, nt);
    stream_copy16(reinterpret_cast<uint4*>(dc.side + (2 * j) * a.nsub), reinterpret_cast<const uint4*>(a.side + (2 * slot) * a.nsub),
                  a.nsub, tid, nt);
    stream_copy16(reinterpret_cast<uint4*>(dc.side + (2 * j + 1) * a.nsub),
                  reinterpret_cast<const uint4*>(a.side + (2 * slot + 1) * a.nsub), a.nsub, tid, nt);
    if (tid == 0) {
        atomicAdd(dc.gate_cin, (unsigned long long)(2 * HEADER_BYTES + dc.p_len[2 * j] + dc.p_len[2 * j + 1]));
        dc.p_off[2 * j] = at;
        dc.p_off[2 * j + 1] = at1;
        if (dc.bump_rw && fresh && dc.p_cap) {
            dc.p_cap[2 * j] = c0;
            dc.p_cap[2 * j + 1] = c1;
            dc.p_capoff[2 * j] = at;
            dc.p_capoff[2 * j + 1] = at1;
        }
        dc.p_len[2 * j] = len0;
        dc.p_len[2 * j + 1] = len1;
        dc.p_codec[2 * j] = dc.p_codec[2 * j + 1] = 1;
        dc.p_delta[2 * j] = dc.p_delta[2 * j + 1] = a.cp.delta;
        dc.sum_sq[j] = sumsq;
        dc.scale[j] = 1.0;
        dc.committed[gslot] = 1;
        if (dc.persist_done) atomicAdd(dc.persist_done, 1ull);
    }
}

// nb bytes from shared memory (any alignment) to dst (generic, any alignment): bytes up to
// dst's first 4-byte boundary, aligned words (one shared word read and a funnel shift each),
// bytes again for the tail — the boundary words belong to the neighbours' bytes too
__device__ __forceinline__ void stream_lane_copy(uint8_t* dst, const uint8_t* srow, uint32_t nb)
{
    uint32_t i = 0;
    const uint32_t head = min(nb, (uint32_t)((0u - (uint32_t)(uintptr_t)dst) & 3u));
    for (; i < head; ++i) dst[i] = srow[i];
    if (i + 4u <= nb) {
        const uint32_t sad = (uint32_t)__cvta_generic_to_shared(srow + i);
        const uint32_t sh = (sad & 3u) << 3;
        uint32_t wa = sad & ~3u, lo;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(wa) : "memory");
        for (; i + 4u <= nb; i += 4u) {
            uint32_t hi;
            wa += 4u;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(wa) : "memory");
            *reinterpret_cast<uint32_t*>(dst + i) = __funnelshift_r(lo, hi, sh);
            lo = hi;
        }
    }
    for (; i < nb; ++i) dst[i] = srow[i];
}

struct StreamPlaneOut {
    double x0;
    int M0, Mlast;
    bool good0, seen;
    int lz1, tz, body;
};

constexpr uint64_t ST_SAT = 1ull << 62;

// RAW: the planes were decoded, gated and snapped into a.X by the split path
// (k_decode_gate) or are the caller's (a load): the walk reads them there and
// only quantizes, emits and sums.
// One slot: `slot` is the CTA's staging slot (out / side / X scratch), `gslot` the
// gate's slot (tables, flags).  The mbarriers are initialised by the kernel;
// stage_phase carries their parity from slot to slot.
template <int ST_LANES, bool RAW>
__device__ __forceinline__ void stream_slot(const FusedArgs& a, uint8_t* redo, const StreamCommit& dc, const uint64_t slot,
                                            const uint64_t gslot, unsigned (&stage_phase)[2])
{
    using StreamShared = StreamSharedT<ST_LANES>;
    constexpr int ST_WARPS = StreamShared::ST_WARPS;
    constexpr int ST_STAGE = StreamShared::ST_STAGE;
    constexpr int ST_ITER = ST_LANES * SUB;  // elements per plane per iteration
    const int tid = threadIdx.x, wl = tid & 31, wp = tid >> 5;
    const bool direct = dc.bump_rw || (dc.direct && *dc.direct);  // (uniform; the pool layout never sets it)
    if (a.zero_slot && a.zero_slot[gslot]) {
        if (direct) {
            // a zero stride already stored as this level's zero encodings (one run token per plane,
            // side entries {0, 32k, 0.0}: write_zero_plane's) is its own output: only the stride's
            // scale and sum change, nothing is written or copied
            const uint64_t j = a.job_stride[gslot];
            if (dc.p_codec[2 * j] == 1 && dc.p_codec[2 * j + 1] == 1 && dc.p_delta[2 * j] == a.cp.delta &&
                dc.p_delta[2 * j + 1] == a.cp.delta) {
                if (tid == 0) {
                    const uint64_t zl = (uint64_t)varint_len(run_token(1, TY_Z, a.n));
                    a.out_len[2 * gslot] = a.out_len[2 * gslot + 1] = zl;
                    if (a.sumsq) a.sumsq[gslot] = 0.0;
                    redo[gslot] = 0;
                    atomicAdd(dc.gate_cin, (unsigned long long)(2 * HEADER_BYTES + dc.p_len[2 * j] + dc.p_len[2 * j + 1]));
                    dc.sum_sq[j] = 0.0;
                    dc.scale[j] = 1.0;
                    dc.committed[gslot] = 1;
                    if (dc.persist_done) atomicAdd(dc.persist_done, 1ull);
                }
                return;
            }
        }
        for (int c = 0; c < 2; ++c) write_zero_plane<true>(a, slot, gslot, c, tid, ST_LANES);
        if (tid == 0) {
            if (a.sumsq) a.sumsq[gslot] = 0.0;
            redo[gslot] = 0;
        }
        if (direct) {
            __shared__ uint64_t zoff;
            const uint64_t zl = (uint64_t)varint_len(run_token(1, TY_Z, a.n));
            __syncthreads();  // (the zero encodings above are this CTA's own global writes)
            stream_commit(a, dc, slot, gslot, a.job_stride[gslot], zl, zl, 0.0, &zoff, tid, ST_LANES);
        } else if (dc.committed && tid == 0) {
            dc.committed[gslot] = 0;
        }
        return;
    }

    extern __shared__ __align__(16) unsigned char smem[];
    StreamShared& S = *reinterpret_cast<StreamShared*>(smem);
    const double td = a.cp.td, inv_td = a.cp.inv_td;
    const uint64_t n = a.n;
    const uint64_t in_stride = a.job_stride[gslot];
    const double scale = RAW ? 1.0 : a.scale[in_stride];
    const bool sc = scale != 1.0;
    // RAW: this slot's planes in X; a slot flagged zero-imaginary has no im plane there
    const double* xg[2] = {nullptr, nullptr};
    if (RAW) {
        xg[0] = a.X + (2 * slot) * a.x_plane_stride;
        xg[1] = (a.im_zero && a.im_zero[gslot]) ? nullptr : a.X + (2 * slot + 1) * a.x_plane_stride;
    }

    // input planes and output slots (k_fused's addressing)
    const uint8_t* in_bytes[2];
    const SideEntry* in_side[2];
    int in_codec[2];
    double in_td[2];
    uint8_t* out[2];
    SideEntry* side[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const uint64_t gpl = 2 * in_stride + p;
        int live_sel = 0;
        if (a.pool) {
            live_sel = (int)((a.p_off[gpl] / a.cap) & 1);
            out[p] = a.out + (2 * gpl + 1 - live_sel) * a.cap;
            side[p] = a.side + (2 * gpl + 1 - live_sel) * a.nsub;
        } else {
            out[p] = a.out + (2 * slot + p) * a.cap;
            side[p] = a.side + (2 * slot + p) * a.nsub;
        }
        in_bytes[p] = (*a.arena_cur ? a.arena1 : a.arena0) + a.p_off[gpl];
        in_codec[p] = a.p_codec[gpl];
        in_td[p] = 2.0 * a.p_delta[gpl];
        in_side[p] = a.pool ? a.side_in + (2 * gpl + live_sel) * a.nsub : a.side_in + gpl * a.nsub;
    }
    // the gate, element-wise
    const int kind = a.kind;
    const int fixed_side = a.diag == 2 ? (int)(gslot & 1) : -1;
    const double mr2 = kind == 3 ? 2.0 * a.mean[0] : 0.0, mi2 = kind == 3 ? 2.0 * a.mean[1] : 0.0;
    // side and control are constant over a lane's 32 elements when their bits are >= 5
    const bool gate_const = kind <= 1 && (fixed_side >= 0 || a.t >= 5) && (a.local_ctl < 0 || a.local_ctl >= 5);

    __syncthreads();  // (a persistent CTA: the previous slot's readers of S are done)
    if (tid == 0) {
        S.out_pos[0] = S.out_pos[1] = 0;
        S.run_start[0] = S.run_start[1] = 0;
        S.m_carry[0] = S.m_carry[1] = 0;
        S.s = 0.0;
    }
    bool bail = false;  // uniform over the CTA
    int why = 0;        // why the slot was left (counters[19 + why]): 0 input not staged, 1 unproven step, 2 first element, 3 sum head, 4 sum event
    __syncthreads();

    for (uint64_t base = 0; base < n; base += ST_ITER) {
        const uint32_t e0 = (uint32_t)base + (uint32_t)tid * SUB;
        const bool have = e0 < n;  // (n is a multiple of SUB: a lane has 32 elements or none)
        const bool final_iter = base + ST_ITER >= n;
        const int active = (int)umin64(ST_LANES, (n - base) / SUB);
        const uint64_t sc0 = base / SUB;

        // A. stage this iteration's payload bytes of both planes (one TMA bulk copy each)
        const uint8_t* src[2] = {nullptr, nullptr};
#pragma unroll
        for (int p = 0; p < 2 && !RAW; ++p) {
            const uint64_t lo = in_side[p][sc0].off & ~uint64_t(15);
            uint64_t hi;
            if (final_iter) {
                hi = a.p_len[2 * in_stride + p];
            } else {
                const SideEntry nx = in_side[p][sc0 + ST_LANES];
                hi = (uint64_t)nx.off + 10 + 8 * (uint64_t)nx.skip;
            }
            const uint64_t nb = hi > lo ? ((hi - lo + 15) & ~uint64_t(15)) : 0;
            src[p] = S.in[p] - lo;
            if (nb > 0 && nb <= ST_STAGE) {  // uniform over the CTA
                if (tid == 0) bulk_g2s(S.in[p], in_bytes[p] + lo, (unsigned)nb, &S.bar[p]);
                mbar_wait(&S.bar[p], stage_phase[p]);
                stage_phase[p] ^= 1u;
            } else {  // more than 3 bytes per element: poorly compressed input, the legacy encoder's
                bail = true;
            }
        }
        if (bail) break;
        const double s_in = S.s;  // the running sum entering this iteration (uniform)
        const bool have_tu = s_in > 0.0 && ilogb(s_in) >= -960;
        const double tu_main = have_tu ? ldexp(1.0, 52 - ilogb(s_in)) : 0.0;
        // the lane's gate when side and control do not change inside it
        bool gate_on = true;
        double gur = 0.0, gui = 0.0;
        if (gate_const) {
            gate_on = a.local_ctl < 0 || ((e0 >> a.local_ctl) & 1u);
            const int sd = fixed_side >= 0 ? fixed_side : (int)((e0 >> a.t) & 1u);
            gur = sd ? a.u[6] : a.u[0];
            gui = sd ? a.u[7] : a.u[1];
        }

        // One walk over the lane's sub-chunk: decode, scale, gate, snap, quantize.
        //  PASS 0  the main pass: tokens into the staging row, first-element
        //          facts into po, sum units of every element under tu (uA) and
        //          under the next binade (uB)
        //  PASS 1  replay: sum units of every element under tu (uA)
        //  PASS 2  replay: the terms t_k of the elements below ST_SERIAL into tdst
        //  PASS 3  replay by the lane holding a sum event: from ms + uA units
        //          (binade of tu) add the elements after k_after until the event,
        //          add it exactly (S.ev_s, S.ev_k), then the units of the lane's
        //          remaining elements under the new binade (S.ev_part)
        // Returns false when a step is neither proven nor a lattice-preserving
        // reference step (the slot is left to the legacy encoder).
        uint64_t uA = 0, uB = 0;
        uint64_t ownB = ST_SAT;  // PASS 3: the walking lane's own next-binade units of the whole sub-chunk (ST_SAT: unknown)
        auto walk = [&](auto pass_tag, StreamPlaneOut* po, double tu, long long k_after, double* tdst,
                        uint64_t ms) -> bool {
            constexpr int PASS = decltype(pass_tag)::value;
            TokReader rd[2];
            if (!RAW) {
#pragma unroll
                for (int p = 0; p < 2; ++p) rd[p].init(src[p], in_codec[p], in_td[p], in_side[p][e0 / SUB]);
            }
            int kx = 0;  // RAW: the next element of the lane's rows in X
            int Mprev[2] = {0, 0};
            int run[2] = {0, 0};
            uint32_t wa[2] = {0, 0}, wa0[2] = {0, 0};  // shared-window address of the next token byte / the body
            if (PASS == 0) {
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    wa0[p] = wa[p] = (uint32_t)__cvta_generic_to_shared(S.rows + (size_t)(p * ST_LANES + tid) * ST_ROW + ST_LEAD);
                    po[p].seen = false;
                    po[p].lz1 = 0;
                }
            }
            uint64_t la = PASS == 3 ? uA : 0, lb = 0;
            uint64_t lbp = 0;  // PASS 3: next-binade units of the elements up to the event
            bool eva = false, evb = false, bad = false, found = false, stop = false;
            double tu2 = 0.0;
            // the next element of both planes: the usual case (both streams at a
            // nonzero code token) in one straight line, anything else by next()
            auto next2 = [&](double& xr, double& xi) {
                if (RAW) {
                    xr = __ldcs(xg[0] + e0 + kx);
                    xi = xg[1] ? __ldcs(xg[1] + e0 + kx) : 0.0;
                    ++kx;
                    return;
                }
                const uint32_t w0 = rd[0].fetch4(rd[0].pos), w1 = rd[1].fetch4(rd[1].pos);
                const uint32_t m0 = ~w0 & 0x80808080u, m1 = ~w1 & 0x80808080u;
                const uint32_t t0 = m0 ^ (m0 - 1u), t1 = m1 ^ (m1 - 1u);
                const uint32_t x0 = w0 & t0, x1 = w1 & t1;
                const uint32_t busy = rd[0].zleft | rd[0].wleft | rd[1].zleft | rd[1].wleft |
                                      (uint32_t)(rd[0].codec ^ 1) | (uint32_t)(rd[1].codec ^ 1) | ((w0 & 3u) ^ 1u) |
                                      ((w1 & 3u) ^ 1u);
                const uint32_t z0 = ((x0 >> 2) & 0x1fu) | ((x0 >> 3) & 0xfe0u) | ((x0 >> 4) & 0x7f000u) | ((x0 >> 5) & 0x3f80000u);
                const uint32_t z1 = ((x1 >> 2) & 0x1fu) | ((x1 >> 3) & 0xfe0u) | ((x1 >> 4) & 0x7f000u) | ((x1 >> 5) & 0x3f80000u);
                const double P0 = __dadd_rn(rd[0].P, __dmul_rn(rd[0].td, (double)((int)(z0 >> 1) ^ -(int)(z0 & 1u))));
                const double P1 = __dadd_rn(rd[1].P, __dmul_rn(rd[1].td, (double)((int)(z1 >> 1) ^ -(int)(z1 & 1u))));
                if (busy == 0u && m0 != 0u && m1 != 0u) {
                    rd[0].pos += (uint32_t)__popc(t0 & 0x01010101u);
                    rd[1].pos += (uint32_t)__popc(t1 & 0x01010101u);
                    rd[0].P = xr = P0;
                    rd[1].P = xi = P1;
                } else {
                    xr = rd[0].next();
                    xi = rd[1].next();
                }
            };
            // scale, gate (run_plan_unit, gate.cpp:405-454) and snap of element k:
            // every element on its own — apply_pair with a zero partner, minus its
            // exact-zero terms (they change a zero's sign at most: snapped)
            auto gate_snap = [&](int k, double& xr, double& xi) {
                if (RAW) {  // gated already; snapped already unless the caller asks
                    if (a.snap) {
                        xr = snap(xr);
                        xi = snap(xi);
                    }
                    return;
                }
                if (sc) {
                    xr = __dmul_rn(xr, scale);
                    xi = __dmul_rn(xi, scale);
                }
                if (kind <= 1) {
                    bool on = gate_on;
                    double ur = gur, ui = gui;
                    if (!gate_const) {
                        const uint32_t gi = e0 + (uint32_t)k;
                        on = a.local_ctl < 0 || ((gi >> a.local_ctl) & 1u);
                        const int sd = fixed_side >= 0 ? fixed_side : (int)((gi >> a.t) & 1u);
                        ur = sd ? a.u[6] : a.u[0];
                        ui = sd ? a.u[7] : a.u[1];
                    }
                    const double orr = __dsub_rn(__dmul_rn(ur, xr), __dmul_rn(ui, xi));
                    const double oi = __dadd_rn(__dmul_rn(ur, xi), __dmul_rn(ui, xr));
                    xr = on ? orr : xr;
                    xi = on ? oi : xi;
                } else if (kind == 2) {
                    if ((uint64_t)e0 + (uint64_t)k == a.flip_off) {
                        xr = -xr;
                        xi = -xi;
                    }
                } else {
                    xr = __dsub_rn(mr2, xr);
                    xi = __dsub_rn(mi2, xi);
                }
                xr = snap(xr);
                xi = snap(xi);
            };
            // the reference step of plane p from the exact predictor (a step the lattice test does not prove)
            auto slow_step = [&](int p, double x, int& M, int& q) {
                double P = __dmul_rn(td, (double)Mprev[p]);
                const int32_t t = ref_step(a.cp, P, x);
                M = Mprev[p] + t;
                q = t;
                if (t == WCODE || M <= -1073741824 || M >= 1073741824 || !same_bits(__dmul_rn(td, (double)M), P)) bad = true;
            };
            // token(s) of code q of plane p (PASS 0): any case
            auto emit_any = [&](int p, int q) {
                if (q == 0) {
                    ++run[p];
                    return;
                }
                if (!po[p].seen) {  // the lane's leading zero run goes with the lead tokens
                    po[p].seen = true;
                    po[p].lz1 = run[p];
                } else if (run[p] > 0) {  // a zero run inside the lane (< 32: one byte)
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(wa[p]), "r"((uint32_t)run[p] << 2) : "memory");
                    ++wa[p];
                }
                run[p] = 0;
                const uint32_t z = ((uint32_t)q << 1) ^ (uint32_t)(q >> 31);
                const uint32_t v = (z << 2) | 1u;
                const bool l2 = v >= 128u, l3 = v >= 16384u;
                asm volatile("st.shared.u8 [%0], %1;" ::"r"(wa[p]), "r"((v & 0x7fu) | (l2 ? 0x80u : 0u)) : "memory");
                if (l2)
                    asm volatile("st.shared.u8 [%0+1], %1;" ::"r"(wa[p]), "r"(((v >> 7) & 0x7fu) | (l3 ? 0x80u : 0u)) : "memory");
                if (l3) asm volatile("st.shared.u8 [%0+2], %1;" ::"r"(wa[p]), "r"(v >> 14) : "memory");
                wa[p] += 1u + (uint32_t)l2 + (uint32_t)l3;
            };
            // sum-of-squares bookkeeping of element k from the lattice indices
            auto sums = [&](int k, int M0, int M1) {
                const double r0v = __dmul_rn(td, (double)M0), r1v = __dmul_rn(td, (double)M1);
                const double t = __dadd_rn(__dmul_rn(r0v, r0v), __dmul_rn(r1v, r1v));
                if (PASS == 0 || PASS == 1) {
                    const double y0 = t * tu;
                    const double r0 = rint(y0);
                    eva = eva || y0 >= 9007199254740992.0 || fabs(y0 - r0) == 0.5;
                    la += (uint64_t)r0;
                    if (PASS == 0) {
                        const double y1 = y0 * 0.5;
                        const double r1 = rint(y1);
                        evb = evb || y1 >= 9007199254740992.0 || fabs(y1 - r1) == 0.5;
                        lb += (uint64_t)r1;
                    }
                } else if (PASS == 2) {
                    const uint32_t gi = e0 + (uint32_t)k;
                    if (gi < ST_SERIAL) tdst[gi] = t;
                } else {
                    const long long gi = (long long)e0 + k;
                    if (gi > k_after) {
                        const double y = t * (found ? tu2 : tu);
                        const double ry = rint(y);
                        const bool beyond = y >= 9007199254740992.0;
                        const bool tie = !beyond && fabs(y - ry) == 0.5;
                        const uint64_t c = beyond ? (1ull << 53) : (uint64_t)ry;
                        // the same element one binade up (exact halving), for the shortcut below
                        const double yb = y * 0.5;
                        const double rb = rint(yb);
                        const bool oddb = yb >= 9007199254740992.0 || fabs(yb - rb) == 0.5;
                        if (found) {
                            evb = evb || beyond || tie;
                            lb += c;
                        } else if (beyond || tie || ms + la + c >= (1ull << 53)) {
                            const double sn = __dadd_rn((double)(ms + la) / tu, t);
                            S.ev_s = sn;
                            S.ev_k = (uint32_t)gi;
                            if (a.counters) atomicAdd(&a.counters[tie ? 6 : 7], 1ull);
                            found = true;
                            tu2 = (sn > 0.0 && ilogb(sn) >= -960 && ilogb(sn) < 1000) ? ldexp(1.0, 52 - ilogb(sn)) : 0.0;
                            // a plain crossing into the next binade: the rest of the sub-chunk is the
                            // lane's next-binade units of the main pass minus those walked — stop here
                            if (ownB < ST_SAT && !oddb && tu2 == tu * 0.5 && k_after < (long long)e0) {
                                lb = ownB - lbp - (uint64_t)rb;
                                stop = true;
                            }
                        } else {
                            la += c;
                            lbp += (uint64_t)rb;
                            if (oddb) ownB = ST_SAT;  // (a tie or overflow one binade up: no shortcut)
                        }
                    }
                }
            };
            // element 0: its code needs the left neighbour's last index (step C)
            {
                double xr, xi;
                next2(xr, xi);
                gate_snap(0, xr, xi);
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const double x = p ? xi : xr;
                    const double y = __dmul_rn(x, inv_td);
                    const int M = __double2int_rn(y);
                    const double fr = fabs(__dsub_rn(y, (double)M));
                    if (PASS == 0) {
                        po[p].M0 = M;
                        po[p].x0 = x;
                        po[p].good0 = fabs(y) < 1073741824.0 && fr < 0.5 - 1.9073486328125e-06;
                    }
                    Mprev[p] = M;
                }
                sums(0, Mprev[0], Mprev[1]);
            }
#pragma unroll 2
            for (int k = 1; k < SUB; ++k) {
                if (PASS == 3 && stop) break;
                double xr, xi;
                next2(xr, xi);
                gate_snap(k, xr, xi);
                // quantize on the lattice anchored at 0, both planes side by side
                const double y0 = __dmul_rn(xr, inv_td), y1 = __dmul_rn(xi, inv_td);
                int M0 = __double2int_rn(y0), M1 = __double2int_rn(y1);
                const double f0 = fabs(__dsub_rn(y0, (double)M0)), f1 = fabs(__dsub_rn(y1, (double)M1));
                int q0 = M0 - Mprev[0], q1 = M1 - Mprev[1];
                const bool g0 = fabs(y0) < 1073741824.0 && f0 < 0.5 - 1.9073486328125e-06 && (unsigned)(q0 + 32766) <= 65532u;
                const bool g1 = fabs(y1) < 1073741824.0 && f1 < 0.5 - 1.9073486328125e-06 && (unsigned)(q1 + 32766) <= 65532u;
                if (!(g0 && g1)) {
                    if (!g0) slow_step(0, xr, M0, q0);
                    if (!g1) slow_step(1, xi, M1, q1);
                }
                if (PASS == 0) {
                    if (q0 != 0 && q1 != 0 && (run[0] | run[1]) == 0 && po[0].seen && po[1].seen) {
                        // two code tokens, nothing else: one straight line
                        const uint32_t z0 = ((uint32_t)q0 << 1) ^ (uint32_t)(q0 >> 31), z1 = ((uint32_t)q1 << 1) ^ (uint32_t)(q1 >> 31);
                        const uint32_t v0 = (z0 << 2) | 1u, v1 = (z1 << 2) | 1u;
                        const bool a2 = v0 >= 128u, a3 = v0 >= 16384u, b2 = v1 >= 128u, b3 = v1 >= 16384u;
                        asm volatile("st.shared.u8 [%0], %1;" ::"r"(wa[0]), "r"((v0 & 0x7fu) | (a2 ? 0x80u : 0u)) : "memory");
                        asm volatile("st.shared.u8 [%0], %1;" ::"r"(wa[1]), "r"((v1 & 0x7fu) | (b2 ? 0x80u : 0u)) : "memory");
                        if (a2) asm volatile("st.shared.u8 [%0+1], %1;" ::"r"(wa[0]), "r"(((v0 >> 7) & 0x7fu) | (a3 ? 0x80u : 0u)) : "memory");
                        if (b2) asm volatile("st.shared.u8 [%0+1], %1;" ::"r"(wa[1]), "r"(((v1 >> 7) & 0x7fu) | (b3 ? 0x80u : 0u)) : "memory");
                        if (a3) asm volatile("st.shared.u8 [%0+2], %1;" ::"r"(wa[0]), "r"(v0 >> 14) : "memory");
                        if (b3) asm volatile("st.shared.u8 [%0+2], %1;" ::"r"(wa[1]), "r"(v1 >> 14) : "memory");
                        wa[0] += 1u + (uint32_t)a2 + (uint32_t)a3;
                        wa[1] += 1u + (uint32_t)b2 + (uint32_t)b3;
                    } else {
                        emit_any(0, q0);
                        emit_any(1, q1);
                    }
                }
                Mprev[0] = M0;
                Mprev[1] = M1;
                sums(k, M0, M1);
            }
            if (PASS == 0) {
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    po[p].body = (int)(wa[p] - wa0[p]);
                    po[p].Mlast = Mprev[p];
                    po[p].tz = run[p];
                    if (!po[p].seen) po[p].lz1 = SUB - 1;
                }
            }
            if (PASS == 0 || PASS == 1) uA = (eva || la > ST_SAT) ? ST_SAT : la;
            if (PASS == 0) uB = (evb || lb > ST_SAT) ? ST_SAT : lb;
            if (PASS == 3) {
                S.ev_part = (evb || lb > ST_SAT) ? ST_SAT : lb;
                S.ev_any = found ? 1 : 0;
            }
            return !bad;
        };

        // B. main pass
        StreamPlaneOut po[2];
        bool ok = true;
        if (have) ok = walk(std::integral_constant<int, 0>{}, po, tu_main, -1, nullptr, 0);
        if (have) {
            S.mlast[0][tid] = po[0].Mlast;
            S.mlast[1][tid] = po[1].Mlast;
        }
        if (__syncthreads_or(!ok)) {
            bail = true;
            why = 1;
            break;
        }

        // C. first elements, runs across lanes, lead tokens, byte offsets
        uint32_t val[2] = {0, 0};     // start of the lane's trailing zero run, 0: the lane is one zero run
        int q0[2] = {0, 0};
        int Mleft[2] = {0, 0};
        bool bad = false;
        if (have) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                Mleft[p] = tid > 0 ? S.mlast[p][tid - 1] : S.m_carry[p];
                const int q = po[p].M0 - Mleft[p];
                if (po[p].good0 && (unsigned)(q + 32766) <= 65532u) {
                    q0[p] = q;
                } else {  // the reference step; must agree with the lattice point the lane continued from
                    double P = __dmul_rn(td, (double)Mleft[p]);
                    const int32_t t = ref_step(a.cp, P, po[p].x0);
                    if (t == WCODE || Mleft[p] + t != po[p].M0 || po[p].M0 <= -1073741824 || po[p].M0 >= 1073741824 ||
                        !same_bits(__dmul_rn(td, (double)po[p].M0), P))
                        bad = true;
                    q0[p] = (int)t;
                }
                const bool full = q0[p] == 0 && !po[p].seen;
                val[p] = full ? 0u : (po[p].seen ? e0 + SUB - (uint32_t)po[p].tz : e0 + 1u);
            }
        }
        // exclusive max-scan of val over the lanes (per plane)
        uint32_t rs[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t inc = val[p];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (wl >= o) inc = max(inc, t);
            }
            if (wl == 31) S.wmax[p][wp] = inc;
            uint32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
            if (wl == 0) ex = 0;
            rs[p] = ex;
        }
        if (__syncthreads_or(bad)) {
            bail = true;
            why = 2;
            break;
        }
        uint32_t lead_len[2] = {0, 0}, nbytes[2] = {0, 0}, ent[2] = {0, 0};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t r = max(rs[p], S.run_start[p]);
            for (int i = 0; i < wp; ++i) r = max(r, S.wmax[p][i]);
            rs[p] = r;  // first element of the zero run entering this lane (e0: none)
            if (!have) continue;
            const uint32_t E = e0 - r;
            ent[p] = E;
            uint8_t* row = S.rows + (size_t)(p * ST_LANES + tid) * ST_ROW;
            uint8_t tmp[ST_LEAD];
            uint32_t ll = 0;
            const bool full = q0[p] == 0 && !po[p].seen;
            if (q0[p] != 0) {
                if (E > 0) {
                    put_varint(tmp, (uint64_t)E << 2);
                    ll = (uint32_t)varint_len((uint64_t)E << 2);
                }
                {
                    const int q = q0[p];
                    const uint32_t v = ((((uint32_t)q << 1) ^ (uint32_t)(q >> 31)) << 2) | 1u;
                    const uint32_t len = 1u + (v >= 128u) + (v >= 16384u);
                    tmp[ll] = (uint8_t)((v & 0x7fu) | (len > 1u ? 0x80u : 0u));
                    if (len > 1u) tmp[ll + 1] = (uint8_t)(((v >> 7) & 0x7fu) | (len > 2u ? 0x80u : 0u));
                    if (len > 2u) tmp[ll + 2] = (uint8_t)(v >> 14);
                    ll += len;
                }
                if (po[p].seen && po[p].lz1 > 0) tmp[ll++] = (uint8_t)(po[p].lz1 << 2);
            } else if (!full) {
                const uint64_t v = (uint64_t)(E + 1u + (uint32_t)po[p].lz1) << 2;
                put_varint(tmp, v);
                ll = (uint32_t)varint_len(v);
            }
            for (uint32_t i = 0; i < ll; ++i) row[ST_LEAD - ll + i] = tmp[i];
            lead_len[p] = ll;
            uint32_t nb = ll + (uint32_t)po[p].body;
            // the plane's last lane closes the run still open
            if (final_iter && tid + 1 == active) {
                const uint32_t open_start = full ? r : val[p];
                const uint32_t open = e0 + SUB - open_start;
                if (open > 0) {
                    const uint64_t v = (uint64_t)open << 2;
                    put_varint(row + ST_LEAD + po[p].body, v);
                    nb += (uint32_t)varint_len(v);
                }
            }
            nbytes[p] = nb;
        }
        // exclusive sum-scan of the lanes' bytes (per plane)
        uint32_t bst[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t inc = nbytes[p];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (wl >= o) inc += t;
            }
            if (wl == 31) S.wbytes[p][wp] = inc;
            bst[p] = inc - nbytes[p];
        }
        // (the warps' sum units of the main pass ride on the same barrier: an
        // iteration without a sum event needs nothing more, step D)
        {
            uint64_t u = have ? uA : 0;
#pragma unroll
            for (int o = 16; o; o >>= 1) u = sat_add(u, __shfl_xor_sync(0xffffffffu, u, o));
            if (wl == 0) S.wunits[wp] = u;
        }
        __syncthreads();
        uint64_t bstart[2], obase[2];
        uint32_t iter_bytes[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t pre = 0, tot = 0;
            for (int i = 0; i < ST_WARPS; ++i) {
                if (i < wp) pre += S.wbytes[p][i];
                tot += S.wbytes[p][i];
            }
            iter_bytes[p] = tot;
            obase[p] = S.out_pos[p];
            bstart[p] = obase[p] + pre + bst[p];
        }
        // The token bytes leave the rows after the sum (step E): the rows are
        // packed into the plane's contiguous image first, in the input staging
        // buffer (dead by then), and stored with 16-byte words.  RAW keeps the
        // lane-by-lane stores here (its replays read X, the serial head the rows).
        constexpr bool LATE_COPY = !RAW;
        // copy the rows out, 32 consecutive bytes per store, and the side index
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (!LATE_COPY && nbytes[p] != 0u)
                stream_lane_copy(out[p] + bstart[p], S.rows + (size_t)(p * ST_LANES + tid) * ST_ROW + ST_LEAD - lead_len[p], nbytes[p]);
            if (have) {
                SideEntry se;
                if (q0[p] == 0) {
                    se.off = (uint32_t)bstart[p];
                    se.skip = ent[p];
                } else {
                    se.off = (uint32_t)bstart[p] + (ent[p] > 0 ? (uint32_t)varint_len((uint64_t)ent[p] << 2) : 0u);
                    se.skip = 0;
                }
                se.pred = __dmul_rn(td, (double)Mleft[p]);
                side[p][e0 / SUB] = se;
            }
        }
        // the carry is read above by every lane: update it behind a barrier
        // (the packing barrier of step E when the copy is late)
        auto carry_update = [&]() {
            if (tid + 1 == active) {
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const bool full = q0[p] == 0 && !po[p].seen;
                    S.run_start[p] = full ? rs[p] : val[p];
                    S.m_carry[p] = po[p].Mlast;
                    S.out_pos[p] += iter_bytes[p];
                }
            }
        };
        if (!LATE_COPY) {
            __syncthreads();
            carry_update();
        }

        // D. stored sum of squares: s plus the units of the lanes after
        // `owner` (uA, under the binade of s) plus `part` (the rest of owner's
        // own sub-chunk); hasB: uB holds the same lanes' units one binade up
        if (a.sumsq) {
            double s = s_in;
            long long k_after = -1;
            int owner = -1;
            uint64_t part = 0;
            bool hasB = have_tu;
            if (!have_tu) {
                // s is still 0: the first terms double it again and again; add
                // the first ST_SERIAL in the reference's order on one thread
                // (RAW: the rows are free, copied out above; else this slot's part of the split path's scratch X)
                double* tser = LATE_COPY ? const_cast<double*>(a.X) + 2 * slot * a.x_plane_stride : reinterpret_cast<double*>(S.rows);
                if (have && e0 < ST_SERIAL) walk(std::integral_constant<int, 2>{}, nullptr, 0.0, -1, tser, 0);
                __syncthreads();
                const int m = (int)umin64(ST_SERIAL, n - base);
                if (tid == 0) {
                    double acc = s;
#pragma unroll 4
                    for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, tser[k]);
                    S.ev_s = acc;
                }
                __syncthreads();
                s = S.ev_s;
                if (base != 0 || !(s > 0.0 && ilogb(s) >= -960)) {  // an all-zero or tiny head: the legacy kernel's cases
                    bail = true;
                    why = 3;
                    break;
                }
                owner = m / SUB - 1;
                uA = 0;
                if (have && tid > owner) walk(std::integral_constant<int, 1>{}, nullptr, ldexp(1.0, 52 - ilogb(s)), -1, nullptr, 0);
            }
            bool summed = false;
            if (have_tu) {  // the usual iteration: no event, the totals of step C are all it takes
                const double to_units = ldexp(1.0, 52 - ilogb(s));
                const uint64_t ms = (uint64_t)(s * to_units);
                uint64_t total = 0;
                for (int i = 0; i < ST_WARPS; ++i) total = sat_add(total, S.wunits[i]);
                if (ms + total < (1ull << 53)) {
                    s = (double)(ms + total) / to_units;
                    summed = true;
                }
            }
            while (!summed) {
                const double to_units = ldexp(1.0, 52 - ilogb(s));
                const uint64_t ms = (uint64_t)(s * to_units);
                const uint64_t mine = (have && tid > owner) ? uA : 0;
                uint64_t inc = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (wl >= o) inc = sat_add(inc, t);
                }
                uint64_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
                if (wl == 0) excl = 0;
                __syncthreads();  // (S.wunits / S.ev_* of the previous round are read)
                if (wl == 31) S.wunits[wp] = inc;
                if (tid == 0) S.ev_any = 0;
                __syncthreads();
                uint64_t total = part, pre = part;
                for (int i = 0; i < ST_WARPS; ++i) {
                    if (i < wp) pre = sat_add(pre, S.wunits[i]);
                    total = sat_add(total, S.wunits[i]);
                }
                if (ms + total < (1ull << 53)) {
                    s = (double)(ms + total) / to_units;
                    break;
                }
                // an event (binade crossing or tie) lies ahead: in the rest of
                // owner's sub-chunk, or in the first lane whose inclusive
                // prefix reaches the binade's end.  That lane walks to it.
                const uint64_t LIM = (1ull << 53) - ms;
                const bool in_part = part >= LIM;
                const uint64_t offx = sat_add(pre, excl);
                const bool me = in_part ? tid == owner : (have && tid > owner && offx < LIM && sat_add(offx, mine) >= LIM);
                if (me) {
                    ownB = (hasB && !in_part && uB < ST_SAT) ? uB : ST_SAT;
                    uA = in_part ? 0 : offx;
                    walk(std::integral_constant<int, 3>{}, nullptr, to_units, k_after, nullptr, ms);
                    S.ev_owner = tid;
                }
                __syncthreads();
                if (!S.ev_any) {  // cannot happen; never spin
                    bail = true;
                    why = 4;
                    break;
                }
                const double sn = S.ev_s;
                const int e_old = ilogb(s), e_new = (sn > 0.0) ? ilogb(sn) : -100000;
                if (!(sn > 0.0 && e_new >= -960 && e_new < 1000)) {
                    bail = true;
                    why = 4;
                    break;
                }
                owner = S.ev_owner;
                k_after = (long long)S.ev_k;
                part = S.ev_part;
                s = sn;
                if (e_new == e_old) {
                    // a tie inside the binade: the later lanes' units stand
                } else if (e_new == e_old + 1 && hasB) {
                    uA = uB;
                    hasB = false;
                } else {  // re-measure the later lanes under the new binade
                    hasB = false;
                    uA = 0;
                    if (have && tid > owner) walk(std::integral_constant<int, 1>{}, nullptr, ldexp(1.0, 52 - e_new), -1, nullptr, 0);
                }
            }
            if (tid == 0) S.s = s;
        }
        if (bail) break;
        // E. token bytes out
        if (LATE_COPY) {
            bool packed[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                packed[p] = iter_bytes[p] + 16u <= (uint32_t)ST_STAGE;  // uniform
                if (nbytes[p] != 0u) {
                    // the image keeps the destination's 16-byte phase
                    uint8_t* dst = packed[p] ? S.in[p] + (obase[p] & 15u) + (bstart[p] - obase[p]) : out[p] + bstart[p];
                    stream_lane_copy(dst, S.rows + (size_t)(p * ST_LANES + tid) * ST_ROW + ST_LEAD - lead_len[p], nbytes[p]);
                }
            }
            __syncthreads();
            carry_update();
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                if (!packed[p] || iter_bytes[p] == 0u) continue;
                const uint8_t* img = S.in[p] + (obase[p] & 15u);
                uint8_t* dst = out[p] + obase[p];
                const uint32_t nb = iter_bytes[p];
                const uint32_t hb = min(nb, (16u - (uint32_t)(obase[p] & 15u)) & 15u);
                const uint32_t n16 = (nb - hb) / 16u;
                const uint32_t tb = nb - hb - 16u * n16;
                if ((uint32_t)tid < hb) dst[tid] = img[tid];
                const uint4* s4 = reinterpret_cast<const uint4*>(img + hb);
                uint4* d4 = reinterpret_cast<uint4*>(dst + hb);
                for (uint32_t i = (uint32_t)tid; i < n16; i += ST_LANES) d4[i] = s4[i];
                if ((uint32_t)tid < tb) dst[hb + 16u * n16 + tid] = img[hb + 16u * n16 + tid];
            }
        }
        __syncthreads();

        // ladder early exit (k_fused's): a level before the last gives up once
        // theta is out of reach of the bytes already closed
        if (a.ladder_theta > 0.0 && !final_iter) {
            const uint64_t lb = 2 * HEADER_BYTES + S.out_pos[0] + S.out_pos[1];
            if ((double)(16 * n) / (double)lb < a.ladder_theta) {
                if (tid == 0) {
                    a.out_len[2 * gslot] = 1ull << 50;
                    a.out_len[2 * gslot + 1] = 1ull << 50;
                    if (a.counters) atomicAdd(&a.counters[15], 1ull);
                    redo[gslot] = 0;
                    if (dc.committed) dc.committed[gslot] = 0;
                }
                return;
            }
        }
    }
    __syncthreads();
    if (direct && !bail) {
        stream_commit(a, dc, slot, gslot, in_stride, S.out_pos[0], S.out_pos[1], a.sumsq ? S.s : 0.0,
                      reinterpret_cast<uint64_t*>(&S.ev_part), tid, ST_LANES);
    } else if (dc.committed && tid == 0) {
        dc.committed[gslot] = 0;
    }
    if (tid == 0) {
        if (bail) {
            redo[gslot] = 1;
            if (a.counters) {
                atomicAdd(&a.counters[17], 1ull);
                atomicAdd(&a.counters[19 + why], 1ull);
            }
        } else {
            redo[gslot] = 0;
            a.out_len[2 * gslot] = S.out_pos[0];
            a.out_len[2 * gslot + 1] = S.out_pos[1];
            if (a.sumsq) a.sumsq[gslot] = S.s;
            if (a.counters) atomicAdd(&a.counters[18], 1ull);
        }
    }
}

// one CTA per slot of the launch (a wave, or the whole gate in the small layout)
template <int ST_LANES, bool RAW>
__global__ void __launch_bounds__(ST_LANES, 512 / ST_LANES) k_stream(FusedArgs a, uint8_t* redo, StreamCommit dc)
{
    if (a.err && *a.err) return;
    const int b = a.order ? (int)(a.order[a.slot_base + blockIdx.x] - a.slot_base) : (int)blockIdx.x;
    const uint64_t gslot = a.slot_base + (uint64_t)b;
    if (a.pending && !a.pending[gslot]) return;
    extern __shared__ __align__(16) unsigned char smem[];
    StreamSharedT<ST_LANES>& S = *reinterpret_cast<StreamSharedT<ST_LANES>*>(smem);
    if (threadIdx.x == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
    }
    unsigned stage_phase[2] = {0, 0};
    stream_slot<ST_LANES, RAW>(a, redo, dc, (uint64_t)b, gslot, stage_phase);
}

// Persistent form (wave layout, single-level ladder): as many CTAs as staging
// slots, each taking the gate's slots one after the other from a queue — no
// waves, no kernel boundary between them, and the CTAs' end-of-stride copies
// fall at different times.  A CTA's staging slot is its own (blockIdx.x): free
// again once its stride is installed.  Slots already installed (a resumed
// gate) are skipped.
template <int ST_LANES>
__global__ void __launch_bounds__(ST_LANES, 512 / ST_LANES) k_stream_persist(FusedArgs a, uint8_t* redo, StreamCommit dc,
                                                                             uint64_t n_slots, unsigned long long* q_head)
{
    extern __shared__ __align__(16) unsigned char smem[];
    StreamSharedT<ST_LANES>& S = *reinterpret_cast<StreamSharedT<ST_LANES>*>(smem);
    __shared__ unsigned long long s_idx;
    if (threadIdx.x == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
    }
    unsigned stage_phase[2] = {0, 0};
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_idx = (a.err && *reinterpret_cast<const volatile int*>(a.err)) ? ~0ull : atomicAdd(q_head, 1ull);
        __syncthreads();
        const unsigned long long idx = s_idx;
        if (idx >= n_slots) break;
        const uint64_t gslot = a.order ? (uint64_t)a.order[idx] : (uint64_t)idx;
        if ((a.pending && !a.pending[gslot]) || dc.committed[gslot]) continue;
        stream_slot<ST_LANES, false>(a, redo, dc, (uint64_t)blockIdx.x, gslot, stage_phase);
    }
}

}  // namespace qcs
