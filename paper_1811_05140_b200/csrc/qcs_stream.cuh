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
// argument of fused_sumsq; an iteration holding a binade crossing or a tie
// replays the lanes after it (decode + gate + quantize again) under the new
// binade instead of re-reading stored values.
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
    uint32_t ev_k;
    int ev_any;
};
static_assert(sizeof(StreamSharedT<128>) <= 55 * 1024 + 768, "four 128-lane streaming CTAs per SM");
static_assert(sizeof(StreamSharedT<256>) <= 112 * 1024, "two 256-lane streaming CTAs per SM");
static_assert(sizeof(StreamSharedT<512>) <= 226 * 1024, "one 512-lane streaming CTA per SM");

// Sequential reader of one plane's token stream from a side-index entry
// (decode_sub's walk, one element per call).
struct TokReader {
    const uint8_t* in;
    uint64_t pos;
    uint64_t w;
    int avail;
    int codec;
    uint32_t skip;
    uint32_t zleft, wleft;
    double td, P;

    __device__ __forceinline__ void init(const uint8_t* in_, int codec_, double td_, SideEntry se)
    {
        in = in_;
        pos = se.off;
        w = 0;
        avail = 0;
        codec = codec_;
        skip = se.skip;
        zleft = wleft = 0;
        td = td_;
        P = se.pred;
    }
    __device__ __forceinline__ uint64_t varint()
    {
        if (avail < 5) {
            w = load8_at(in, pos);
            avail = 8;
        }
        const uint64_t stop = ~w & 0x8080808080808080ull;
        const int nb = stop ? (__ffsll((long long)stop) >> 3) : 9;
        if (nb <= 4 && nb <= avail) {
            const uint32_t x = (uint32_t)w & (0xffffffffu >> (8 * (4 - nb)));
            const uint32_t v = (x & 0x7fu) | ((x >> 1) & 0x3f80u) | ((x >> 2) & 0x1fc000u) | ((x >> 3) & 0xfe00000u);
            pos += nb;
            avail -= nb;
            w >>= 8 * nb;
            return v;
        }
        avail = 0;
        return get_varint(in, pos);
    }
    __device__ __forceinline__ double word()
    {
        const double x = __longlong_as_double((long long)load8_at(in, pos));
        pos += 8;
        avail = 0;
        return x;
    }
    // the next element's decoded value (before the stride scale)
    __device__ __forceinline__ double next()
    {
        if (zleft) {
            --zleft;
            return codec == 1 ? P : 0.0;
        }
        if (wleft) {
            --wleft;
            const double x = word();
            if (codec == 1) P = x;
            return x;
        }
        const uint64_t v = varint();
        if (codec == 1) {
            const unsigned tag = (unsigned)(v & 3u);
            const uint64_t arg = v >> 2;
            if (tag == 1) {
                P = __dadd_rn(P, __dmul_rn(td, (double)(int)unzigzag(arg)));
                return P;
            }
            const uint32_t left = (uint32_t)(arg - skip) - 1u;
            if (tag == 0) {
                zleft = left;
                skip = 0;
                return P;
            }
            pos += 8ull * skip;
            skip = 0;
            wleft = left;
            P = word();
            return P;
        }
        const uint64_t run = v >> 1;
        const uint32_t left = (uint32_t)(run - skip) - 1u;
        if ((v & 1u) == 0) {
            zleft = left;
            skip = 0;
            return 0.0;
        }
        pos += 8ull * skip;
        skip = 0;
        wleft = left;
        return word();
    }
};

// code token of q (|q| < 32768): 1..3 bytes at o, returns the length
__device__ __forceinline__ uint32_t put_code_token(uint8_t* o, int q)
{
    const uint32_t v = ((((uint32_t)q << 1) ^ (uint32_t)(q >> 31)) << 2) | 1u;
    const uint32_t len = 1u + (v >= 128u) + (v >= 16384u);
    o[0] = (uint8_t)((v & 0x7fu) | (len > 1u ? 0x80u : 0u));
    if (len > 1u) o[1] = (uint8_t)(((v >> 7) & 0x7fu) | (len > 2u ? 0x80u : 0u));
    if (len > 2u) o[2] = (uint8_t)(v >> 14);
    return len;
}

struct StreamPlaneOut {
    double M0, x0, Mlast;
    bool good0, seen, bad;
    int lz1, tz, body;
};

template <int ST_LANES>
__global__ void __launch_bounds__(ST_LANES, 512 / ST_LANES) k_stream(FusedArgs a, uint8_t* redo)
{
    using StreamShared = StreamSharedT<ST_LANES>;
    constexpr int ST_WARPS = StreamShared::ST_WARPS;
    constexpr int ST_STAGE = StreamShared::ST_STAGE;
    constexpr int ST_ITER = ST_LANES * SUB;  // elements per plane per iteration
    if (a.err && *a.err) return;
    const int b = a.order ? (int)(a.order[a.slot_base + blockIdx.x] - a.slot_base) : (int)blockIdx.x;
    const uint64_t slot = (uint64_t)b;
    const uint64_t gslot = a.slot_base + slot;
    if (a.pending && !a.pending[gslot]) return;
    const int tid = threadIdx.x, wl = tid & 31, wp = tid >> 5;
    if (a.zero_slot && a.zero_slot[gslot]) {
        for (int c = 0; c < 2; ++c) write_zero_plane<true>(a, slot, gslot, c, tid, ST_LANES);
        if (tid == 0) {
            if (a.sumsq) a.sumsq[gslot] = 0.0;
            redo[gslot] = 0;
        }
        return;
    }

    extern __shared__ __align__(16) unsigned char smem[];
    StreamShared& S = *reinterpret_cast<StreamShared*>(smem);
    const CodecParams cp = a.cp;
    const uint64_t n = a.n;
    const uint64_t in_stride = a.job_stride[gslot];
    const double scale = a.scale[in_stride];
    const bool sc = scale != 1.0;

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

    if (tid == 0) {
        S.out_pos[0] = S.out_pos[1] = 0;
        S.run_start[0] = S.run_start[1] = 0;
        S.m_carry[0] = S.m_carry[1] = 0;
        S.s = 0.0;
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
    }
    unsigned stage_phase[2] = {0, 0};
    bool bail = false;  // uniform over the CTA
    __syncthreads();

    for (uint64_t base = 0; base < n; base += ST_ITER) {
        const uint32_t e0 = (uint32_t)base + (uint32_t)tid * SUB;
        const bool have = e0 < n;  // (n is a multiple of SUB: a lane has 32 elements or none)
        const bool final_iter = base + ST_ITER >= n;
        const int active = (int)umin64(ST_LANES, (n - base) / SUB);
        const uint64_t sc0 = base / SUB;

        // A. stage this iteration's payload bytes of both planes (one TMA bulk copy each)
        const uint8_t* src[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const uint64_t lo = in_side[p][sc0].off & ~uint64_t(15);
            uint64_t hi;
            if (final_iter) {
                hi = a.p_len[2 * in_stride + p];
            } else {
                const SideEntry nx = in_side[p][sc0 + ST_LANES];
                hi = (uint64_t)nx.off + 10 + 8 * (uint64_t)nx.skip;
            }
            const uint64_t nb = hi > lo ? ((hi - lo + 15) & ~uint64_t(15)) : 0;
            src[p] = in_bytes[p];
            if (nb > 0 && nb <= ST_STAGE) {  // uniform over the CTA
                if (tid == 0) bulk_g2s(S.in[p], in_bytes[p] + lo, (unsigned)nb, &S.bar[p]);
                mbar_wait(&S.bar[p], stage_phase[p]);
                stage_phase[p] ^= 1u;
                src[p] = S.in[p] - lo;
            }
        }
        const double s_in = S.s;  // the running sum entering this iteration (uniform)
        const bool have_tu = s_in > 0.0 && ilogb(s_in) >= -960;
        const double tu_main = have_tu ? ldexp(1.0, 52 - ilogb(s_in)) : 0.0;

        // One walk over the lane's sub-chunk.  PASS 0: the main pass (tokens
        // into the staging rows, first-element facts into po, sum units under
        // tu for every element).  PASS 1: sum units under tu for the elements
        // after k_after only (replay).  PASS 2: the terms t_k of the elements
        // below ST_SERIAL into tdst (replay).  Returns the units.
        auto walk = [&](auto pass_tag, StreamPlaneOut* po, double tu, long long k_after, double* tdst) -> uint64_t {
            constexpr int PASS = decltype(pass_tag)::value;
            TokReader rd[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) rd[p].init(src[p], in_codec[p], in_td[p], in_side[p][e0 / SUB]);
            double Mprev[2] = {0.0, 0.0};
            int run[2] = {0, 0};
            uint8_t* rowp[2];
            if (PASS == 0) {
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    rowp[p] = S.rows + (size_t)(p * ST_LANES + tid) * ST_ROW + ST_LEAD;
                    po[p].seen = false;
                    po[p].lz1 = 0;
                    po[p].body = 0;
                }
            }
            uint64_t loc = 0;
            bool bad = false;
            for (int k = 0; k < SUB; ++k) {
                double xr = rd[0].next(), xi = rd[1].next();
                if (sc) {
                    xr = __dmul_rn(xr, scale);
                    xi = __dmul_rn(xi, scale);
                }
                // gate (run_plan_unit, gate.cpp:405-454), every element on its own
                const uint64_t gi = (uint64_t)e0 + (uint64_t)k;
                if (kind <= 1) {
                    if (!(a.local_ctl >= 0 && !((gi >> a.local_ctl) & 1))) {
                        const int sd = fixed_side >= 0 ? fixed_side : (int)((gi >> a.t) & 1);
                        // apply_pair with a zero partner, minus its exact-zero
                        // terms (they change a zero's sign at most: snapped)
                        const double ur = sd ? a.u[6] : a.u[0], ui = sd ? a.u[7] : a.u[1];
                        const double orr = __dsub_rn(__dmul_rn(ur, xr), __dmul_rn(ui, xi));
                        const double oi = __dadd_rn(__dmul_rn(ur, xi), __dmul_rn(ui, xr));
                        xr = orr;
                        xi = oi;
                    }
                } else if (kind == 2) {
                    if (gi == a.flip_off) {
                        xr = -xr;
                        xi = -xi;
                    }
                } else {
                    xr = __dsub_rn(mr2, xr);
                    xi = __dsub_rn(mi2, xi);
                }
                xr = snap(xr);
                xi = snap(xi);
                // quantize on the lattice anchored at 0
                double rv[2];
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const double x = p ? xi : xr;
                    const double y = __dmul_rn(x, cp.inv_td);
                    double M = rint(y);
                    const double fr = fabs(__dsub_rn(y, M));
                    bool good = fabs(y) < 1073741824.0 && fr < 0.5 - 1.9073486328125e-06;
                    if (k == 0) {
                        if (PASS == 0) {
                            po[p].M0 = M;
                            po[p].x0 = x;
                            po[p].good0 = good;
                        }
                    } else {
                        const double q = __dsub_rn(M, Mprev[p]);
                        good = good && fabs(q) <= 32766.0;
                        if (!good) {  // the reference step from the exact predictor
                            double P = __dadd_rn(0.0, __dmul_rn(cp.td, Mprev[p]));
                            const int32_t t = ref_step(cp, P, x);
                            M = __dadd_rn(Mprev[p], (double)t);
                            if (t == WCODE || !(fabs(M) < 1073741824.0) ||
                                !same_bits(__dadd_rn(0.0, __dmul_rn(cp.td, M)), P))
                                bad = true;
                        }
                        if (PASS == 0) {
                            const int qi = (int)__dsub_rn(M, Mprev[p]);
                            if (qi == 0) {
                                ++run[p];
                            } else {
                                if (!po[p].seen) {
                                    po[p].seen = true;
                                    po[p].lz1 = run[p];
                                } else if (run[p] > 0) {
                                    rowp[p][po[p].body++] = (uint8_t)(run[p] << 2);  // zero run < 32: one byte
                                }
                                po[p].body += (int)put_code_token(rowp[p] + po[p].body, qi);
                                run[p] = 0;
                            }
                        }
                    }
                    Mprev[p] = M;
                    rv[p] = __dadd_rn(0.0, __dmul_rn(cp.td, M));
                }
                const double t = __dadd_rn(__dmul_rn(rv[0], rv[0]), __dmul_rn(rv[1], rv[1]));
                if (PASS == 2) {
                    if (gi < ST_SERIAL) tdst[gi] = t;
                } else if ((long long)gi > k_after) {
                    loc = sat_add(loc, sq_units_y(t * tu));
                }
            }
            if (PASS == 0) {
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    po[p].Mlast = Mprev[p];
                    po[p].tz = run[p];
                    if (!po[p].seen) po[p].lz1 = SUB - 1;
                }
                po[0].bad = bad;
            }
            return loc;
        };

        // B. main pass
        StreamPlaneOut po[2];
        po[0].bad = false;
        uint64_t loc = 0;
        if (have) loc = walk(std::integral_constant<int, 0>{}, po, tu_main, have_tu ? -1ll : (long long)n, nullptr);
        if (have) {
            S.mlast[0][tid] = (int)po[0].Mlast;
            S.mlast[1][tid] = (int)po[1].Mlast;
        }
        if (__syncthreads_or(have && po[0].bad)) {
            bail = true;
            break;
        }

        // C. first elements, runs across lanes, lead tokens, byte offsets
        uint32_t val[2] = {0, 0};     // start of the lane's trailing zero run, 0: the lane is one zero run
        int q0[2] = {0, 0};
        double Mleft[2] = {0.0, 0.0};
        bool bad = false;
        if (have) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                Mleft[p] = (double)(tid > 0 ? S.mlast[p][tid - 1] : S.m_carry[p]);
                const double q = __dsub_rn(po[p].M0, Mleft[p]);
                if (po[p].good0 && fabs(q) <= 32766.0) {
                    q0[p] = (int)q;
                } else {  // the reference step; must agree with the lattice point the lane continued from
                    double P = __dadd_rn(0.0, __dmul_rn(cp.td, Mleft[p]));
                    const int32_t t = ref_step(cp, P, po[p].x0);
                    if (t == WCODE || !same_bits(__dadd_rn(Mleft[p], (double)t), po[p].M0) ||
                        !(fabs(po[p].M0) < 1073741824.0) ||
                        !same_bits(__dadd_rn(0.0, __dmul_rn(cp.td, po[p].M0)), P))
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
                ll += put_code_token(tmp + ll, q0[p]);
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
        // (the units of the sum ride on the same barrier)
        {
            uint64_t u = loc;
#pragma unroll
            for (int o = 16; o; o >>= 1) u = sat_add(u, __shfl_xor_sync(0xffffffffu, u, o));
            if (wl == 0) S.wunits[wp] = u;
        }
        __syncthreads();
        uint64_t bstart[2];
        uint32_t iter_bytes[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t pre = 0, tot = 0;
            for (int i = 0; i < ST_WARPS; ++i) {
                if (i < wp) pre += S.wbytes[p][i];
                tot += S.wbytes[p][i];
            }
            iter_bytes[p] = tot;
            bstart[p] = S.out_pos[p] + pre + bst[p];
        }
        // copy the rows out, 32 consecutive bytes per store, and the side index
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const uint32_t my_nb = nbytes[p];
            const uint32_t my_lead = lead_len[p];
            for (unsigned todo = __ballot_sync(0xffffffffu, my_nb != 0u); todo; todo &= todo - 1u) {
                const int j = __ffs(todo) - 1;
                const uint32_t nb = __shfl_sync(0xffffffffu, my_nb, j);
                const uint32_t ld = __shfl_sync(0xffffffffu, my_lead, j);
                const uint64_t bs = __shfl_sync(0xffffffffu, bstart[p], j);
                const uint8_t* srow = S.rows + (size_t)(p * ST_LANES + (tid & ~31) + j) * ST_ROW + ST_LEAD - ld;
                uint8_t* dst = out[p] + bs;
                if (nb <= 64u) {
                    const uint8_t b0 = wl < nb ? srow[wl] : (uint8_t)0;
                    const uint8_t b1 = wl + 32u < nb ? srow[wl + 32u] : (uint8_t)0;
                    if (wl < nb) dst[wl] = b0;
                    if (wl + 32u < nb) dst[wl + 32u] = b1;
                } else {
                    for (uint32_t k = wl; k < nb; k += 32) dst[k] = srow[k];
                }
            }
            if (have) {
                SideEntry se;
                if (q0[p] == 0) {
                    se.off = (uint32_t)bstart[p];
                    se.skip = ent[p];
                } else {
                    se.off = (uint32_t)bstart[p] + (ent[p] > 0 ? (uint32_t)varint_len((uint64_t)ent[p] << 2) : 0u);
                    se.skip = 0;
                }
                se.pred = __dadd_rn(0.0, __dmul_rn(cp.td, Mleft[p]));
                side[p][e0 / SUB] = se;
            }
        }
        // the carry is read above by every lane: update it behind a barrier
        __syncthreads();
        if (tid + 1 == active) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const bool full = q0[p] == 0 && !po[p].seen;
                S.run_start[p] = full ? rs[p] : val[p];
                S.m_carry[p] = (int)po[p].Mlast;
                S.out_pos[p] += iter_bytes[p];
            }
        }

        // D. stored sum of squares
        if (a.sumsq) {
            double s = s_in;
            long long k_after = -1;  // elements up to here are in s
            double* tser = reinterpret_cast<double*>(S.rows);  // (the rows are free: copied out above)
            if (!have_tu) {
                // s is still 0: the first terms double it again and again; add
                // the first ST_SERIAL in the reference's order on one thread
                __syncthreads();
                if (have && e0 < ST_SERIAL) walk(std::integral_constant<int, 2>{}, nullptr, 0.0, -1, tser);
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
                k_after = (long long)base + m - 1;
                if (base != 0 || !(s > 0.0 && ilogb(s) >= -960)) {  // an all-zero or tiny head: the legacy kernel's cases
                    bail = true;
                    break;
                }
                loc = 0;
                if (have && (long long)e0 + SUB - 1 > k_after)
                    loc = walk(std::integral_constant<int, 1>{}, nullptr, ldexp(1.0, 52 - ilogb(s)), k_after, nullptr);
                uint64_t u = loc;
#pragma unroll
                for (int o = 16; o; o >>= 1) u = sat_add(u, __shfl_xor_sync(0xffffffffu, u, o));
                __syncthreads();
                if (wl == 0) S.wunits[wp] = u;
                __syncthreads();
            }
            for (;;) {
                const int e = ilogb(s);
                const double to_units = ldexp(1.0, 52 - e);
                const uint64_t ms = (uint64_t)(s * to_units);
                uint64_t total = 0, pre = 0;
                for (int i = 0; i < ST_WARPS; ++i) {
                    if (i < wp) pre = sat_add(pre, S.wunits[i]);
                    total = sat_add(total, S.wunits[i]);
                }
                if (ms + total < (1ull << 53)) {
                    s = (double)(ms + total) / to_units;
                    break;
                }
                // an event (binade crossing or tie) lies in this iteration: the
                // lane whose inclusive prefix reaches the binade's end walks to
                // it and adds it exactly; everything after it is re-measured
                uint64_t inc = loc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (wl >= o) inc = sat_add(inc, t);
                }
                const uint64_t LIM = (1ull << 53) - ms;
                if (tid == 0) S.ev_any = 0;
                __syncthreads();
                uint64_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
                if (wl == 0) excl = 0;
                const uint64_t offx = sat_add(pre, excl);
                if (have && offx < LIM && sat_add(offx, loc) >= LIM) {
                    // replay this lane's terms up to the event
                    TokReader rd[2];
#pragma unroll
                    for (int p = 0; p < 2; ++p) rd[p].init(src[p], in_codec[p], in_td[p], in_side[p][e0 / SUB]);
                    double Mprev[2] = {0.0, 0.0};
                    uint64_t acc = offx;
                    for (int k = 0; k < SUB; ++k) {
                        double xr = rd[0].next(), xi = rd[1].next();
                        if (sc) {
                            xr = __dmul_rn(xr, scale);
                            xi = __dmul_rn(xi, scale);
                        }
                        const uint64_t gi = (uint64_t)e0 + (uint64_t)k;
                        if (kind <= 1) {
                            if (!(a.local_ctl >= 0 && !((gi >> a.local_ctl) & 1))) {
                                const int sd = fixed_side >= 0 ? fixed_side : (int)((gi >> a.t) & 1);
                                const double ur = sd ? a.u[6] : a.u[0], ui = sd ? a.u[7] : a.u[1];
                                const double orr = __dsub_rn(__dmul_rn(ur, xr), __dmul_rn(ui, xi));
                                const double oi = __dadd_rn(__dmul_rn(ur, xi), __dmul_rn(ui, xr));
                                xr = orr;
                                xi = oi;
                            }
                        } else if (kind == 2) {
                            if (gi == a.flip_off) {
                                xr = -xr;
                                xi = -xi;
                            }
                        } else {
                            xr = __dsub_rn(mr2, xr);
                            xi = __dsub_rn(mi2, xi);
                        }
                        xr = snap(xr);
                        xi = snap(xi);
                        double rv[2];
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            const double x = p ? xi : xr;
                            const double y = __dmul_rn(x, cp.inv_td);
                            double M = rint(y);
                            if (k > 0) {
                                const double fr = fabs(__dsub_rn(y, M));
                                const double q = __dsub_rn(M, Mprev[p]);
                                if (!(fabs(y) < 1073741824.0 && fr < 0.5 - 1.9073486328125e-06 && fabs(q) <= 32766.0)) {
                                    double P = __dadd_rn(0.0, __dmul_rn(cp.td, Mprev[p]));
                                    const int32_t t = ref_step(cp, P, x);
                                    M = __dadd_rn(Mprev[p], (double)t);
                                }
                            }
                            Mprev[p] = M;
                            rv[p] = __dadd_rn(0.0, __dmul_rn(cp.td, M));
                        }
                        if ((long long)gi <= k_after) continue;
                        const double t = __dadd_rn(__dmul_rn(rv[0], rv[0]), __dmul_rn(rv[1], rv[1]));
                        const double y = t * to_units;
                        const double ry = rint(y);
                        const bool beyond = y >= 9007199254740992.0;
                        const bool tie = !beyond && fabs(y - ry) == 0.5;
                        const uint64_t c = beyond ? (1ull << 53) : (uint64_t)ry;
                        if (beyond || tie || ms + acc + c >= (1ull << 53)) {
                            S.ev_s = __dadd_rn((double)(ms + acc) / to_units, t);
                            S.ev_k = (uint32_t)gi;
                            S.ev_any = 1;
                            if (a.counters) atomicAdd(&a.counters[tie ? 6 : 7], 1ull);
                            break;
                        }
                        acc += c;
                    }
                }
                __syncthreads();
                if (!S.ev_any) {  // cannot happen; never spin
                    bail = true;
                    break;
                }
                s = S.ev_s;
                k_after = (long long)S.ev_k;
                if (!(s > 0.0 && ilogb(s) >= -960)) {
                    bail = true;
                    break;
                }
                loc = 0;
                if (have && (long long)e0 + SUB - 1 > k_after)
                    loc = walk(std::integral_constant<int, 1>{}, nullptr, ldexp(1.0, 52 - ilogb(s)), k_after, nullptr);
                uint64_t u = loc;
#pragma unroll
                for (int o = 16; o; o >>= 1) u = sat_add(u, __shfl_xor_sync(0xffffffffu, u, o));
                __syncthreads();
                if (wl == 0) S.wunits[wp] = u;
                __syncthreads();
            }
            if (tid == 0) S.s = s;
        }
        __syncthreads();
        if (bail) break;

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
                }
                return;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (bail) {
            redo[gslot] = 1;
            if (a.counters) atomicAdd(&a.counters[17], 1ull);
        } else {
            redo[gslot] = 0;
            a.out_len[2 * gslot] = S.out_pos[0];
            a.out_len[2 * gslot + 1] = S.out_pos[1];
            if (a.sumsq) a.sumsq[gslot] = S.s;
            if (a.counters) atomicAdd(&a.counters[18], 1ull);
        }
    }
}

}  // namespace qcs
