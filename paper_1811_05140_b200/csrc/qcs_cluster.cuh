// Sharded state driven by ONE host process, included at the
// end of qcs_engine.cu (it drives the shards' engine states directly).
//
// Rank = the top g qubits of the amplitude index (the top g bits of the stride
// index); rank r holds its 2^(n-g-s) strides in an ordinary engine state of
// n-g qubits on devices[r].  The reference has no distribution;
// the driver reproduces its single-process semantics bit for bit:
//   * gates on local qubits run unchanged on every shard; a control on a rank
//     qubit turns into "this shard applies the uncontrolled gate or nothing"
//     (make_stride_plan's control-bit skip, gate.cpp:351-379);
//   * a target on a rank qubit: a lazy qubit permutation over the stride bits
//     swaps that rank bit with a local stride bit (the local qubit needed
//     furthest in the future is evicted, Belady over the program): partner
//     shards exchange half their strides as device stride images
//     (qcs_pack_strides_range / qcs_unpack_strides: blocks verbatim, side
//     index, scale, sum) with grouped ncclSend/ncclRecv over NVLink, or a
//     device copy (loopback backend: several shards on one GPU, for tests) --
//     and the permutation stays;
//   * per gate, on the device and without a host round trip: the shards'
//     (scale, sum_sq) tables and stride reports are gathered to shard 0's
//     device, one kernel folds the lazy renormalisation (aalc.cpp:410-419)
//     and the GateRecord (aalc.cpp:612-631) in LOGICAL global stride / unit
//     order through a device copy of the permutation, and every shard scales
//     by the factor from device memory; reflect_mean's mean (aalc.cpp:270-295)
//     is folded the same way before the gate.
// One host synchronisation per qcs_cluster_run_program call (plus the rare
// exchanges).  NCCL is loaded at run time (dlopen libnccl.so.2) only by the
// NCCL backend.
#include <dlfcn.h>

#include <nccl.h>

namespace {

// ---- NCCL, resolved at run time -------------------------------------------
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string& why)
    {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            why = "cannot load libnccl.so.2";
            return false;
        }
#define QCS_SYM(f)                                                   \
    f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f));          \
    if (!f) {                                                        \
        why = "libnccl lacks nccl" #f;                               \
        return false;                                                \
    }
        QCS_SYM(CommInitAll)
        QCS_SYM(CommDestroy)
        QCS_SYM(GroupStart)
        QCS_SYM(GroupEnd)
        QCS_SYM(Send)
        QCS_SYM(Recv)
        QCS_SYM(GetErrorString)
#undef QCS_SYM
        return true;
    }
};
NcclApi g_nccl;

// ---- device folds ------------------------------------------------------------
constexpr int FOLD_THREADS = 256;
constexpr int FOLD_CHUNK = 2048;

// Gathered report i -> its position in the reference's global unit order
// (ascending logical lo stride, a pair unit's lo before its hi): slot
// 2*lo + hi of a dense table (empty entries are -1).
__global__ void k_cluster_scatter(const qcs_stride_report* rep, const uint64_t* p2l, uint64_t base, uint64_t count,
                                  uint64_t phys0, uint64_t pbit, int64_t* pos_map)
{
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint64_t lg = p2l[phys0 + rep[base + i].stride_index];
    const uint64_t key = pbit ? 2 * (lg & ~pbit) + ((lg & pbit) ? 1 : 0) : 2 * lg;
    pos_map[key] = (int64_t)(base + i);
}

// mode 0: reflect_mean's mean from the gathered per-stride sums (partial
// [2*phys]), serial in logical order (aalc.cpp:292-294), into out[1..2].
// mode 1: lazy renormalisation + re-measure in logical order (aalc.cpp:410-419)
// into out[0] (f) and out[3] (norm_sq), and the GateRecord of the reports
// (pos_map, reset to -1 as it is read) into *rec.
__global__ void __launch_bounds__(FOLD_THREADS) k_cluster_fold(int mode, uint64_t NS, int n_qubits, const uint64_t* l2p,
                                                              const double* scale, const double* sum,
                                                              const double* partial, const qcs_stride_report* rep,
                                                              int64_t* pos_map, const uint64_t* cin, int R,
                                                              double* out, qcs_gate_record* rec, uint64_t gate_index)
{
    __shared__ double sh_a[FOLD_CHUNK], sh_b[FOLD_CHUNK];
    __shared__ double sh_f;
    __shared__ int sh_do;
    const int tid = threadIdx.x;
    if (mode == 0) {
        double sr = 0.0, si = 0.0;
        for (uint64_t c0 = 0; c0 < NS; c0 += FOLD_CHUNK) {
            const int m = (int)umin64(FOLD_CHUNK, NS - c0);
            __syncthreads();
            for (int i = tid; i < m; i += FOLD_THREADS) {
                const uint64_t ph = l2p[c0 + i];
                sh_a[i] = partial[2 * ph];
                sh_b[i] = partial[2 * ph + 1];
            }
            __syncthreads();
            if (tid == 0)
                for (int i = 0; i < m; ++i) {
                    sr = __dadd_rn(sr, sh_a[i]);
                    si = __dadd_rn(si, sh_b[i]);
                }
        }
        if (tid == 0) {
            const double na = (double)(1ull << n_qubits);
            out[1] = __ddiv_rn(sr, na);
            out[2] = __ddiv_rn(si, na);
        }
        return;
    }
    auto fold = [&](double f, bool by_f) {
        double total = 0.0;
        for (uint64_t c0 = 0; c0 < NS; c0 += FOLD_CHUNK) {
            const int m = (int)umin64(FOLD_CHUNK, NS - c0);
            __syncthreads();
            for (int i = tid; i < m; i += FOLD_THREADS) {
                const uint64_t ph = l2p[c0 + i];
                const double a = by_f ? __dmul_rn(scale[ph], f) : scale[ph];
                sh_a[i] = __dmul_rn(__dmul_rn(a, a), sum[ph]);
            }
            __syncthreads();
            if (tid == 0)
                for (int i = 0; i < m; ++i) total = __dadd_rn(total, sh_a[i]);
        }
        return total;
    };
    const double total = fold(1.0, false);
    if (tid == 0) {
        sh_do = total > 0.0;
        sh_f = sh_do ? __ddiv_rn(1.0, __dsqrt_rn(total)) : 1.0;
    }
    __syncthreads();
    const double f = sh_f;
    const double nsq = fold(f, sh_do != 0);
    if (tid == 0) {
        out[0] = f;
        out[3] = nsq;
    }
    // GateRecord: reports in global unit order (2*NS dense positions)
    qcs_gate_record r;
    r.min_ratio = INFINITY;
    r.max_chosen_delta = 0.0;
    double rs = 0.0;
    uint64_t b_in = 0, b_out = 0, viol = 0, cnt = 0;
    for (uint64_t c0 = 0; c0 < 2 * NS; c0 += FOLD_CHUNK) {
        const int m = (int)umin64(FOLD_CHUNK, 2 * NS - c0);
        __syncthreads();
        for (int i = tid; i < m; i += FOLD_THREADS) {
            const int64_t k = pos_map[c0 + i];
            sh_b[i] = k >= 0 ? 1.0 : 0.0;
            if (k >= 0) {
                pos_map[c0 + i] = -1;
                const qcs_stride_report& q = rep[k];
                sh_a[i] = q.ratio;
                r.min_ratio = fmin(r.min_ratio, q.ratio);
                r.max_chosen_delta = fmax(r.max_chosen_delta, q.chosen_delta);
                b_in += q.bytes_in;
                b_out += q.bytes_out;
                viol += q.threshold_met ? 0 : 1;
                ++cnt;
            }
        }
        __syncthreads();
        if (tid == 0)
            for (int i = 0; i < m; ++i)
                if (sh_b[i] != 0.0) rs = __dadd_rn(rs, sh_a[i]);
    }
    __shared__ double red_min[FOLD_THREADS / 32], red_max[FOLD_THREADS / 32];
    __shared__ uint64_t red_in[FOLD_THREADS / 32], red_out[FOLD_THREADS / 32], red_v[FOLD_THREADS / 32],
        red_c[FOLD_THREADS / 32];
    for (int o = 16; o; o >>= 1) {
        r.min_ratio = fmin(r.min_ratio, __shfl_xor_sync(0xffffffffu, r.min_ratio, o));
        r.max_chosen_delta = fmax(r.max_chosen_delta, __shfl_xor_sync(0xffffffffu, r.max_chosen_delta, o));
        b_in += __shfl_xor_sync(0xffffffffu, b_in, o);
        b_out += __shfl_xor_sync(0xffffffffu, b_out, o);
        viol += __shfl_xor_sync(0xffffffffu, viol, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    const int w = tid >> 5;
    if ((tid & 31) == 0) {
        red_min[w] = r.min_ratio;
        red_max[w] = r.max_chosen_delta;
        red_in[w] = b_in;
        red_out[w] = b_out;
        red_v[w] = viol;
        red_c[w] = cnt;
    }
    __syncthreads();
    if (tid != 0 || !rec) return;
    r.min_ratio = INFINITY;
    r.max_chosen_delta = 0.0;
    r.bytes_before = r.bytes_after = r.threshold_violations = 0;
    uint64_t n_rep = 0;
    for (int i = 0; i < FOLD_THREADS / 32; ++i) {
        r.min_ratio = fmin(r.min_ratio, red_min[i]);
        r.max_chosen_delta = fmax(r.max_chosen_delta, red_max[i]);
        r.bytes_before += red_in[i];
        r.bytes_after += red_out[i];
        r.threshold_violations += red_v[i];
        n_rep += red_c[i];
    }
    r.gate_index = gate_index;
    r.stride_count = n_rep;
    r.mean_ratio = n_rep ? __ddiv_rn(rs, (double)n_rep) : 0.0;
    r.elapsed_ns = 0;
    r.norm_after = __dsqrt_rn(nsq);
    uint64_t ci = 0;
    for (int k = 0; k < R; ++k) ci += cin[k];
    r.compressed_in = ci;
    *rec = r;
}

__global__ void k_scale_all_dev(double* scale, uint64_t ns, const double* f)
{
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j < ns) scale[j] = __dmul_rn(scale[j], *f);
}

__global__ void k_copy_gate_cin(const Dev d, uint64_t* dst, int ran) { *dst = ran ? d.sc->gate_cin : 0; }
__global__ void k_put_mean(Dev d, const double* m)
{
    d.sc->mean[0] = m[1];
    d.sc->mean[1] = m[2];
}

}  // namespace

struct qcs_cluster {
    int n = 0, s = 0, g = 0, R = 1, backend = 0;
    uint64_t NS = 0, nsl = 0, L = 0;
    std::vector<qcs_dev_state*> sh;
    std::vector<int> dev;
    // lazy permutation of the stride-index bits: logical bit p at physical pi[p]
    std::vector<int> pi, inv;
    std::vector<int64_t> last_use;
    std::vector<std::vector<uint64_t>> next_target;
    bool sched = false;
    // fold side, on shard 0's device and stream
    double *g_scale = nullptr, *g_sum = nullptr, *g_partial = nullptr, *fold_out = nullptr;
    qcs_stride_report* g_rep = nullptr;
    int64_t* pos_map = nullptr;
    uint64_t *l2p = nullptr, *p2l = nullptr, *g_cin = nullptr;
    qcs_gate_record* rec = nullptr;
    uint64_t rec_cap = 0;
    std::vector<double*> f_sh;       // fold_out mirrored on every shard's device
    std::vector<cudaEvent_t> ev_sh;  // shard r's gate done
    cudaEvent_t ev_fold = nullptr;
    std::vector<void*> allocs;       // fold-side allocations (device 0) and per-shard mirrors
    std::vector<int> alloc_dev;
    // exchanges
    std::vector<uint8_t*> img_send, img_recv;
    uint64_t img_cap = 0;
    uint64_t exchanges = 0, exchange_bytes = 0;
    double exchange_ns = 0.0;
    std::vector<ncclComm_t> comms;
};

namespace {

int cl_alloc(qcs_cluster* c, int device, void** p, size_t bytes)
{
    cudaSetDevice(device);
    if (cudaMalloc(p, std::max<size_t>(bytes, 16)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(QCS_E_NOMEM, "cluster: cudaMalloc(%zu) failed", bytes);
    }
    c->allocs.push_back(*p);
    c->alloc_dev.push_back(device);
    return 0;
}

// physical global stride -> logical, and back, from the permutation
void cl_tables(const qcs_cluster* c, std::vector<uint64_t>& l2p, std::vector<uint64_t>& p2l)
{
    const int nb = c->n - c->s;
    l2p.assign(c->NS, 0);
    p2l.assign(c->NS, 0);
    for (uint64_t jl = 0; jl < c->NS; ++jl) {
        uint64_t jp = 0;
        for (int p = 0; p < nb; ++p) jp |= ((jl >> p) & 1ull) << c->pi[p];
        l2p[jl] = jp;
        p2l[jp] = jl;
    }
}

int cl_upload_tables(qcs_cluster* c)
{
    std::vector<uint64_t> l2p, p2l;
    cl_tables(c, l2p, p2l);
    cudaSetDevice(c->dev[0]);
    CU(cudaMemcpy(c->l2p, l2p.data(), 8 * c->NS, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->p2l, p2l.data(), 8 * c->NS, cudaMemcpyHostToDevice));
    return 0;
}

int cl_sync_all(qcs_cluster* c)
{
    for (int r = 0; r < c->R; ++r) {
        cudaSetDevice(c->dev[r]);
        CU(cudaStreamSynchronize(c->sh[r]->stream));
    }
    return 0;
}

// Swap rank bit b with local stride bit qb: partner shards r, r ^ 2^b exchange
// the strides whose local bit qb differs from their own rank bit; received
// stride j lands at j ^ 2^qb.  Streamed in chunks (the same count on every
// shard) so the images stay below img_cap.
int cl_swap(qcs_cluster* c, int b, int qb)
{
    const auto t0 = std::chrono::steady_clock::now();
    int rc = cl_sync_all(c);
    if (rc) return rc;
    const uint64_t half = c->nsl / 2;
    uint64_t k = half;
    for (int r = 0; r < c->R; ++r) {
        const int send_bit = ((r >> b) & 1) ? 0 : 1;
        uint64_t all = 0;
        rc = qcs_pack_strides_range(c->sh[r], qb, send_bit, 0, UINT64_MAX, nullptr, 0, &all);
        if (rc) return rc;
        const uint64_t per = std::max<uint64_t>(1, all / std::max<uint64_t>(1, half)) + 256;
        k = std::min<uint64_t>(k, std::max<uint64_t>(1, (c->img_cap - 4096) / per));
    }
    std::vector<uint64_t> len(c->R);
    for (uint64_t first = 0; first < half; first += k) {
        for (int r = 0; r < c->R; ++r) {
            const int send_bit = ((r >> b) & 1) ? 0 : 1;
            rc = qcs_pack_strides_range(c->sh[r], qb, send_bit, first, k, c->img_send[r], c->img_cap, &len[r]);
            if (rc) return rc;
            c->exchange_bytes += len[r];
        }
        if (c->backend == 1) {
            if (g_nccl.GroupStart() != ncclSuccess) return set_err(QCS_E_RUNTIME, "ncclGroupStart failed");
            for (int r = 0; r < c->R; ++r) {
                const int peer = r ^ (1 << b);
                cudaSetDevice(c->dev[r]);
                g_nccl.Send(c->img_send[r], len[r], ncclUint8, peer, c->comms[r], c->sh[r]->stream);
                g_nccl.Recv(c->img_recv[r], len[peer], ncclUint8, peer, c->comms[r], c->sh[r]->stream);
            }
            const ncclResult_t e = g_nccl.GroupEnd();
            if (e != ncclSuccess) return set_err(QCS_E_RUNTIME, "NCCL exchange failed: %s", g_nccl.GetErrorString(e));
        } else {  // loopback: device (or peer) copies between the shards' buffers
            for (int r = 0; r < c->R; ++r) {
                const int peer = r ^ (1 << b);
                cudaSetDevice(c->dev[r]);
                CU(cudaMemcpyPeerAsync(c->img_recv[r], c->dev[r], c->img_send[peer], c->dev[peer], len[peer],
                                       c->sh[r]->stream));
            }
        }
        rc = cl_sync_all(c);
        if (rc) return rc;
        for (int r = 0; r < c->R; ++r) {
            const int peer = r ^ (1 << b);
            rc = qcs_unpack_strides(c->sh[r], c->img_recv[r], len[peer], 1ull << qb);
            if (rc) return rc;
        }
    }
    ++c->exchanges;
    c->exchange_ns += (double)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    return 0;
}

uint64_t cl_next_use(const qcs_cluster* c, int p, uint64_t index)
{
    const auto& u = c->next_target[p];
    const auto it = std::upper_bound(u.begin(), u.end(), index);
    return it == u.end() ? (1ull << 62) : *it;
}

// physical local position of logical stride bit p (swapping it in from a rank
// bit if needed; `keep` is never evicted)
int cl_make_local(qcs_cluster* c, int p, int keep, uint64_t index, int* out)
{
    const int nloc = (c->n - c->g) - c->s;
    const int q = c->pi[p];
    if (q < nloc) {
        *out = q;
        return 0;
    }
    int v = -1;
    // (when the control holds the only local stride bit it is evicted: it becomes
    // a rank bit, and a control on a rank bit is the rank-level skip)
    if (nloc == 1) keep = -1;
    for (int cand = 0; cand < nloc; ++cand) {
        if (cand == keep) continue;
        if (v < 0) {
            v = cand;
            continue;
        }
        if (c->sched) {
            const uint64_t a = cl_next_use(c, c->inv[cand], index), bb = cl_next_use(c, c->inv[v], index);
            if (a > bb) v = cand;  // furthest next use; ties keep the lower position
        } else if (c->last_use[c->inv[cand]] < c->last_use[c->inv[v]]) {
            v = cand;
        }
    }
    if (v < 0) return set_err(QCS_E_INVALID, "cluster: no local stride bit");
    int rc = cl_swap(c, q - nloc, v);
    if (rc) return rc;
    const int pv = c->inv[v];
    c->pi[p] = v;
    c->pi[pv] = q;
    c->inv[v] = p;
    c->inv[q] = pv;
    rc = cl_upload_tables(c);
    if (rc) return rc;
    *out = v;
    return 0;
}

// One gate on every shard plus its device-side fold; no host synchronisation
// (exchanges aside).  The record lands in c->rec[rec_index].
int cl_enqueue_gate(qcs_cluster* c, const qcs_gate_desc* gate, const double* lad, int nl, double theta,
                    uint64_t rec_index, uint64_t gate_index)
{
    const int Q = c->n - c->g, s = c->s, nloc = Q - s;
    std::vector<qcs_gate_desc> local(c->R, *gate);
    std::vector<bool> part(c->R, true);
    uint64_t pbit = 0;
    if (gate->kind == 0 || gate->kind == 1) {
        const int t = gate->target, ctl = gate->kind == 1 ? gate->control : -1;
        int ctl_phys = (ctl >= s) ? c->pi[ctl - s] : -1;
        int lt = t;
        if (t >= s) {
            pbit = 1ull << (t - s);
            int pos = 0;
            const int rc = cl_make_local(c, t - s, (ctl_phys >= 0 && ctl_phys < nloc) ? ctl_phys : -1, gate_index, &pos);
            if (rc) return rc;
            lt = s + pos;
            c->last_use[t - s] = (int64_t)gate_index;
            if (ctl >= s) ctl_phys = c->pi[ctl - s];
        }
        for (int r = 0; r < c->R; ++r) {
            local[r].target = lt;
            if (ctl >= s) {
                if (ctl_phys >= nloc) {  // control on a rank bit: the uncontrolled gate, or nothing
                    part[r] = ((r >> (ctl_phys - nloc)) & 1) != 0;
                    local[r].kind = 0;
                    local[r].control = -1;
                } else {
                    local[r].control = s + ctl_phys;
                }
            }
        }
        if (ctl >= s) c->last_use[ctl - s] = (int64_t)gate_index;
    } else if (gate->kind == 2) {
        uint64_t jp = 0;
        const uint64_t jl = gate->flip_index >> s;
        for (int p = 0; p < c->n - s; ++p) jp |= ((jl >> p) & 1ull) << c->pi[p];
        for (int r = 0; r < c->R; ++r) {
            part[r] = (int)(jp >> nloc) == r;
            local[r].flip_index = ((jp & ((1ull << nloc) - 1)) << s) | (gate->flip_index & (c->L - 1));
        }
    }
    const int d0 = c->dev[0];
    cudaStream_t fs = c->sh[0]->stream;
    const double* given = nullptr;
    if (gate->kind == 3) {  // reflect_mean: global mean first (aalc.cpp:270-295)
        for (int r = 0; r < c->R; ++r) {
            Dev& d = c->sh[r]->d;
            cudaSetDevice(c->dev[r]);
            k_stride_partial<<<(unsigned)d.NS, 128, 0, c->sh[r]->stream>>>(d);
            ++c->sh[r]->launches;
            CU(cudaEventRecord(c->ev_sh[r], c->sh[r]->stream));
        }
        cudaSetDevice(d0);
        for (int r = 0; r < c->R; ++r) {
            CU(cudaStreamWaitEvent(fs, c->ev_sh[r], 0));
            CU(cudaMemcpyPeerAsync(c->g_partial + 2 * r * c->nsl, d0, c->sh[r]->d.partial, c->dev[r], 16 * c->nsl, fs));
        }
        k_cluster_fold<<<1, FOLD_THREADS, 0, fs>>>(0, c->NS, c->n, c->l2p, nullptr, nullptr, c->g_partial, nullptr,
                                                   nullptr, nullptr, c->R, c->fold_out, nullptr, 0);
        CU(cudaEventRecord(c->ev_fold, fs));
        for (int r = 0; r < c->R; ++r) {
            cudaSetDevice(c->dev[r]);
            CU(cudaStreamWaitEvent(c->sh[r]->stream, c->ev_fold, 0));
            if (r) CU(cudaMemcpyPeerAsync(c->f_sh[r], c->dev[r], c->fold_out, d0, 32, c->sh[r]->stream));
            k_put_mean<<<1, 1, 0, c->sh[r]->stream>>>(c->sh[r]->d, r ? c->f_sh[r] : c->fold_out);
        }
        given = kMeanPreset;
    }
    std::vector<uint64_t> n_rep(c->R, 0);
    for (int r = 0; r < c->R; ++r) {
        qcs_dev_state* st = c->sh[r];
        cudaSetDevice(c->dev[r]);
        st->d.rec = nullptr;
        if (part[r]) {
            uint64_t ns = 0;
            const int rc = enqueue_gate(st, &local[r], lad, nl, theta, -1, gate_index, &ns, 0, given);
            if (rc) return rc;
            n_rep[r] = ns;
        }
    }
    // Wave-layout shards (large states) can suspend inside the gate when their
    // arena fills (QCS_SUSPEND): check them before the fold reads their tables
    // -- one host synchronisation per gate, for such shards only -- and resume
    // after a compaction, exactly as qcs_run_program does for one state.
    for (int r = 0; r < c->R; ++r) {
        qcs_dev_state* st = c->sh[r];
        if (!st->big || !part[r]) continue;
        cudaSetDevice(c->dev[r]);
        int64_t pg = -2;
        uint64_t pu = 0, unit = 0;
        for (;;) {
            int rc = sync_and_check(st);
            if (rc) return rc;
            if (st->h_sc->err != QCS_SUSPEND) break;
            int64_t gi;
            rc = handle_suspend(st, &gi, &unit, pg, pu);
            if (rc) return rc;
            pg = gi, pu = unit;
            uint64_t ns = 0;
            rc = enqueue_gate(st, &local[r], lad, nl, theta, -1, gate_index, &ns, 0, kMeanPreset, nullptr, 0, 0, unit,
                              true);
            if (rc) return rc;
        }
    }
    for (int r = 0; r < c->R; ++r) {
        qcs_dev_state* st = c->sh[r];
        cudaSetDevice(c->dev[r]);
        k_copy_gate_cin<<<1, 1, 0, st->stream>>>(st->d, reinterpret_cast<uint64_t*>(c->f_sh[r] + 4), part[r] ? 1 : 0);
        CU(cudaEventRecord(c->ev_sh[r], st->stream));
    }
    // gather to the fold device, fold, scale every shard
    cudaSetDevice(d0);
    for (int r = 0; r < c->R; ++r) {
        CU(cudaStreamWaitEvent(fs, c->ev_sh[r], 0));
        const Dev& d = c->sh[r]->d;
        CU(cudaMemcpyPeerAsync(c->g_scale + r * c->nsl, d0, d.scale, c->dev[r], 8 * c->nsl, fs));
        CU(cudaMemcpyPeerAsync(c->g_sum + r * c->nsl, d0, d.sum_sq, c->dev[r], 8 * c->nsl, fs));
        CU(cudaMemcpyPeerAsync(c->g_cin + r, d0, c->f_sh[r] + 4, c->dev[r], 8, fs));
        if (n_rep[r]) {
            CU(cudaMemcpyPeerAsync(c->g_rep + r * c->nsl, d0, d.reports, c->dev[r], sizeof(qcs_stride_report) * n_rep[r], fs));
            k_cluster_scatter<<<(unsigned)((n_rep[r] + 255) / 256), 256, 0, fs>>>(c->g_rep, c->p2l, r * c->nsl, n_rep[r],
                                                                               (uint64_t)r * c->nsl, pbit, c->pos_map);
        }
    }
    k_cluster_fold<<<1, FOLD_THREADS, 0, fs>>>(1, c->NS, c->n, c->l2p, c->g_scale, c->g_sum, nullptr, c->g_rep,
                                               c->pos_map, c->g_cin, c->R, c->fold_out, c->rec + rec_index, gate_index);
    CU(cudaEventRecord(c->ev_fold, fs));
    for (int r = 0; r < c->R; ++r) {
        qcs_dev_state* st = c->sh[r];
        cudaSetDevice(c->dev[r]);
        CU(cudaStreamWaitEvent(st->stream, c->ev_fold, 0));
        if (r) CU(cudaMemcpyPeerAsync(c->f_sh[r], c->dev[r], c->fold_out, d0, 32, st->stream));
        k_scale_all_dev<<<(unsigned)((c->nsl + 255) / 256), 256, 0, st->stream>>>(st->d.scale, c->nsl,
                                                                                  r ? c->f_sh[r] : c->fold_out);
        st->launches += 2;
    }
    CU(cudaGetLastError());
    return 0;
}

}  // namespace

extern "C" {

int qcs_cluster_create(int n, int s, int rank_bits, uint64_t basis, const int* devices, int n_devices, int backend,
                       qcs_cluster_t* out)
{
    if (!out || !devices) return set_err(QCS_E_INVALID, "null argument");
    if (rank_bits < 0 || rank_bits > 3) return set_err(QCS_E_INVALID, "rank_bits must be in [0, 3]");
    const int R = 1 << rank_bits;
    if (n_devices != R) return set_err(QCS_E_INVALID, "need one device entry per rank (%d)", R);
    if (n < 1 || n > 59 || s < 0 || n - rank_bits < s + 1)
        return set_err(QCS_E_INVALID, "each rank needs at least two strides (n - rank_bits > stride_bits)");
    if (basis >= (1ull << n)) return set_err(QCS_E_RANGE, "basis index out of range");
    if (backend != 0 && backend != 1) return set_err(QCS_E_INVALID, "backend: 0 loopback, 1 nccl");
    auto* c = new qcs_cluster();
    c->n = n, c->s = s, c->g = rank_bits, c->R = R, c->backend = backend;
    c->L = 1ull << s;
    c->NS = 1ull << (n - s);
    c->nsl = c->NS >> rank_bits;
    c->dev.assign(devices, devices + R);
    const int Q = n - rank_bits;
    const int nb = n - s;
    c->pi.resize(nb);
    c->inv.resize(nb);
    for (int p = 0; p < nb; ++p) c->pi[p] = c->inv[p] = p;
    c->last_use.assign(nb, -1);
    auto fail = [&](int rc) {
        qcs_cluster_destroy(c);
        return rc;
    };
    if (backend == 1) {
        std::string why;
        if (!g_nccl.load(why)) return fail(set_err(QCS_E_RUNTIME, "NCCL backend: %s", why.c_str()));
        for (int r = 0; r < R; ++r)
            for (int q = 0; q < r; ++q)
                if (c->dev[q] == c->dev[r]) return fail(set_err(QCS_E_INVALID, "NCCL backend: one device per rank"));
        c->comms.resize(R);
        const ncclResult_t e = g_nccl.CommInitAll(c->comms.data(), R, c->dev.data());
        if (e != ncclSuccess) {
            c->comms.clear();
            return fail(set_err(QCS_E_RUNTIME, "ncclCommInitAll failed: %s", g_nccl.GetErrorString(e)));
        }
    }
    const uint64_t owner = basis >> Q;
    c->sh.assign(R, nullptr);
    for (int r = 0; r < R; ++r) {
        const uint64_t b = ((uint64_t)r == owner) ? (basis & ((1ull << Q) - 1)) : ~0ull;
        const int rc = qcs_state_create(Q, s, b, c->dev[r], &c->sh[r]);
        if (rc) return fail(rc);
    }
    {  // peer access between the shards' devices (fold tables, loopback copies)
        for (int r = 0; r < R; ++r)
            for (int q = 0; q < R; ++q)
                if (c->dev[r] != c->dev[q]) {
                    cudaSetDevice(c->dev[r]);
                    cudaDeviceEnablePeerAccess(c->dev[q], 0);
                    cudaGetLastError();
                }
    }
    const int d0 = c->dev[0];
    int rc = 0;
    void* p = nullptr;
#define CL_ALLOC(dst, dev_, bytes)                      \
    do {                                                \
        rc = cl_alloc(c, dev_, &p, bytes);              \
        if (rc) return fail(rc);                        \
        dst = reinterpret_cast<decltype(dst)>(p);       \
    } while (0)
    CL_ALLOC(c->g_scale, d0, 8 * c->NS);
    CL_ALLOC(c->g_sum, d0, 8 * c->NS);
    CL_ALLOC(c->g_partial, d0, 16 * c->NS);
    CL_ALLOC(c->g_rep, d0, sizeof(qcs_stride_report) * c->NS);
    CL_ALLOC(c->pos_map, d0, 16 * c->NS);
    CL_ALLOC(c->l2p, d0, 8 * c->NS);
    CL_ALLOC(c->p2l, d0, 8 * c->NS);
    CL_ALLOC(c->g_cin, d0, 8 * R);
    CL_ALLOC(c->fold_out, d0, 32);
    cudaSetDevice(d0);
    CU(cudaMemset(c->pos_map, 0xff, 16 * c->NS));
    CU(cudaMemset(c->g_cin, 0, 8 * R));
    c->f_sh.assign(R, nullptr);
    c->ev_sh.assign(R, nullptr);
    for (int r = 0; r < R; ++r) {
        CL_ALLOC(c->f_sh[r], c->dev[r], 64);  // [0..3] the fold's output, [4] the shard's gate C_in
        cudaSetDevice(c->dev[r]);
        cudaEventCreateWithFlags(&c->ev_sh[r], cudaEventDisableTiming);
    }
    cudaSetDevice(d0);
    cudaEventCreateWithFlags(&c->ev_fold, cudaEventDisableTiming);
    // exchange buffers: QCS_EXCHANGE_CHUNK_BYTES per direction per shard
    // (default 2 GiB, capped near a shard's worst-case half state)
    uint64_t cap = 2ull << 30;
    if (const char* e = getenv("QCS_EXCHANGE_CHUNK_BYTES")) cap = std::max<uint64_t>(1 << 16, strtoull(e, nullptr, 10));
    const uint64_t worst = (c->nsl / 2) * (2 * payload_cap(c->L) + 2 * c->sh[0]->d.nsub * sizeof(SideEntry) + 256) + 4096;
    c->img_cap = std::min<uint64_t>(cap, worst);
    c->img_send.assign(R, nullptr);
    c->img_recv.assign(R, nullptr);
    for (int r = 0; r < R; ++r) {
        CL_ALLOC(c->img_send[r], c->dev[r], c->img_cap);
        CL_ALLOC(c->img_recv[r], c->dev[r], c->img_cap);
    }
#undef CL_ALLOC
    rc = cl_upload_tables(c);
    if (rc) return fail(rc);
    *out = c;
    return 0;
}

void qcs_cluster_destroy(qcs_cluster_t c)
{
    if (!c) return;
    for (int r = 0; r < (int)c->sh.size(); ++r)
        if (c->sh[r]) qcs_state_destroy(c->sh[r]);
    for (size_t i = 0; i < c->allocs.size(); ++i) {
        cudaSetDevice(c->alloc_dev[i]);
        cudaFree(c->allocs[i]);
    }
    for (size_t r = 0; r < c->ev_sh.size(); ++r)
        if (c->ev_sh[r]) cudaEventDestroy(c->ev_sh[r]);
    if (c->ev_fold) cudaEventDestroy(c->ev_fold);
    for (auto cm : c->comms) g_nccl.CommDestroy(cm);
    delete c;
}

int qcs_cluster_set_schedule(qcs_cluster_t c, const qcs_gate_desc* gates, uint64_t n_gates)
{
    if (!c || (!gates && n_gates)) return set_err(QCS_E_INVALID, "null argument");
    c->next_target.assign(c->n - c->s, {});
    for (uint64_t i = 0; i < n_gates; ++i)
        if ((gates[i].kind == 0 || gates[i].kind == 1) && gates[i].target >= c->s && gates[i].target < c->n)
            c->next_target[gates[i].target - c->s].push_back(i);
    c->sched = true;
    return 0;
}

int qcs_cluster_run_program(qcs_cluster_t c, const qcs_gate_desc* gates, uint64_t n_gates, uint64_t first_index,
                            const double* lad, int nl, double theta, qcs_gate_record* records, uint64_t* n_done)
{
    if (!c || (!gates && n_gates)) return set_err(QCS_E_INVALID, "null argument");
    if (n_done) *n_done = 0;
    int rc = validate_ladder(lad, nl, theta);
    if (rc) return rc;
    for (uint64_t i = 0; i < n_gates; ++i) {  // GateOp::validate (gate.cpp:109-137) against n
        const qcs_gate_desc& q = gates[i];
        const unsigned long long gi = (unsigned long long)(first_index + i);
        if (q.kind < 0 || q.kind > 3) return set_err(QCS_E_INVALID, "gate %llu failed: unknown gate kind %d", gi, q.kind);
        if (q.kind <= 1 && (q.target < 0 || q.target >= c->n))
            return set_err(QCS_E_RANGE, "gate %llu failed: target qubit out of range", gi);
        if (q.kind == 1 && (q.control < 0 || q.control >= c->n))
            return set_err(QCS_E_RANGE, "gate %llu failed: control qubit out of range", gi);
        if (q.kind == 1 && q.control == q.target)
            return set_err(QCS_E_INVALID, "gate %llu failed: control qubit equals target qubit", gi);
        if (q.kind == 2 && q.flip_index >= (1ull << c->n))
            return set_err(QCS_E_RANGE, "gate %llu failed: flip index out of range", gi);
    }
    g_err.clear();
    if (c->rec_cap < n_gates) {
        void* p = nullptr;
        rc = cl_alloc(c, c->dev[0], &p, sizeof(qcs_gate_record) * std::max<uint64_t>(1, n_gates));
        if (rc) return rc;
        c->rec = static_cast<qcs_gate_record*>(p);
        c->rec_cap = n_gates;
    }
    const int d0 = c->dev[0];
    std::vector<cudaEvent_t> ev(n_gates + 1);
    cudaSetDevice(d0);
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(ev[0], c->sh[0]->stream);
    uint64_t done = 0;
    for (uint64_t i = 0; i < n_gates; ++i) {
        rc = cl_enqueue_gate(c, &gates[i], lad, nl, theta, i, first_index + i);
        if (rc) break;
        cudaSetDevice(d0);
        cudaEventRecord(ev[i + 1], c->sh[0]->stream);
        done = i + 1;
    }
    int rc2 = cl_sync_all(c);
    for (int r = 0; r < c->R && !rc2; ++r)
        if (c->sh[r]->h_sc) {
            cudaSetDevice(c->dev[r]);
            cudaMemcpy(c->sh[r]->h_sc, c->sh[r]->d.sc, sizeof(Dev::Scal), cudaMemcpyDeviceToHost);
            if (c->sh[r]->h_sc->err) rc2 = report_device_error(c->sh[r]);
        }
    if (!rc2 && done) {
        std::vector<qcs_gate_record> h(done);
        cudaSetDevice(d0);
        cudaMemcpy(h.data(), c->rec, done * sizeof(qcs_gate_record), cudaMemcpyDeviceToHost);
        for (uint64_t i = 0; i < done; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            // between the folds of gates i-1 and i on shard 0's stream (the
            // fold waits for every shard; an exchange before the gate runs on
            // the shards' streams in between, so it is included)
            h[i].elapsed_ns = (uint64_t)((double)ms * 1e6);
            if (records) records[i] = h[i];
        }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (n_done) *n_done = rc2 ? 0 : done;
    if (rc2) return rc2;
    return rc;
}

// Logical amplitudes (interleaved re/im, 2^(n+1) doubles): logical stride j is
// physical stride l2p[j], i.e. shard l2p[j] >> (n-g-s), local l2p[j] & (nsl-1).
int qcs_cluster_to_amplitudes(qcs_cluster_t c, double* amps)
{
    if (!c || !amps) return set_err(QCS_E_INVALID, "null argument");
    std::vector<uint64_t> l2p, p2l;
    cl_tables(c, l2p, p2l);
    const uint64_t L = c->L;
    std::vector<double> re(L), im(L);
    for (uint64_t j = 0; j < c->NS; ++j) {
        const uint64_t jp = l2p[j];
        const int rc = qcs_read_stride(c->sh[jp / c->nsl], jp % c->nsl, 1, re.data(), im.data());
        if (rc) return rc;
        for (uint64_t i = 0; i < L; ++i) {
            amps[2 * (j * L + i)] = re[i];
            amps[2 * (j * L + i) + 1] = im[i];
        }
    }
    return 0;
}

// exchanges, exchange payload bytes (images sent, all shards), exchange wall
// seconds, norm_sq of the last gate's fold
int qcs_cluster_stats(qcs_cluster_t c, uint64_t* exchanges, uint64_t* exchange_bytes, double* exchange_s,
                      double* norm_sq)
{
    if (!c) return set_err(QCS_E_INVALID, "null cluster");
    if (exchanges) *exchanges = c->exchanges;
    if (exchange_bytes) *exchange_bytes = c->exchange_bytes;
    if (exchange_s) *exchange_s = c->exchange_ns * 1e-9;
    if (norm_sq) {
        int rc = cl_sync_all(c);
        if (rc) return rc;
        double out[4];
        cudaSetDevice(c->dev[0]);
        CU(cudaMemcpy(out, c->fold_out, 32, cudaMemcpyDeviceToHost));
        *norm_sq = out[3];
    }
    return 0;
}

// The shard of rank r (an ordinary engine state of n-g qubits, for per-shard
// queries: qcs_state_stats, qcs_state_memory, ...).  Owned by the cluster.
qcs_dev_state_t qcs_cluster_shard(qcs_cluster_t c, int r)
{
    return (c && r >= 0 && r < c->R) ? c->sh[r] : nullptr;
}

}  // extern "C"
