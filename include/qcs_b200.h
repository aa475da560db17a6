/*
 * qcs_b200.h — C-ABI of the B200-native compressed-state gate engine.
 *
 * Drop-in boundary for the reference's per-gate hot path
 * (/root/reference/proj, C++ API, no C-ABI of its own).
 * Every entry point names the reference interface it replaces.  Plain
 * pointers and sizes only; all buffers are HOST memory unless a name says
 * otherwise.  Calls are synchronous at the ABI (stream-ordered inside) and
 * return 0 or a QCS_E_* code; qcs_last_error() gives the message.  A state
 * is not thread-safe; the caller serialises (aalc.hpp:126-129).
 *
 * Results are bit-identical to the reference's: codes, block bytes, decoded
 * amplitudes, per-stride sums, scales and every GateRecord field except the
 * wall time (DESIGN.md §4 explains how the parallel kernels stay exact).
 */
#ifndef QCS_B200_H
#define QCS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  1:1 with the reference's exception kinds. */
enum {
    QCS_OK = 0,
    QCS_E_RUNTIME = 1,        /* std::runtime_error                           */
    QCS_E_INVALID = 2,        /* std::invalid_argument  (config error)         */
    QCS_E_RANGE = 3,          /* std::out_of_range                             */
    QCS_E_CAPACITY = 4,       /* caller buffer too small (ABI only)            */
    QCS_E_CUDA = 5,           /* CUDA runtime failure / no device              */
    QCS_E_NOMEM = 6,          /* device arena exhausted                        */
    QCS_E_BAD_MAGIC = 10,     /* CodecError::bad_magic       codec.hpp:38      */
    QCS_E_TRUNCATED = 11,     /* CodecError::truncated       codec.hpp:39      */
    QCS_E_UNKNOWN_CODEC = 12, /* CodecError::unknown_codec   codec.hpp:40      */
    QCS_E_BAD_VALUE = 13      /* CodecError::bad_value       codec.hpp:41      */
};

/* GateOp (gate.hpp:43-63).  kind: 0 single, 1 controlled, 2 diag_phase_flip,
 * 3 reflect_mean (GateKind, gate.hpp:36-41).  u = {u11r,u11i,u12r,u12i,
 * u21r,u21i,u22r,u22i} (UnitaryParts, gate.cpp:141-151).  control = -1 when
 * absent.  72 bytes. */
typedef struct {
    int32_t kind;
    int32_t target;
    int32_t control;
    int32_t pad_;
    uint64_t flip_index;
    double u[8];
} qcs_gate_desc;

/* StrideCompressReport (aalc.hpp:62-69). 48 bytes. */
typedef struct {
    uint64_t stride_index;
    uint64_t bytes_in;
    uint64_t bytes_out;
    double chosen_delta;
    double ratio;
    int32_t threshold_met;
    int32_t pad_;
} qcs_stride_report;

/* GateRecord (metrics.hpp:13-24) plus the gate's threshold-violation count
 * (RunMetrics::threshold_violations, aalc.cpp:624).  elapsed_ns is device
 * time of the gate (CUDA events), not host wall time. */
typedef struct {
    uint64_t gate_index;
    uint64_t stride_count;
    double min_ratio;
    double mean_ratio;
    double max_chosen_delta;
    uint64_t bytes_before;
    uint64_t bytes_after;
    uint64_t elapsed_ns;
    double norm_after;
    uint64_t threshold_violations;
    uint64_t compressed_in;  /* stored bytes (headers included) of the blocks the
                                gate read and rewrote: the roofline's C_in */
} qcs_gate_record;

typedef struct qcs_dev_state* qcs_dev_state_t;

const char* qcs_last_error(void);
int qcs_version(void);

/* CompressedState::basis_state (aalc.cpp:140-174) on `device`.
 * StateGeometry::make validation (core.cpp:9-23).  basis = UINT64_MAX creates
 * an all-zero state (a shard that holds none of the amplitude). */
int qcs_state_create(int n_qubits, int stride_bits, uint64_t basis, int device,
                     qcs_dev_state_t* out);
void qcs_state_destroy(qcs_dev_state_t st);

/* CompressedState::apply_gate (aalc.cpp:261-420) incl. GateOp::validate,
 * make_stride_plan, the AALC ladder (ErrorBoundLadder::make checks,
 * aalc.cpp:56-72; RatioThreshold, aalc.hpp:51-60) and the lazy global
 * renormalisation.  reports (optional, capacity = 2^(n-s)) receive the
 * stride reports in the reference's unit order.  On error the state is
 * unchanged. */
int qcs_apply_gate(qcs_dev_state_t st, const qcs_gate_desc* gate, const double* ladder,
                   int n_levels, double theta, qcs_stride_report* reports,
                   uint64_t* n_reports, double* norm_after);

/* Wave layout (states too large for two slots per plane, e.g. C3): a gate's
 * units are committed wave by wave, so an out-of-memory failure after the
 * first wave leaves the gate part-applied; the state is then refused by every
 * later call (QCS_E_RUNTIME).  Every other failure leaves the state unchanged. */

/* qcs_apply_gate with flags, for a state that is one shard of a larger one.
 * QCS_NO_RENORM skips the lazy renormalisation (aalc.cpp:410-419) so the
 * caller renormalises globally from qcs_stride_norms + qcs_scale_all in the
 * reference's stride order.  QCS_GIVEN_MEAN makes reflect_mean use mean[2]
 * (re, im) instead of this shard's own mean pass (aalc.cpp:270-295); the
 * caller combines qcs_stride_sums of every shard in global stride order. */
#define QCS_NO_RENORM 1
#define QCS_GIVEN_MEAN 2
int qcs_apply_gate_ex(qcs_dev_state_t st, const qcs_gate_desc* gate, const double* ladder,
                      int n_levels, double theta, int flags, const double* mean,
                      qcs_stride_report* reports, uint64_t* n_reports, double* norm_after);
/* Stride images for sharded runs: the reference has no
 * distribution; these move whole strides between shards as
 * device-resident images (both blocks + side index + scale + sum), e.g. with
 * NCCL send/recv over NVLink.  qcs_pack_strides packs every stride j with bit
 * `bit` of j equal to `value`, ascending, into dev_buf (device memory, cap
 * bytes); with dev_buf null it only reports *len.  qcs_unpack_strides installs
 * an image: stride j of the image becomes stride j ^ xor_mask, blocks verbatim,
 * through the ordinary commit path. */
int qcs_pack_strides(qcs_dev_state_t st, int bit, int value, void* dev_buf, uint64_t cap,
                     uint64_t* len);
/* qcs_pack_strides restricted to the strides whose position among those with
 * bit `bit` == value is in [first, first + count): an exchange streamed in
 * chunks, so a 37-qubit shard's half-state never needs one image buffer. */
int qcs_pack_strides_range(qcs_dev_state_t st, int bit, int value, uint64_t first, uint64_t count,
                           void* dev_buf, uint64_t cap, uint64_t* len);
int qcs_unpack_strides(qcs_dev_state_t st, const void* dev_buf, uint64_t len, uint64_t xor_mask);
/* Per-stride amplitude sums (stride_amplitude_sum, gate.cpp:303-311) of the
 * decompressed, scaled strides: partial[2j] = re, partial[2j+1] = im. */
int qcs_stride_sums(qcs_dev_state_t st, double* partial);
/* Per-stride pending scale and stored sum of squares (StrideStorage,
 * aalc.hpp:162-167), 2^(n-s) doubles each; either pointer may be null. */
int qcs_stride_norms(qcs_dev_state_t st, double* scales, double* sums);
/* scale *= f for every stride (the renormalisation step, aalc.cpp:413). */
int qcs_scale_all(qcs_dev_state_t st, double f);

/* apply_program_range (aalc.cpp:588-634) over gates[0..n_gates): one
 * GateRecord per gate, gate_index = first_index + i.  Launches are queued
 * back to back; one host synchronisation at the end.  On error at gate i,
 * gates before i are applied, the state reflects them, *n_done = i. */
int qcs_run_program(qcs_dev_state_t st, const qcs_gate_desc* gates, uint64_t n_gates,
                    uint64_t first_index, const double* ladder, int n_levels,
                    double theta, qcs_gate_record* records, uint64_t* n_done);

/* stored_stride / decompress_stride (aalc.cpp:191-209). */
int qcs_read_stride(qcs_dev_state_t st, uint64_t stride, int apply_scale, double* re,
                    double* im);
/* Device-resident variant for large states: strides [first, first+count)
 * decoded (and scaled if apply_scale) into dev_out, a device buffer of
 * count * 2 * 2^s doubles laid out [stride][re|im][element]. */
int qcs_read_strides_device(qcs_dev_state_t st, uint64_t first, uint64_t count, int apply_scale,
                            double* dev_out);
/* Inverse of qcs_read_strides_device: strides [first, first+count) are
 * replaced by the compression of dev_planes (device memory, count * 2 * 2^s
 * doubles laid out [stride][re|im][element]) through the ladder, exactly as
 * compress_stride_adaptive does (aalc.cpp:117-138: the planes are zero-snapped
 * IN PLACE first, then each level is tried until the ratio reaches theta);
 * scale 1 and the stored sum of squares of what was stored (aalc.cpp:46-52).
 * No renormalisation.  The reference has no from-amplitudes constructor; its
 * equivalent is a QCKP file of compress()ed blocks read by
 * CompressedState::load (aalc.cpp:496-586). */
int qcs_load_strides_device(qcs_dev_state_t st, uint64_t first, uint64_t count, double* dev_planes,
                            const double* ladder, int n_levels, double theta);
/* to_amplitudes (aalc.cpp:211-223): interleaved re/im, 2^(n+1) doubles. */
int qcs_to_amplitudes(qcs_dev_state_t st, double* amps);
/* compressed_bytes / min_stride_ratio / norm_sq_tracked (aalc.cpp:233-259). */
int qcs_state_stats(qcs_dev_state_t st, uint64_t* compressed_bytes,
                    double* min_stride_ratio, double* norm_sq_tracked);
/* stride_scale (aalc.cpp:225-231) plus the stored sum and payload sizes. */
int qcs_stride_info(qcs_dev_state_t st, uint64_t stride, double* scale, double* sum_sq,
                    uint64_t* re_payload, uint64_t* im_payload);
/* Serialized QCS1 blocks of one stride, re then im (serialize_block_append,
 * codec.cpp:369-381) — the per-stride body of a QCKP checkpoint
 * (aalc.cpp:466-494).  cap may be 0 to query *len. */
int qcs_export_blocks(qcs_dev_state_t st, uint64_t stride, uint8_t* buf, uint64_t cap,
                      uint64_t* len, double* scale, double* sum_sq);
/* Inverse of qcs_export_blocks (parse_block, codec.cpp:391-420; load,
 * aalc.cpp:496-586): validates and installs the blocks verbatim. */
int qcs_import_blocks(qcs_dev_state_t st, uint64_t stride, const uint8_t* buf,
                      uint64_t len, double scale, double sum_sq);
/* Device-side accounting for benchmarks: resident bytes of the block store
 * (payload arena in use + side index). */
int qcs_state_memory(qcs_dev_state_t st, uint64_t* arena_bytes, uint64_t* side_bytes,
                     uint64_t* scratch_bytes);
/* Number of kernel launches issued by this state so far (bench accounting). */
uint64_t qcs_state_launches(qcs_dev_state_t st);
/* Per-kernel-class device timing with CUDA events on the engine's stream
 * (bench roofline accounting).  Classes: 0 decode (k_decode_gate, input
 * passes), 1 serial chain (k_serial_chain), 2 encode (k_fused),
 * 3 commit+norm, 4 mean pass, 5 bookkeeping.  enable: 0 off, 1 every class,
 * 2 the encode class only (two events per encoder launch instead of two per
 * kernel).  Enabling resets the totals; totals cover every gate enqueued
 * while enabled. */
int qcs_state_profile(qcs_dev_state_t st, int enable);
int qcs_state_kernel_time(qcs_dev_state_t st, int kernel_class, double* total_ns,
                          uint64_t* launches);
/* Cumulative device diagnostics of the codec kernel: [0] lanes whose entry
 * predictor guess was wrong and were re-run serially, [1] passes of the exact
 * sum-of-squares emulation, [2] bytes slid to close carried word runs,
 * [3] lanes finished by the serial chain, [4] in-place arena compactions
 * and [5] slots per wave (wave layout for large states, 0 otherwise),
 * [8..14] cycles per kernel phase (input, rounds, final, sum, token count,
 * token write, tail), [17] slots the streaming kernel left to the legacy
 * encoder, [18] slots it encoded.  n <= 24. */
int qcs_state_counters(qcs_dev_state_t st, uint64_t* out, int n);

/* ---- Sharded state in one host process ----
 * The reference has no distribution.  Rank = the top rank_bits
 * qubits: rank r's strides live in an engine state of n - rank_bits qubits on
 * devices[r].  A gate whose target is a rank qubit exchanges half of the
 * partner shards' strides as device stride images (lazy qubit permutation, no
 * swap back): backend 1 = grouped ncclSend/ncclRecv (ncclCommInitAll, one
 * device per rank, libnccl.so.2 loaded at run time), backend 0 = loopback
 * device copies (several ranks may share one GPU: tests).  Renormalisation,
 * reflect_mean's mean and the GateRecords are folded on the device in the
 * reference's global stride / unit order, so results are bit-identical to a
 * single state for any rank count. */
typedef struct qcs_cluster* qcs_cluster_t;
int qcs_cluster_create(int n_qubits, int stride_bits, int rank_bits, uint64_t basis, const int* devices,
                       int n_devices, int backend, qcs_cluster_t* out);
void qcs_cluster_destroy(qcs_cluster_t c);
/* The program's gates, so an exchange evicts the local qubit needed furthest
 * in the future (Belady); without it, the least recently used one. */
int qcs_cluster_set_schedule(qcs_cluster_t c, const qcs_gate_desc* gates, uint64_t n_gates);
/* apply_program_range (aalc.cpp:588-634) across the shards: one GateRecord per
 * gate (elapsed_ns: device time between the gate's fold and the previous one,
 * exchanges included), one host synchronisation at the end (plus one per gate
 * for shards in the wave layout, and the exchanges). */
int qcs_cluster_run_program(qcs_cluster_t c, const qcs_gate_desc* gates, uint64_t n_gates, uint64_t first_index,
                            const double* ladder, int n_levels, double theta, qcs_gate_record* records,
                            uint64_t* n_done);
/* to_amplitudes of the LOGICAL state (interleaved re/im, 2^(n+1) doubles). */
int qcs_cluster_to_amplitudes(qcs_cluster_t c, double* amps);
int qcs_cluster_stats(qcs_cluster_t c, uint64_t* exchanges, uint64_t* exchange_bytes, double* exchange_s,
                      double* norm_sq);
/* Rank r's shard (owned by the cluster), for per-shard queries. */
qcs_dev_state_t qcs_cluster_shard(qcs_cluster_t c, int r);

/* Codec plugin (codec.hpp:80-105): compress(x, ErrorBound(delta)) then
 * serialize_block.  out receives the 29-byte QCS1 header + payload; cap may
 * be 0 to query *len. */
int qcs_codec_compress(const double* x, uint64_t n, double delta, uint8_t* out,
                       uint64_t cap, uint64_t* len);
/* parse_block + decompress_into of one serialized block into out[n]. */
int qcs_codec_decompress(const uint8_t* block, uint64_t len, double* out, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
