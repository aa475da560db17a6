/*
 * qcs_oracle — CPU restatement of the reference's compressed-state gate path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline leg).
 * The product library (libqcs_b200.so) never links, loads or calls it.
 *
 * Every function restates a reference function (file:line under
 * /root/reference/proj) and is pinned against the compiled reference
 * (oracle/_ref/libqcsref.so) and the golden vectors in tests/golden/.
 * All arithmetic is IEEE binary64 round-to-nearest with FP contraction off,
 * matching the reference's default x86-64 build.
 */
#ifndef QCS_ORACLE_H
#define QCS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (shared numbering with include/qcs_b200.h). */
enum {
    QO_OK = 0,
    QO_E_RUNTIME = 1,       /* std::runtime_error */
    QO_E_INVALID = 2,       /* std::invalid_argument */
    QO_E_RANGE = 3,         /* std::out_of_range */
    QO_E_CAPACITY = 4,      /* caller buffer too small (ABI-only) */
    QO_E_BAD_MAGIC = 10,    /* CodecError::bad_magic     codec.hpp:38 */
    QO_E_TRUNCATED = 11,    /* CodecError::truncated     codec.hpp:39 */
    QO_E_UNKNOWN_CODEC = 12,/* CodecError::unknown_codec codec.hpp:40 */
    QO_E_BAD_VALUE = 13     /* CodecError::bad_value     codec.hpp:41 */
};

#define QO_HEADER_BYTES 29u  /* codec.hpp:54 */

/* Gate descriptor: kind follows GateKind (gate.hpp:36-41):
 * 0 single, 1 controlled, 2 diag_phase_flip, 3 reflect_mean.
 * u[8] = {u11r,u11i,u12r,u12i,u21r,u21i,u22r,u22i} (gate.cpp:141-151). */
typedef struct {
    int32_t kind;
    int32_t target;
    int32_t control;
    int32_t pad_;
    uint64_t flip_index;
    double u[8];
} qo_gate;

/* StrideCompressReport (aalc.hpp:62-69). */
typedef struct {
    uint64_t stride_index;
    uint64_t bytes_in;
    uint64_t bytes_out;
    double chosen_delta;
    double ratio;
    int32_t threshold_met;
    int32_t pad_;
} qo_report;

const char* qo_last_error(void);

/* ---- codec (codec.cpp) ---- */
/* compress(): payload only (no header).  delta == 0 -> lossless. */
int qo_compress_payload(const double* x, uint64_t n, double delta, uint8_t* out,
                        uint64_t cap, uint64_t* len);
/* serialize_block(compress(x)) : 29-byte QCS1 header + payload. */
int qo_compress(const double* x, uint64_t n, double delta, uint8_t* out,
                uint64_t cap, uint64_t* len);
/* decompress a payload of the given codec id. */
int qo_decompress_payload(int codec, double delta, const uint8_t* p, uint64_t plen,
                          double* out, uint64_t n);
/* parse_block + decompress_into on a serialized block. */
int qo_decompress(const uint8_t* blk, uint64_t len, double* out, uint64_t n);

/* ---- stride gate kernels on decompressed planes (gate.cpp:166-301) ---- */
int qo_apply_unit(int n_qubits, int stride_bits, const qo_gate* g,
                  uint64_t lo_index, double* lo_re, double* lo_im,
                  uint64_t hi_index, double* hi_re, double* hi_im,
                  double mean_re, double mean_im);

/* ---- engine (aalc.cpp) ---- */
typedef struct qo_state qo_state;
int qo_state_create(int n_qubits, int stride_bits, uint64_t basis, qo_state** out);
void qo_state_destroy(qo_state* st);
int qo_state_clone(const qo_state* st, qo_state** out);
int qo_apply_gate(qo_state* st, const qo_gate* g, const double* ladder, int n_levels,
                  double theta, qo_report* reports, uint64_t* n_reports,
                  double* norm_after);
int qo_to_amplitudes(const qo_state* st, double* amps /* 2*2^n interleaved */);
int qo_stored_stride(const qo_state* st, uint64_t j, int apply_scale, double* re,
                     double* im);
int qo_stats(const qo_state* st, uint64_t* compressed_bytes, double* min_ratio,
             double* norm_sq_tracked);
int qo_stride_info(const qo_state* st, uint64_t j, double* scale, double* sum_sq,
                   uint64_t* re_payload, uint64_t* im_payload);
/* Serialized blocks (QCS1 re block then im block) of stride j. */
int qo_export_blocks(const qo_state* st, uint64_t j, uint8_t* buf, uint64_t cap,
                     uint64_t* len);

/* ---- sharded-run hooks (same contract as the C-ABI's) ---- */
int qo_apply_gate_ex(qo_state* st, const qo_gate* g, const double* ladder, int n_levels,
                     double theta, int flags, const double* mean, qo_report* reports,
                     uint64_t* n_reports, double* norm_after);
int qo_stride_sums(const qo_state* st, double* partial);
int qo_stride_norms(const qo_state* st, double* scales, double* sums);
int qo_scale_all(qo_state* st, double f);
int qo_import_blocks(qo_state* st, uint64_t j, const uint8_t* buf, uint64_t len, double scale,
                     double sum_sq);

/* ---- dense oracle (dense.cpp) ---- */
int qo_dense_run(int n_qubits, const qo_gate* gates, uint64_t n_gates,
                 uint64_t basis, double* amps);
double qo_fidelity(const double* a, const double* b, uint64_t n_amps);

#ifdef __cplusplus
}
#endif
#endif
