/*
 * qcs_oracle.c — plain-C restatement of the reference's per-gate
 * decompress -> gate -> recompress path.  TEST INFRASTRUCTURE ONLY (see
 * qcs_oracle.h).  Citations are /root/reference/proj/<file>:<line>.
 *
 * Pinned by tests/test_oracle_pin.py against oracle/_ref/libqcsref.so (the
 * unmodified reference, built by oracle/Makefile) and tests/golden/.
 * Build flags: -ffp-contract=off (no FMA), exactly like the reference's
 * default x86-64 Release build.
 */
#include "qcs_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* qo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* byte buffer                                                              */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint8_t* p;
    uint64_t len, cap;
} bytes_t;

static void bt_push(bytes_t* b, uint8_t v)
{
    if (b->len == b->cap) {
        b->cap = b->cap ? 2 * b->cap : 64;
        b->p = (uint8_t*)realloc(b->p, b->cap);
    }
    b->p[b->len++] = v;
}

/* codec.cpp:22-29 */
static void put_varint(bytes_t* b, uint64_t v)
{
    while (v >= 0x80) {
        bt_push(b, (uint8_t)v | 0x80);
        v >>= 7;
    }
    bt_push(b, (uint8_t)v);
}

/* codec.cpp:62-67 */
static void put_word(bytes_t* b, uint64_t w)
{
    for (int i = 0; i < 8; ++i) bt_push(b, (uint8_t)(w >> (8 * i)));
}

/* codec.cpp:31-48.  Returns 0 or an error code. */
static int get_varint(const uint8_t* in, uint64_t n, uint64_t* pos, uint64_t* out)
{
    uint64_t v = 0;
    int shift = 0;
    for (;;) {
        if (*pos >= n) return fail(QO_E_TRUNCATED, "payload ends inside a varint");
        uint8_t b = in[(*pos)++];
        if (shift >= 63 && (b & 0x7e) != 0)
            return fail(QO_E_BAD_VALUE, "varint overflows 64 bits");
        v |= (uint64_t)(b & 0x7f) << (shift & 63);
        if ((b & 0x80) == 0) {
            *out = v;
            return 0;
        }
        shift += 7;
    }
}

/* codec.cpp:50-60 */
static uint64_t zigzag(int64_t q) { return ((uint64_t)q << 1) ^ (uint64_t)(q >> 63); }
static int64_t unzigzag(uint64_t z) { return (int64_t)(z >> 1) ^ -(int64_t)(z & 1); }

/* codec.cpp:69-81 */
static int get_word(const uint8_t* in, uint64_t n, uint64_t* pos, uint64_t* w)
{
    if (*pos + 8 > n) return fail(QO_E_TRUNCATED, "payload ends inside a raw word");
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)in[*pos + i] << (8 * i);
    *pos += 8;
    *w = v;
    return 0;
}

static uint64_t bits_of(double x)
{
    uint64_t w;
    memcpy(&w, &x, 8);
    return w;
}

static double from_bits(uint64_t w)
{
    double x;
    memcpy(&x, &w, 8);
    return x;
}

/* codec.cpp:83-91 */
static int require_finite(const double* x, uint64_t n)
{
    for (uint64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return fail(QO_E_BAD_VALUE, "NaN/Inf cannot be compressed");
    return 0;
}

/* ------------------------------------------------------------------------ */
/* codecs                                                                   */
/* ------------------------------------------------------------------------ */

/* compress_lossless, codec.cpp:118-147 */
static int compress_lossless(const double* x, uint64_t n, bytes_t* out)
{
    int rc = require_finite(x, n);
    if (rc) return rc;
    uint64_t i = 0;
    while (i < n) {
        if (bits_of(x[i]) == 0) {
            uint64_t j = i;
            while (j < n && bits_of(x[j]) == 0) ++j;
            put_varint(out, (j - i) << 1);
            i = j;
        } else {
            uint64_t j = i;
            while (j < n && bits_of(x[j]) != 0) ++j;
            put_varint(out, ((j - i) << 1) | 1u);
            for (uint64_t k = i; k < j; ++k) put_word(out, bits_of(x[k]));
            i = j;
        }
    }
    return 0;
}

/* LossyEmitter, codec.cpp:153-202: maximal zero-code runs and escape runs. */
typedef struct {
    bytes_t* out;
    uint64_t zero_run;
    uint64_t* esc;
    uint64_t n_esc, cap_esc;
} emitter_t;

static void em_flush_zeros(emitter_t* e)
{
    if (e->zero_run > 0) {
        put_varint(e->out, e->zero_run << 2);
        e->zero_run = 0;
    }
}

static void em_flush_escapes(emitter_t* e)
{
    if (e->n_esc > 0) {
        put_varint(e->out, (e->n_esc << 2) | 2u);
        for (uint64_t i = 0; i < e->n_esc; ++i) put_word(e->out, e->esc[i]);
        e->n_esc = 0;
    }
}

static void em_zero_code(emitter_t* e)
{
    em_flush_escapes(e);
    ++e->zero_run;
}

static void em_code(emitter_t* e, int64_t q)
{
    em_flush_escapes(e);
    em_flush_zeros(e);
    put_varint(e->out, (zigzag(q) << 2) | 1u);
}

static void em_escape(emitter_t* e, double x)
{
    em_flush_zeros(e);
    if (e->n_esc == e->cap_esc) {
        e->cap_esc = e->cap_esc ? 2 * e->cap_esc : 16;
        e->esc = (uint64_t*)realloc(e->esc, e->cap_esc * 8);
    }
    e->esc[e->n_esc++] = bits_of(x);
}

#define QUANT_RADIUS 32768 /* codec.cpp:11 */

/* compress_lossy, codec.cpp:206-250 */
static int compress_lossy(const double* x, uint64_t n, double delta, bytes_t* out)
{
    if (!(delta > 0.0)) return fail(QO_E_BAD_VALUE, "lossy compression requires delta > 0");
    int rc = require_finite(x, n);
    if (rc) return rc;
    const double two_delta = 2.0 * delta;
    const double escape_limit = two_delta * (double)QUANT_RADIUS;
    emitter_t em = {out, 0, NULL, 0, 0};
    double pred = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double xi = x[i];
        const double diff = xi - pred;
        int coded = 0;
        if (fabs(diff) < escape_limit) {
            const int64_t q = llround(diff / two_delta);
            if (q > -QUANT_RADIUS && q < QUANT_RADIUS) {
                const double recon = pred + two_delta * (double)q;
                if (fabs(xi - recon) <= delta) {
                    if (q == 0) em_zero_code(&em);
                    else em_code(&em, q);
                    pred = recon;
                    coded = 1;
                }
            }
        }
        if (!coded) {
            em_escape(&em, xi);
            pred = xi;
        }
    }
    em_flush_escapes(&em); /* finish(): codec.cpp:197-201 */
    em_flush_zeros(&em);
    free(em.esc);
    return 0;
}

/* ErrorBound ctor (codec.cpp:111-116) + compress dispatch (codec.cpp:252-256) */
static int compress_any(const double* x, uint64_t n, double delta, bytes_t* out)
{
    if (!(delta >= 0.0) || !isfinite(delta))
        return fail(QO_E_INVALID, "error bound must be finite and >= 0");
    return delta == 0.0 ? compress_lossless(x, n, out) : compress_lossy(x, n, delta, out);
}

/* decompress_lossless_into, codec.cpp:260-286 */
static int decompress_lossless(const uint8_t* in, uint64_t len, double* out, uint64_t n)
{
    uint64_t pos = 0, produced = 0;
    while (produced < n) {
        uint64_t v;
        int rc = get_varint(in, len, &pos, &v);
        if (rc) return rc;
        const uint64_t run = v >> 1;
        if (run == 0 || run > n - produced)
            return fail(QO_E_BAD_VALUE, "run length inconsistent with scalar count");
        if ((v & 1u) == 0) {
            for (uint64_t k = 0; k < run; ++k) out[produced++] = 0.0;
        } else {
            for (uint64_t k = 0; k < run; ++k) {
                uint64_t w = 0;
                rc = get_word(in, len, &pos, &w);
                if (rc) return rc;
                out[produced++] = from_bits(w);
            }
        }
    }
    if (pos != len) return fail(QO_E_BAD_VALUE, "trailing bytes after final token");
    return 0;
}

/* decompress_lossy_into, codec.cpp:288-340 */
static int decompress_lossy(const uint8_t* in, uint64_t len, double delta, double* out,
                            uint64_t n)
{
    uint64_t pos = 0, produced = 0;
    const double two_delta = 2.0 * delta;
    double pred = 0.0;
    while (produced < n) {
        uint64_t v;
        int rc = get_varint(in, len, &pos, &v);
        if (rc) return rc;
        const unsigned tag = (unsigned)(v & 3u);
        const uint64_t arg = v >> 2;
        switch (tag) {
            case 0:
                if (arg == 0 || arg > n - produced)
                    return fail(QO_E_BAD_VALUE, "zero-run length inconsistent");
                for (uint64_t k = 0; k < arg; ++k) out[produced++] = pred;
                break;
            case 1: {
                const int64_t q = unzigzag(arg);
                if (q == 0 || q <= -QUANT_RADIUS || q >= QUANT_RADIUS)
                    return fail(QO_E_BAD_VALUE, "quantization code out of range");
                pred = pred + two_delta * (double)q;
                out[produced++] = pred;
                break;
            }
            case 2:
                if (arg == 0 || arg > n - produced)
                    return fail(QO_E_BAD_VALUE, "escape-run length inconsistent");
                for (uint64_t k = 0; k < arg; ++k) {
                    uint64_t w = 0;
                    rc = get_word(in, len, &pos, &w);
                    if (rc) return rc;
                    pred = from_bits(w);
                    out[produced++] = pred;
                }
                break;
            default:
                return fail(QO_E_BAD_VALUE, "unknown payload token");
        }
    }
    if (pos != len) return fail(QO_E_BAD_VALUE, "trailing bytes after final token");
    return 0;
}

int qo_decompress_payload(int codec, double delta, const uint8_t* p, uint64_t plen,
                          double* out, uint64_t n)
{
    /* decompress_into dispatch, codec.cpp:344-360 */
    if (codec == 0) return decompress_lossless(p, plen, out, n);
    if (codec == 1) return decompress_lossy(p, plen, delta, out, n);
    return fail(QO_E_UNKNOWN_CODEC, "unknown codec id %d", codec);
}

int qo_compress_payload(const double* x, uint64_t n, double delta, uint8_t* out,
                        uint64_t cap, uint64_t* len)
{
    bytes_t b = {0};
    int rc = compress_any(x, n, delta, &b);
    if (!rc) {
        *len = b.len;
        if (out) {
            if (b.len > cap) rc = fail(QO_E_CAPACITY, "output buffer too small");
            else if (b.len) memcpy(out, b.p, b.len);
        }
    }
    free(b.p);
    return rc;
}

static void put_u64_le(uint8_t* p, uint64_t v)
{
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

static uint64_t read_u64_le(const uint8_t* p)
{
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

/* serialize_block_append, codec.cpp:369-381 */
static void write_header(uint8_t* p, int codec, double delta, uint64_t count,
                         uint64_t payload_len)
{
    p[0] = 'Q';
    p[1] = 'C';
    p[2] = 'S';
    p[3] = '1';
    p[4] = (uint8_t)codec;
    put_u64_le(p + 5, bits_of(delta));
    put_u64_le(p + 13, count);
    put_u64_le(p + 21, payload_len);
}

int qo_compress(const double* x, uint64_t n, double delta, uint8_t* out, uint64_t cap,
                uint64_t* len)
{
    bytes_t b = {0};
    int rc = compress_any(x, n, delta, &b);
    if (!rc) {
        *len = QO_HEADER_BYTES + b.len;
        if (out) {
            if (*len > cap) {
                rc = fail(QO_E_CAPACITY, "output buffer too small");
            } else {
                write_header(out, delta == 0.0 ? 0 : 1, delta, n, b.len);
                if (b.len) memcpy(out + QO_HEADER_BYTES, b.p, b.len);
            }
        }
    }
    free(b.p);
    return rc;
}

/* parse_block, codec.cpp:391-420 */
static int parse_block(const uint8_t* bytes, uint64_t size, uint64_t* offset, int* codec,
                       double* delta, uint64_t* count, const uint8_t** payload,
                       uint64_t* plen)
{
    if (*offset + QO_HEADER_BYTES > size)
        return fail(QO_E_TRUNCATED, "block header extends past end of data");
    const uint8_t* p = bytes + *offset;
    if (p[0] != 'Q' || p[1] != 'C' || p[2] != 'S' || p[3] != '1')
        return fail(QO_E_BAD_MAGIC, "bad block magic");
    *codec = p[4];
    if (*codec != 0 && *codec != 1) return fail(QO_E_UNKNOWN_CODEC, "unknown codec id %d", *codec);
    *delta = from_bits(read_u64_le(p + 5));
    *count = read_u64_le(p + 13);
    const uint64_t pl = read_u64_le(p + 21);
    *offset += QO_HEADER_BYTES;
    if (*offset + pl > size) return fail(QO_E_TRUNCATED, "block payload extends past end of data");
    *payload = bytes + *offset;
    *plen = pl;
    *offset += pl;
    return 0;
}

int qo_decompress(const uint8_t* blk, uint64_t len, double* out, uint64_t n)
{
    uint64_t off = 0, count, plen;
    int codec;
    double delta;
    const uint8_t* payload;
    int rc = parse_block(blk, len, &off, &codec, &delta, &count, &payload, &plen);
    if (rc) return rc;
    if (count != n) return fail(QO_E_INVALID, "output span does not match scalar count");
    return qo_decompress_payload(codec, delta, payload, plen, out, n);
}

/* ------------------------------------------------------------------------ */
/* gate kernels (gate.cpp)                                                  */
/* ------------------------------------------------------------------------ */

/* apply_pair arithmetic, gate.cpp:153-162 (left-to-right, no FMA) */
static inline void pair_update(const double* m, double* r0, double* i0, double* r1,
                               double* i1)
{
    const double t0r = *r0, t0i = *i0, t1r = *r1, t1i = *i1;
    *r0 = m[0] * t0r - m[1] * t0i + m[2] * t1r - m[3] * t1i;
    *i0 = m[0] * t0i + m[1] * t0r + m[2] * t1i + m[3] * t1r;
    *r1 = m[4] * t0r - m[5] * t0i + m[6] * t1r - m[7] * t1i;
    *i1 = m[4] * t0i + m[5] * t0r + m[6] * t1i + m[7] * t1r;
}

/* apply_single_in_stride gate.cpp:166-185; apply_controlled_in_stride :218-242 */
static void in_stride(uint64_t L, const double* m, int target, int control, double* re,
                      double* im)
{
    const uint64_t half = (uint64_t)1 << target, lo_mask = half - 1;
    const uint64_t cbit = control >= 0 ? (uint64_t)1 << control : 0;
    for (uint64_t i = 0; i < L / 2; ++i) {
        const uint64_t i0 = ((i & ~lo_mask) << 1) | (i & lo_mask);
        if (control >= 0 && !(i0 & cbit)) continue;
        const uint64_t i1 = i0 | half;
        pair_update(m, &re[i0], &im[i0], &re[i1], &im[i1]);
    }
}

/* apply_single_cross_stride gate.cpp:187-216; controlled :244-277 */
static void cross_stride(uint64_t L, const double* m, int control, double* lre,
                         double* lim, double* hre, double* him)
{
    const uint64_t cbit = control >= 0 ? (uint64_t)1 << control : 0;
    for (uint64_t i = 0; i < L; ++i) {
        if (control >= 0 && !(i & cbit)) continue;
        pair_update(m, &lre[i], &lim[i], &hre[i], &him[i]);
    }
}

/* GateOp::validate, gate.cpp:109-137 */
static int validate_gate(int n, const qo_gate* g)
{
    switch (g->kind) {
        case 0:
        case 1:
            if (g->target < 0 || g->target >= n) return fail(QO_E_RANGE, "target qubit out of range");
            if (g->kind == 1) {
                if (g->control < 0 || g->control >= n)
                    return fail(QO_E_RANGE, "control qubit out of range");
                if (g->control == g->target)
                    return fail(QO_E_INVALID, "control qubit equals target qubit");
            }
            return 0;
        case 2:
            if (g->flip_index >= ((uint64_t)1 << n)) return fail(QO_E_RANGE, "flip index out of range");
            return 0;
        case 3:
            return 0;
        default:
            return fail(QO_E_INVALID, "unknown gate kind %d", g->kind);
    }
}

/* run_plan_unit, gate.cpp:405-454, for one unit of make_stride_plan. */
int qo_apply_unit(int n, int s, const qo_gate* g, uint64_t lo_index, double* lo_re,
                  double* lo_im, uint64_t hi_index, double* hi_re, double* hi_im,
                  double mean_re, double mean_im)
{
    int rc = validate_gate(n, g);
    if (rc) return rc;
    const uint64_t L = (uint64_t)1 << s;
    if (g->kind == 0 || g->kind == 1) {
        const int t = g->target;
        const int c = g->kind == 1 ? g->control : -1;
        if (t < s) {
            if (c < 0) in_stride(L, g->u, t, -1, lo_re, lo_im);           /* single */
            else if (c < s) in_stride(L, g->u, t, c, lo_re, lo_im);       /* controlled */
            else if (lo_index & ((uint64_t)1 << (c - s)))                 /* plain_single */
                in_stride(L, g->u, t, -1, lo_re, lo_im);
        } else {
            if (!hi_re) return fail(QO_E_INVALID, "pair unit needs both strides");
            if (c >= 0 && c < s) cross_stride(L, g->u, c, lo_re, lo_im, hi_re, hi_im);
            else if (c < 0 || (lo_index & ((uint64_t)1 << (c - s))))
                cross_stride(L, g->u, -1, lo_re, lo_im, hi_re, hi_im);
        }
        (void)hi_index;
        return 0;
    }
    if (g->kind == 2) {
        /* apply_phase_flip_in_stride gate.cpp:279-286 */
        if ((g->flip_index >> s) == lo_index) {
            const uint64_t off = g->flip_index & (L - 1);
            lo_re[off] = -lo_re[off];
            lo_im[off] = -lo_im[off];
        }
        return 0;
    }
    /* apply_reflect_mean_in_stride gate.cpp:288-301 */
    const double mr2 = 2.0 * mean_re, mi2 = 2.0 * mean_im;
    for (uint64_t i = 0; i < L; ++i) {
        lo_re[i] = mr2 - lo_re[i];
        lo_im[i] = mi2 - lo_im[i];
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* engine (aalc.cpp)                                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
    int codec;
    double delta;
    uint64_t count;
    uint8_t* payload;
    uint64_t len;
} block_t;

typedef struct {
    block_t re, im;
    double scale, sum_sq;
} stride_t;

struct qo_state {
    int n, s;
    uint64_t L, n_strides;
    stride_t* st;
    double norm_sq;
};

static uint64_t block_total(const block_t* b) { return QO_HEADER_BYTES + b->len; }

static void block_free(block_t* b)
{
    free(b->payload);
    b->payload = NULL;
    b->len = 0;
}

static int block_make(const double* x, uint64_t n, double delta, block_t* b)
{
    bytes_t out = {0};
    int rc = compress_any(x, n, delta, &out);
    if (rc) {
        free(out.p);
        return rc;
    }
    b->codec = delta == 0.0 ? 0 : 1;
    b->delta = delta;
    b->count = n;
    b->payload = out.p;
    b->len = out.len;
    return 0;
}

static void block_copy(const block_t* a, block_t* b)
{
    *b = *a;
    b->payload = a->len ? (uint8_t*)malloc(a->len) : NULL;
    if (a->len) memcpy(b->payload, a->payload, a->len);
}

static int block_decode(const block_t* b, double* out, uint64_t n)
{
    if (b->count != n) return fail(QO_E_INVALID, "output span does not match scalar count");
    return qo_decompress_payload(b->codec, b->delta, b->payload, b->len, out, n);
}

/* StrideBuffer::sum_sq, core.cpp:30-37 */
static double sum_sq(const double* re, const double* im, uint64_t L)
{
    double s = 0.0;
    for (uint64_t i = 0; i < L; ++i) s += re[i] * re[i] + im[i] * im[i];
    return s;
}

/* StrideBuffer::snap_zeros, core.cpp:39-47 (threshold core.hpp:22) */
static void snap_zeros(double* x, uint64_t L)
{
    for (uint64_t i = 0; i < L; ++i)
        if (fabs(x[i]) < 1e-300) x[i] = 0.0;
}

/* CompressedState::basis_state, aalc.cpp:140-174 */
int qo_state_create(int n, int s, uint64_t basis, qo_state** out)
{
    if (n < 1 || n > 59) return fail(QO_E_INVALID, "n_qubits must be in [1, 59], got %d", n);
    if (s < 0 || s > n) return fail(QO_E_INVALID, "stride_bits must be in [0, n_qubits], got %d", s);
    const int zero_state = basis == ~(uint64_t)0;  /* shard holding no amplitude */
    if (!zero_state && basis >= ((uint64_t)1 << n)) return fail(QO_E_RANGE, "basis index out of range");
    qo_state* st = (qo_state*)calloc(1, sizeof *st);
    st->n = n;
    st->s = s;
    st->L = (uint64_t)1 << s;
    st->n_strides = (uint64_t)1 << (n - s);
    st->st = (stride_t*)calloc(st->n_strides, sizeof(stride_t));
    double* buf = (double*)calloc(st->L, sizeof(double));
    block_t zero;
    block_make(buf, st->L, 0.0, &zero);
    const uint64_t hot = zero_state ? ~(uint64_t)0 : basis >> s;
    for (uint64_t j = 0; j < st->n_strides; ++j) {
        stride_t* t = &st->st[j];
        if (j == hot) {
            buf[basis & (st->L - 1)] = 1.0;
            block_make(buf, st->L, 0.0, &t->re);
            buf[basis & (st->L - 1)] = 0.0;
            block_make(buf, st->L, 0.0, &t->im);
            t->sum_sq = 1.0;
        } else {
            block_copy(&zero, &t->re);
            block_copy(&zero, &t->im);
            t->sum_sq = 0.0;
        }
        t->scale = 1.0;
    }
    block_free(&zero);
    free(buf);
    st->norm_sq = zero_state ? 0.0 : 1.0;
    *out = st;
    return 0;
}

void qo_state_destroy(qo_state* st)
{
    if (!st) return;
    for (uint64_t j = 0; j < st->n_strides; ++j) {
        block_free(&st->st[j].re);
        block_free(&st->st[j].im);
    }
    free(st->st);
    free(st);
}

int qo_state_clone(const qo_state* a, qo_state** out)
{
    qo_state* b = (qo_state*)calloc(1, sizeof *b);
    *b = *a;
    b->st = (stride_t*)calloc(a->n_strides, sizeof(stride_t));
    for (uint64_t j = 0; j < a->n_strides; ++j) {
        b->st[j] = a->st[j];
        block_copy(&a->st[j].re, &b->st[j].re);
        block_copy(&a->st[j].im, &b->st[j].im);
    }
    *out = b;
    return 0;
}

/* CompressedState::decompress_into, aalc.cpp:176-189 */
static int decompress_stride(const qo_state* st, uint64_t j, double* re, double* im,
                             int apply_scale)
{
    const stride_t* t = &st->st[j];
    int rc = block_decode(&t->re, re, st->L);
    if (!rc) rc = block_decode(&t->im, im, st->L);
    if (rc) return rc;
    if (apply_scale && t->scale != 1.0) {
        for (uint64_t i = 0; i < st->L; ++i) re[i] *= t->scale;
        for (uint64_t i = 0; i < st->L; ++i) im[i] *= t->scale;
    }
    return 0;
}

/* CompressedState::norm_sq_tracked, aalc.cpp:233-240 */
static double norm_sq_tracked(const qo_state* st)
{
    double total = 0.0;
    for (uint64_t j = 0; j < st->n_strides; ++j)
        total += st->st[j].scale * st->st[j].scale * st->st[j].sum_sq;
    return total;
}

typedef struct {
    uint64_t index;
    block_t re, im;
    double sum_sq;
} staged_t;

/* ErrorBoundLadder::make validation, aalc.cpp:56-72 */
static int check_ladder(const double* lad, int nl, double theta)
{
    if (nl <= 0) return fail(QO_E_INVALID, "error-bound ladder must not be empty");
    for (int i = 0; i < nl; ++i) {
        if (!(lad[i] >= 0.0) || !isfinite(lad[i]))
            return fail(QO_E_INVALID, "error bounds must be finite and >= 0");
        if (i > 0 && !(lad[i] > lad[i - 1]))
            return fail(QO_E_INVALID, "error bounds must be strictly increasing");
    }
    if (!(theta >= 1.0)) return fail(QO_E_INVALID, "ratio threshold must be >= 1");
    return 0;
}

/* CompressedState::apply_gate, aalc.cpp:261-420 (serial over units; the
 * reference result is independent of the worker count, aalc.hpp:127-129). */

int qo_apply_gate(qo_state* st, const qo_gate* g, const double* lad, int nl,
                  double theta, qo_report* reports, uint64_t* n_reports,
                  double* norm_after)
{
    return qo_apply_gate_ex(st, g, lad, nl, theta, 0, NULL, reports, n_reports, norm_after);
}

int qo_apply_gate_ex(qo_state* st, const qo_gate* g, const double* lad, int nl,
                     double theta, int flags, const double* given_mean, qo_report* reports,
                     uint64_t* n_reports, double* norm_after)
{
    const int no_renorm = flags & 1;
    int rc = validate_gate(st->n, g);
    if (rc) return rc;
    rc = check_ladder(lad, nl, theta);
    if (rc) return rc;
    const int s = st->s;
    const uint64_t L = st->L, NS = st->n_strides;

    /* make_stride_plan, gate.cpp:313-403 */
    uint64_t* lo = (uint64_t*)malloc(NS * sizeof(uint64_t));
    uint64_t* hi = (uint64_t*)malloc(NS * sizeof(uint64_t));
    int* is_pair = (int*)malloc(NS * sizeof(int));
    uint64_t nu = 0;
    int needs_mean = 0;
    if (g->kind == 0 || g->kind == 1) {
        const int t = g->target, c = g->kind == 1 ? g->control : -1;
        if (t < s) {
            const uint64_t cb = (c >= s) ? (uint64_t)1 << (c - s) : 0;
            for (uint64_t j = 0; j < NS; ++j)
                if (!cb || (j & cb)) { lo[nu] = j; is_pair[nu] = 0; ++nu; }
        } else {
            const uint64_t pb = (uint64_t)1 << (t - s);
            const uint64_t cb = (c >= s) ? (uint64_t)1 << (c - s) : 0;
            for (uint64_t j = 0; j < NS; ++j) {
                if (j & pb) continue;
                if (!cb || (j & cb)) { lo[nu] = j; hi[nu] = j | pb; is_pair[nu] = 1; ++nu; }
            }
        }
    } else if (g->kind == 2) {
        lo[0] = g->flip_index >> s;
        is_pair[0] = 0;
        nu = 1;
    } else {
        for (uint64_t j = 0; j < NS; ++j) { lo[nu] = j; is_pair[nu] = 0; ++nu; }
        needs_mean = 1;
    }

    double* a_re = (double*)malloc(L * sizeof(double));
    double* a_im = (double*)malloc(L * sizeof(double));
    double* b_re = (double*)malloc(L * sizeof(double));
    double* b_im = (double*)malloc(L * sizeof(double));

    /* mean pass, aalc.cpp:270-295 */
    double mean_re = 0.0, mean_im = 0.0;
    if (needs_mean && (flags & 2)) {
        mean_re = given_mean[0];
        mean_im = given_mean[1];
    } else if (needs_mean) {
        double sr_tot = 0.0, si_tot = 0.0;
        for (uint64_t j = 0; j < NS && !rc; ++j) {
            rc = decompress_stride(st, j, a_re, a_im, 1);
            double sr = 0.0, si = 0.0; /* stride_amplitude_sum gate.cpp:303-311 */
            for (uint64_t i = 0; i < L && !rc; ++i) {
                sr += a_re[i];
                si += a_im[i];
            }
            sr_tot += sr;
            si_tot += si;
        }
        const double na = (double)((uint64_t)1 << st->n);
        mean_re = sr_tot / na;
        mean_im = si_tot / na;
    }

    staged_t* stg = (staged_t*)calloc(2 * NS, sizeof(staged_t));
    uint64_t ns = 0, nr = 0;
    const uint64_t bytes_in = L * 16;
    for (uint64_t u = 0; u < nu && !rc; ++u) {
        rc = decompress_stride(st, lo[u], a_re, a_im, 1);
        if (rc) break;
        if (!is_pair[u]) {
            qo_apply_unit(st->n, s, g, lo[u], a_re, a_im, 0, NULL, NULL, mean_re, mean_im);
            /* compress_stride_adaptive, aalc.cpp:117-138 */
            snap_zeros(a_re, L);
            snap_zeros(a_im, L);
            block_t re = {0}, im = {0};
            double ratio = 0.0, chosen = 0.0;
            for (int k = 0; k < nl; ++k) {
                block_free(&re);
                block_free(&im);
                rc = block_make(a_re, L, lad[k], &re);
                if (!rc) rc = block_make(a_im, L, lad[k], &im);
                if (rc) break;
                chosen = lad[k];
                ratio = (double)bytes_in / (double)(block_total(&re) + block_total(&im));
                if (ratio >= theta) break;
            }
            if (rc) { block_free(&re); block_free(&im); break; }
            staged_t* sg = &stg[ns++];
            sg->index = lo[u];
            sg->re = re;
            sg->im = im;
            /* stored_sum_sq, aalc.cpp:46-52 */
            rc = block_decode(&re, a_re, L);
            if (!rc) rc = block_decode(&im, a_im, L);
            sg->sum_sq = sum_sq(a_re, a_im, L);
            if (reports) {
                qo_report* r = &reports[nr];
                r->stride_index = lo[u];
                r->chosen_delta = chosen;
                r->ratio = ratio;
                r->bytes_in = bytes_in;
                r->bytes_out = block_total(&re) + block_total(&im);
                r->threshold_met = ratio >= theta;
            }
            ++nr;
        } else {
            rc = decompress_stride(st, hi[u], b_re, b_im, 1);
            if (rc) break;
            qo_apply_unit(st->n, s, g, lo[u], a_re, a_im, hi[u], b_re, b_im, mean_re, mean_im);
            snap_zeros(a_re, L);
            snap_zeros(a_im, L);
            snap_zeros(b_re, L);
            snap_zeros(b_im, L);
            /* joint ladder, aalc.cpp:340-356 */
            block_t lr = {0}, li = {0}, hr = {0}, hii = {0};
            double chosen = 0.0, rlo = 0.0, rhi = 0.0;
            for (int k = 0; k < nl; ++k) {
                block_free(&lr); block_free(&li); block_free(&hr); block_free(&hii);
                rc = block_make(a_re, L, lad[k], &lr);
                if (!rc) rc = block_make(a_im, L, lad[k], &li);
                if (!rc) rc = block_make(b_re, L, lad[k], &hr);
                if (!rc) rc = block_make(b_im, L, lad[k], &hii);
                if (rc) break;
                chosen = lad[k];
                rlo = (double)bytes_in / (double)(block_total(&lr) + block_total(&li));
                rhi = (double)bytes_in / (double)(block_total(&hr) + block_total(&hii));
                if ((rlo < rhi ? rlo : rhi) >= theta) break;
            }
            if (rc) { block_free(&lr); block_free(&li); block_free(&hr); block_free(&hii); break; }
            staged_t* sl = &stg[ns++];
            sl->index = lo[u];
            sl->re = lr;
            sl->im = li;
            rc = block_decode(&lr, a_re, L);
            if (!rc) rc = block_decode(&li, a_im, L);
            sl->sum_sq = sum_sq(a_re, a_im, L);
            staged_t* sh = &stg[ns++];
            sh->index = hi[u];
            sh->re = hr;
            sh->im = hii;
            if (!rc) rc = block_decode(&hr, b_re, L);
            if (!rc) rc = block_decode(&hii, b_im, L);
            sh->sum_sq = sum_sq(b_re, b_im, L);
            if (reports) {
                qo_report* r = &reports[nr];
                r->stride_index = lo[u];
                r->chosen_delta = chosen;
                r->ratio = rlo;
                r->bytes_in = bytes_in;
                r->bytes_out = block_total(&lr) + block_total(&li);
                r->threshold_met = rlo >= theta;
                r = &reports[nr + 1];
                r->stride_index = hi[u];
                r->chosen_delta = chosen;
                r->ratio = rhi;
                r->bytes_in = bytes_in;
                r->bytes_out = block_total(&hr) + block_total(&hii);
                r->threshold_met = rhi >= theta;
            }
            nr += 2;
        }
    }

    if (rc) {
        /* error: nothing committed (aalc.cpp:309-393) */
        for (uint64_t i = 0; i < ns; ++i) { block_free(&stg[i].re); block_free(&stg[i].im); }
    } else {
        /* commit, aalc.cpp:395-408 */
        for (uint64_t i = 0; i < ns; ++i) {
            stride_t* t = &st->st[stg[i].index];
            block_free(&t->re);
            block_free(&t->im);
            t->re = stg[i].re;
            t->im = stg[i].im;
            t->sum_sq = stg[i].sum_sq;
            t->scale = 1.0;
        }
        /* lazy renormalisation, aalc.cpp:410-418 */
        const double total = no_renorm ? 0.0 : norm_sq_tracked(st);
        if (total > 0.0) {
            const double f = 1.0 / sqrt(total);
            for (uint64_t j = 0; j < NS; ++j) st->st[j].scale *= f;
        }
        st->norm_sq = norm_sq_tracked(st);
        if (norm_after) *norm_after = sqrt(st->norm_sq);
        if (n_reports) *n_reports = nr;
    }
    free(stg);
    free(a_re); free(a_im); free(b_re); free(b_im);
    free(lo); free(hi); free(is_pair);
    return rc;
}

/* CompressedState::to_amplitudes, aalc.cpp:211-223 */
int qo_to_amplitudes(const qo_state* st, double* amps)
{
    double* re = (double*)malloc(st->L * sizeof(double));
    double* im = (double*)malloc(st->L * sizeof(double));
    int rc = 0;
    for (uint64_t j = 0; j < st->n_strides && !rc; ++j) {
        rc = decompress_stride(st, j, re, im, 1);
        for (uint64_t i = 0; i < st->L && !rc; ++i) {
            amps[2 * (j * st->L + i)] = re[i];
            amps[2 * (j * st->L + i) + 1] = im[i];
        }
    }
    free(re);
    free(im);
    return rc;
}

/* stored_stride / decompress_stride, aalc.cpp:191-209 */
int qo_stored_stride(const qo_state* st, uint64_t j, int apply_scale, double* re, double* im)
{
    if (j >= st->n_strides) return fail(QO_E_RANGE, "stride index out of range");
    return decompress_stride(st, j, re, im, apply_scale);
}

/* compressed_bytes / min_stride_ratio / norm_sq_tracked, aalc.cpp:233-259 */
int qo_stats(const qo_state* st, uint64_t* bytes, double* min_ratio, double* norm_sq)
{
    uint64_t total = 0;
    double m = INFINITY;
    const uint64_t bytes_in = st->L * 16;
    for (uint64_t j = 0; j < st->n_strides; ++j) {
        const uint64_t b = block_total(&st->st[j].re) + block_total(&st->st[j].im);
        total += b;
        const double r = (double)bytes_in / (double)b;
        if (r < m) m = r;
    }
    if (bytes) *bytes = total;
    if (min_ratio) *min_ratio = m;
    if (norm_sq) *norm_sq = norm_sq_tracked(st);
    return 0;
}

int qo_stride_info(const qo_state* st, uint64_t j, double* scale, double* ssq,
                   uint64_t* re_payload, uint64_t* im_payload)
{
    if (j >= st->n_strides) return fail(QO_E_RANGE, "stride index out of range");
    if (scale) *scale = st->st[j].scale;
    if (ssq) *ssq = st->st[j].sum_sq;
    if (re_payload) *re_payload = st->st[j].re.len;
    if (im_payload) *im_payload = st->st[j].im.len;
    return 0;
}

int qo_export_blocks(const qo_state* st, uint64_t j, uint8_t* buf, uint64_t cap, uint64_t* len)
{
    if (j >= st->n_strides) return fail(QO_E_RANGE, "stride index out of range");
    const block_t* b[2] = {&st->st[j].re, &st->st[j].im};
    *len = block_total(b[0]) + block_total(b[1]);
    if (!buf) return 0;
    if (*len > cap) return fail(QO_E_CAPACITY, "output buffer too small");
    uint64_t off = 0;
    for (int k = 0; k < 2; ++k) {
        write_header(buf + off, b[k]->codec, b[k]->delta, b[k]->count, b[k]->len);
        off += QO_HEADER_BYTES;
        if (b[k]->len) memcpy(buf + off, b[k]->payload, b[k]->len);
        off += b[k]->len;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* dense oracle (dense.cpp)                                                 */
/* ------------------------------------------------------------------------ */

/* complex product (u * a) as libstdc++ evaluates it without -ffast-math:
 * re = ur*ar - ui*ai, im = ur*ai + ui*ar. */
static inline void cmul(double ur, double ui, double ar, double ai, double* r, double* i)
{
    *r = ur * ar - ui * ai;
    *i = ur * ai + ui * ar;
}

/* dense_apply, dense.cpp:30-76 */
static void dense_apply(int n, double* a, const qo_gate* g)
{
    const uint64_t N = (uint64_t)1 << n;
    const double* u = g->u;
    if (g->kind == 0 || g->kind == 1) {
        const uint64_t half = (uint64_t)1 << g->target;
        const uint64_t cbit = g->kind == 1 ? (uint64_t)1 << g->control : 0;
        for (uint64_t i = 0; i < N; ++i) {
            if (i & half) continue;
            if (g->kind == 1 && !(i & cbit)) continue;
            const double a0r = a[2 * i], a0i = a[2 * i + 1];
            const double a1r = a[2 * (i | half)], a1i = a[2 * (i | half) + 1];
            double pr, pi, qr, qi;
            cmul(u[0], u[1], a0r, a0i, &pr, &pi);
            cmul(u[2], u[3], a1r, a1i, &qr, &qi);
            a[2 * i] = pr + qr;
            a[2 * i + 1] = pi + qi;
            cmul(u[4], u[5], a0r, a0i, &pr, &pi);
            cmul(u[6], u[7], a1r, a1i, &qr, &qi);
            a[2 * (i | half)] = pr + qr;
            a[2 * (i | half) + 1] = pi + qi;
        }
    } else if (g->kind == 2) {
        a[2 * g->flip_index] = -a[2 * g->flip_index];
        a[2 * g->flip_index + 1] = -a[2 * g->flip_index + 1];
    } else {
        double sr = 0.0, si = 0.0;
        for (uint64_t i = 0; i < N; ++i) {
            sr += a[2 * i];
            si += a[2 * i + 1];
        }
        const double mr = 2.0 * (sr / (double)N), mi = 2.0 * (si / (double)N);
        for (uint64_t i = 0; i < N; ++i) {
            a[2 * i] = mr - a[2 * i];
            a[2 * i + 1] = mi - a[2 * i + 1];
        }
    }
}

/* run_dense, dense.cpp:78-92 */
int qo_dense_run(int n, const qo_gate* gates, uint64_t ng, uint64_t basis, double* amps)
{
    if (n < 1 || n > 30) return fail(QO_E_INVALID, "dense state supports 1 to 30 qubits");
    if (basis >= ((uint64_t)1 << n)) return fail(QO_E_RANGE, "basis index out of range");
    for (uint64_t k = 0; k < ng; ++k) {
        int rc = validate_gate(n, &gates[k]);
        if (rc) return rc;
    }
    memset(amps, 0, sizeof(double) * 2 * ((uint64_t)1 << n));
    amps[2 * basis] = 1.0;
    for (uint64_t k = 0; k < ng; ++k) dense_apply(n, amps, &gates[k]);
    return 0;
}

/* fidelity, dense.cpp:94-108 */
double qo_fidelity(const double* a, const double* b, uint64_t N)
{
    double na = 0.0, nb = 0.0;
    for (uint64_t i = 0; i < N; ++i) na += a[2 * i] * a[2 * i] + a[2 * i + 1] * a[2 * i + 1];
    for (uint64_t i = 0; i < N; ++i) nb += b[2 * i] * b[2 * i] + b[2 * i + 1] * b[2 * i + 1];
    na = sqrt(na);
    nb = sqrt(nb);
    if (na < 1e-150 || nb < 1e-150) return 0.0;
    double orr = 0.0, oi = 0.0;
    for (uint64_t i = 0; i < N; ++i) {
        orr += a[2 * i] * b[2 * i] + a[2 * i + 1] * b[2 * i + 1];
        oi += a[2 * i] * b[2 * i + 1] - a[2 * i + 1] * b[2 * i];
    }
    return hypot(orr, oi) / (na * nb);
}

/* ---- hooks for sharded (multi-rank) runs ---------------------------------- */
/* Per-stride stride_amplitude_sum (gate.cpp:303-311) of the scaled strides,
 * the terms of the mean pass (aalc.cpp:270-295). */
int qo_stride_sums(const qo_state* st, double* partial)
{
    const uint64_t L = st->L;
    double* re = (double*)malloc(L * sizeof(double));
    double* im = (double*)malloc(L * sizeof(double));
    int rc = 0;
    for (uint64_t j = 0; j < st->n_strides && !rc; ++j) {
        rc = decompress_stride(st, j, re, im, 1);
        double sr = 0.0, si = 0.0;
        for (uint64_t i = 0; i < L && !rc; ++i) {
            sr += re[i];
            si += im[i];
        }
        partial[2 * j] = sr;
        partial[2 * j + 1] = si;
    }
    free(re);
    free(im);
    return rc;
}

int qo_stride_norms(const qo_state* st, double* scales, double* sums)
{
    for (uint64_t j = 0; j < st->n_strides; ++j) {
        if (scales) scales[j] = st->st[j].scale;
        if (sums) sums[j] = st->st[j].sum_sq;
    }
    return 0;
}

int qo_scale_all(qo_state* st, double f)
{
    for (uint64_t j = 0; j < st->n_strides; ++j) st->st[j].scale *= f;
    return 0;
}

/* Inverse of qo_export_blocks: two serialized QCS1 blocks installed verbatim. */
int qo_import_blocks(qo_state* st, uint64_t j, const uint8_t* buf, uint64_t len, double scale,
                     double sum_sq)
{
    if (j >= st->n_strides) return fail(QO_E_RANGE, "stride index out of range");
    uint64_t off = 0;
    block_t b[2];
    for (int k = 0; k < 2; ++k) {
        uint64_t count, plen;
        int codec;
        double delta;
        const uint8_t* payload;
        int rc = parse_block(buf, len, &off, &codec, &delta, &count, &payload, &plen);
        if (rc) {
            if (k) block_free(&b[0]);
            return rc;
        }
        if (count != st->L) {
            if (k) block_free(&b[0]);
            return fail(QO_E_INVALID, "block length disagrees with geometry");
        }
        b[k].codec = codec;
        b[k].delta = delta;
        b[k].count = count;
        b[k].len = plen;
        b[k].payload = plen ? (uint8_t*)malloc(plen) : NULL;
        if (plen) memcpy(b[k].payload, payload, plen);
    }
    block_free(&st->st[j].re);
    block_free(&st->st[j].im);
    st->st[j].re = b[0];
    st->st[j].im = b[1];
    st->st[j].scale = scale;
    st->st[j].sum_sq = sum_sq;
    return 0;
}
