/*
 * tcxref — the CPU ORACLE for the tcx hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2206_02874_b200/) never links,
 * imports or calls it, and this file shares no code, header, table or helper with
 * paper_2206_02874_b200/csrc/.
 *
 * What it computes (plain definitions, written out; no blocking, fusion or reordering):
 *
 *   D = A x B + C                              PAPER.md:112 (§II-A, "performs D = A×B + C")
 *   A is m x k, B is k x n ("row.col": B is stored n x k, K-major)
 *
 *   FP (FP16 / BF16 / TF32 inputs, FP32 C/D):
 *     D_ij = RNE_fp32( c_ij + sum_k a_ik * b_kj )
 *     every product exact, the whole sum exact (a Kulisch fixed-point accumulator),
 *     exactly one rounding at the end.  (BASELINE.json north_star: "exact products summed
 *     in an exact-accumulator scheme followed by one final rounding to FP32").
 *   INT8 x INT8 -> INT32:
 *     D_ij = wrap32( c_ij + sum_k a_ik * b_kj ), summed exactly in int64.   (north_star:
 *     "INT8 inputs with INT32 accumulate ... two's-complement wraparound")
 *   2:4 sparse (the paper's mma.sp):
 *     A = expand(sA, e): every group of 4 consecutive K elements keeps 2 values at the
 *     2-bit positions stored in e; then the dense rule above.
 *
 *   Format rounding (SPEC.md:38-46 `quantize`): round-to-nearest-even of an exact value
 *   into FP32 / TF32 (8,10) / BF16 (8,7) / FP16 (5,10) — Table `datatypes`.
 *
 * Every function here is checked by tests/test_oracle_*.py against pins that do not
 * come from this file: brute-force rational arithmetic (fractions.Fraction), closed forms,
 * the paper's zero-error cells and SPEC worked examples (see oracle/README and DESIGN.md).
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <math.h>
#include <pthread.h>

/* format ids — mirrored in oracle/__init__.py (independent of include/tcx.h) */
enum { REF_F16 = 0, REF_BF16 = 1, REF_TF32 = 2, REF_F32 = 3, REF_S8 = 4, REF_S32 = 5 };

/* ------------------------------------------------------------------------------------ */
/* exact decode: value = (-1)^sign * mant * 2^exp                                         */
/* ------------------------------------------------------------------------------------ */
enum { CLS_ZERO = 0, CLS_FINITE = 1, CLS_INF = 2, CLS_NAN = 3 };
typedef struct { int cls; int sign; uint64_t mant; int exp; } refnum;

static refnum decode_bits(int fmt, uint32_t b) {
  refnum r = {CLS_ZERO, 0, 0, 0};
  uint32_t e, f;
  int ebits, fbits, bias;
  switch (fmt) {
    case REF_F16:  ebits = 5; fbits = 10; bias = 15;  b &= 0xFFFFu; break;
    case REF_BF16: ebits = 8; fbits = 7;  bias = 127; b &= 0xFFFFu; break;
    /* TF32 lives in a 32-bit container; the stored bits are read exactly as
       FP32 — the API requires TF32-representable values (low 13 bits zero). */
    case REF_TF32:
    case REF_F32:  ebits = 8; fbits = 23; bias = 127; break;
    default: r.cls = CLS_NAN; return r;
  }
  r.sign = (int)(b >> (ebits + fbits)) & 1;
  e = (b >> fbits) & ((1u << ebits) - 1u);
  f = b & ((1u << fbits) - 1u);
  if (e == (1u << ebits) - 1u) { r.cls = f ? CLS_NAN : CLS_INF; return r; }
  if (e == 0) {
    if (f == 0) { r.cls = CLS_ZERO; return r; }
    r.cls = CLS_FINITE; r.mant = f; r.exp = 1 - bias - fbits; return r;       /* subnormal */
  }
  r.cls = CLS_FINITE; r.mant = f | (1u << fbits); r.exp = (int)e - bias - fbits;
  return r;
}

/* ------------------------------------------------------------------------------------ */
/* big fixed-point magnitude: little-endian u64 words, bit i has weight 2^(i + LSB_EXP)    */
/* ------------------------------------------------------------------------------------ */
#define KW 12                 /* 768 bits */
#define LSB_EXP (-330)        /* FP32*FP32 subnormal products reach 2^-298; FP32 max 2^128*2^128;
                                 768 bits cover [2^-330, 2^438): room for K up to 2^150 terms */
typedef struct { uint64_t w[KW]; } bigmag;

static void big_add_shifted(bigmag *a, uint64_t mant, int shift) {
  /* a += mant << shift, shift >= 0 */
  int word = shift >> 6, bit = shift & 63;
  uint64_t lo = mant << bit;
  uint64_t hi = bit ? (mant >> (64 - bit)) : 0;
  uint64_t carry = 0;
  int i;
  uint64_t s = a->w[word] + lo;
  carry = s < lo;
  a->w[word] = s;
  for (i = word + 1; i < KW; i++) {
    uint64_t add = (i == word + 1) ? hi : 0;
    uint64_t t = a->w[i] + add;
    uint64_t c1 = t < add;
    uint64_t t2 = t + carry;
    uint64_t c2 = t2 < carry;
    a->w[i] = t2;
    carry = c1 | c2;
    if (!carry && i > word + 1) break;
  }
}

static int big_cmp(const bigmag *a, const bigmag *b) {
  int i;
  for (i = KW - 1; i >= 0; i--) {
    if (a->w[i] != b->w[i]) return a->w[i] > b->w[i] ? 1 : -1;
  }
  return 0;
}

static void big_sub(bigmag *r, const bigmag *a, const bigmag *b) { /* r = a - b, a >= b */
  uint64_t borrow = 0;
  int i;
  for (i = 0; i < KW; i++) {
    uint64_t x = a->w[i], y = b->w[i];
    uint64_t d = x - y;
    uint64_t b1 = x < y;
    uint64_t d2 = d - borrow;
    uint64_t b2 = d < borrow;
    r->w[i] = d2;
    borrow = b1 | b2;
  }
}

static int big_msb(const uint64_t *w, int n) {  /* index of highest set bit, -1 if zero */
  int i;
  for (i = n - 1; i >= 0; i--) {
    if (w[i]) return i * 64 + 63 - __builtin_clzll(w[i]);
  }
  return -1;
}

static int big_bit(const uint64_t *w, int n, int i) {
  if (i < 0 || i >= n * 64) return 0;
  return (int)((w[i >> 6] >> (i & 63)) & 1u);
}

static int big_any_below(const uint64_t *w, int n, int i) { /* any bit in [0, i) set */
  int k;
  if (i <= 0) return 0;
  for (k = 0; k < (i >> 6) && k < n; k++) if (w[k]) return 1;
  if ((i & 63) && (i >> 6) < n) {
    uint64_t m = (1ull << (i & 63)) - 1ull;
    if (w[i >> 6] & m) return 1;
  }
  return 0;
}

static uint64_t big_extract(const uint64_t *w, int n, int lo, int nbits) { /* bits [lo, lo+nbits), nbits<=63 */
  uint64_t r = 0;
  int i;
  for (i = 0; i < nbits; i++) r |= (uint64_t)big_bit(w, n, lo + i) << i;
  return r;
}

/* ------------------------------------------------------------------------------------ */
/* round an exact magnitude (words, lsb weight 2^lsb_exp) to a binary format, RNE or RZ.  */
/* P = significand bits incl. hidden, emin/emax = min/max normal exponent.                */
/* returns 0 ok (kept * 2^qexp), 1 overflow (infinity), 2 zero.                           */
/* ------------------------------------------------------------------------------------ */
typedef struct { int P, emin, emax, ebits, fbits, bias; } fmtinfo;

static fmtinfo fmt_info(int fmt) {
  fmtinfo f;
  switch (fmt) {
    case REF_F16:  f.P = 11; f.emin = -14;  f.emax = 15;  f.ebits = 5; f.fbits = 10; f.bias = 15;  break;
    case REF_BF16: f.P = 8;  f.emin = -126; f.emax = 127; f.ebits = 8; f.fbits = 7;  f.bias = 127; break;
    case REF_TF32: f.P = 11; f.emin = -126; f.emax = 127; f.ebits = 8; f.fbits = 10; f.bias = 127; break;
    default:       f.P = 24; f.emin = -126; f.emax = 127; f.ebits = 8; f.fbits = 23; f.bias = 127; break;
  }
  return f;
}

static int round_mag(const uint64_t *w, int n, int lsb_exp, fmtinfo fi, int rz,
                     uint64_t *kept_out, int *qexp_out) {
  int p = big_msb(w, n);
  int E, qexp, q;
  uint64_t kept;
  if (p < 0) return 2;
  E = p + lsb_exp;
  qexp = E - (fi.P - 1);
  if (qexp < fi.emin - (fi.P - 1)) qexp = fi.emin - (fi.P - 1);
  q = qexp - lsb_exp;
  if (q <= 0) {
    kept = big_extract(w, n, 0, p + 1) << (-q);
  } else {
    int rbit, sticky;
    kept = big_extract(w, n, q, p - q + 1 > 0 ? p - q + 1 : 0);
    rbit = big_bit(w, n, q - 1);
    sticky = big_any_below(w, n, q - 1);
    if (!rz && rbit && (sticky || (kept & 1u))) kept++;
    if (kept == (1ull << fi.P)) { kept >>= 1; qexp++; }
  }
  if (kept == 0) return 2;
  if (kept >= (1ull << (fi.P - 1)) && qexp + fi.P - 1 > fi.emax) return 1;
  *kept_out = kept; *qexp_out = qexp;
  return 0;
}

static uint32_t encode_bits(int fmt, int sign, int status, uint64_t kept, int qexp) {
  fmtinfo fi = fmt_info(fmt);
  uint32_t s = (uint32_t)sign, bits;
  uint32_t expall = (1u << fi.ebits) - 1u;
  if (status == 2) bits = s << (fi.ebits + fi.fbits);
  else if (status == 1) bits = (s << (fi.ebits + fi.fbits)) | (expall << fi.fbits);
  else if (kept >= (1ull << (fi.P - 1))) {
    uint32_t be = (uint32_t)(qexp + fi.P - 1 + fi.bias);
    bits = (s << (fi.ebits + fi.fbits)) | (be << fi.fbits) | (uint32_t)(kept - (1ull << (fi.P - 1)));
  } else {
    bits = (s << (fi.ebits + fi.fbits)) | (uint32_t)kept;   /* subnormal */
  }
  if (fmt == REF_TF32) bits <<= 13;   /* TF32 in its 32-bit container, low 13 bits zero */
  return bits;
}

static uint32_t nan_bits(int fmt) {
  switch (fmt) {
    case REF_F16: case REF_BF16: return fmt == REF_F16 ? 0x7E00u : 0x7FC0u;
    default: return 0x7FC00000u;
  }
}

/* quantize(x, fmt, mode) — SPEC.md:38-46.  x is an exact binary64 value. */
uint32_t tcxref_quantize(double x, int fmt, int rz) {
  uint64_t u, mant, w[2] = {0, 0};
  int e, sign, status, qexp = 0;
  uint64_t kept = 0;
  memcpy(&u, &x, 8);
  sign = (int)(u >> 63);
  e = (int)((u >> 52) & 0x7FF);
  mant = u & ((1ull << 52) - 1);
  if (e == 0x7FF) {
    if (mant) return nan_bits(fmt);
    return encode_bits(fmt, sign, 1, 0, 0);
  }
  if (e == 0) { if (mant == 0) return encode_bits(fmt, sign, 2, 0, 0); e = 1; }
  else mant |= 1ull << 52;
  w[0] = mant;
  status = round_mag(w, 2, e - 1075, fmt_info(fmt), rz, &kept, &qexp);
  if (status == 1 && rz) {   /* round toward zero never overflows to inf: max finite */
    fmtinfo fi = fmt_info(fmt);
    return encode_bits(fmt, sign, 0, (1ull << fi.P) - 1, fi.emax - (fi.P - 1));
  }
  return encode_bits(fmt, sign, status, kept, qexp);
}

/* decode to binary64 (exact for every format here) */
double tcxref_decode(int fmt, uint32_t b) {
  refnum r;
  if (fmt == REF_S8) return (double)(int8_t)(b & 0xFF);
  if (fmt == REF_S32) return (double)(int32_t)b;
  r = decode_bits(fmt, b);
  if (r.cls == CLS_NAN) return NAN;
  if (r.cls == CLS_INF) return r.sign ? -INFINITY : INFINITY;
  if (r.cls == CLS_ZERO) return r.sign ? -0.0 : 0.0;
  return (r.sign ? -1.0 : 1.0) * ldexp((double)r.mant, r.exp);
}

/* ------------------------------------------------------------------------------------ */
/* one FP output element:  RNE_fp32(c + sum_k a_k*b_k), exactly                            */
/* a, b: element bits (16- or 32-bit containers); c: FP32 bits                             */
/* abs_out (optional): sum_k |a_k b_k| + |c| rounded down to binary64 (for the FP bound)   */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  bigmag pos, neg, absacc;
  int any_nan, pinf, ninf, all_negzero;
} kacc;

static void kacc_init(kacc *k) { memset(k, 0, sizeof(*k)); k->all_negzero = 1; }

static void kacc_add(kacc *k, int sign, uint64_t mant, int exp) {
  int shift = exp - LSB_EXP;
  big_add_shifted(sign ? &k->neg : &k->pos, mant, shift);
  big_add_shifted(&k->absacc, mant, shift);
}

static void kacc_add_product(kacc *k, refnum a, refnum b) {
  int s = a.sign ^ b.sign;
  if (a.cls == CLS_NAN || b.cls == CLS_NAN) { k->any_nan = 1; return; }
  if (a.cls == CLS_INF || b.cls == CLS_INF) {
    if (a.cls == CLS_ZERO || b.cls == CLS_ZERO) { k->any_nan = 1; return; }   /* inf * 0 */
    if (s) k->ninf = 1; else k->pinf = 1;
    return;
  }
  if (a.cls == CLS_ZERO || b.cls == CLS_ZERO) { if (!s) k->all_negzero = 0; return; }
  k->all_negzero = 0;
  /* exact product: significands <= 24 bits each -> <= 48 bits */
  kacc_add(k, s, a.mant * b.mant, a.exp + b.exp);
}

static void kacc_add_value(kacc *k, refnum c) {
  if (c.cls == CLS_NAN) { k->any_nan = 1; return; }
  if (c.cls == CLS_INF) { if (c.sign) k->ninf = 1; else k->pinf = 1; return; }
  if (c.cls == CLS_ZERO) { if (!c.sign) k->all_negzero = 0; return; }
  k->all_negzero = 0;
  kacc_add(k, c.sign, c.mant, c.exp);
}

static double big_to_double_down(const bigmag *m) {
  int p = big_msb(m->w, KW);
  uint64_t top;
  if (p < 0) return 0.0;
  if (p < 53) return ldexp((double)big_extract(m->w, KW, 0, p + 1), LSB_EXP);
  top = big_extract(m->w, KW, p - 52, 53);
  return ldexp((double)top, p - 52 + LSB_EXP);
}

static uint32_t kacc_round(kacc *k, int out_fmt, int rz, double *abs_out) {
  bigmag mag;
  int sign, status, qexp = 0, c;
  uint64_t kept = 0;
  if (abs_out) *abs_out = big_to_double_down(&k->absacc);
  if (k->any_nan || (k->pinf && k->ninf)) return nan_bits(out_fmt);
  if (k->pinf) return encode_bits(out_fmt, 0, 1, 0, 0);
  if (k->ninf) return encode_bits(out_fmt, 1, 1, 0, 0);
  c = big_cmp(&k->pos, &k->neg);
  if (c == 0) return encode_bits(out_fmt, k->all_negzero, 2, 0, 0);  /* exact zero: +0 unless all addends -0 */
  if (c > 0) { big_sub(&mag, &k->pos, &k->neg); sign = 0; }
  else       { big_sub(&mag, &k->neg, &k->pos); sign = 1; }
  status = round_mag(mag.w, KW, LSB_EXP, fmt_info(out_fmt), rz, &kept, &qexp);
  if (status == 1 && rz) {
    fmtinfo fi = fmt_info(out_fmt);
    return encode_bits(out_fmt, sign, 0, (1ull << fi.P) - 1, fi.emax - (fi.P - 1));
  }
  return encode_bits(out_fmt, sign, status, kept, qexp);
}

static inline uint32_t load_elem(const void *p, int64_t i, int fmt) {
  switch (fmt) {
    case REF_F16: case REF_BF16: return ((const uint16_t *)p)[i];
    case REF_S8: return (uint32_t)(uint8_t)((const int8_t *)p)[i];
    default: return ((const uint32_t *)p)[i];
  }
}

/* D element (i,j):  a = A + i*lda (K elems), b = B + j*ldb (K elems, "col" B = N x K)
   General form: c given in c_fmt (FP32, or FP16 for the FP16-accumulate MMA variant of
   PAPER.md:428-429 / Table FP16-FP16-numeric-profiling), the exact sum rounded ONCE into
   out_fmt (FP32 or FP16) with RNE (rz = 0) or toward zero (rz = 1). */
uint32_t tcxref_dot_fp2(int ab, int64_t K, const void *a, const void *b, int c_fmt, uint32_t c_bits,
                        int out_fmt, int rz, double *abs_out) {
  kacc k;
  int64_t t;
  kacc_init(&k);
  for (t = 0; t < K; t++)
    kacc_add_product(&k, decode_bits(ab, load_elem(a, t, ab)), decode_bits(ab, load_elem(b, t, ab)));
  kacc_add_value(&k, decode_bits(c_fmt, c_bits));
  return kacc_round(&k, out_fmt, rz, abs_out);
}

uint32_t tcxref_dot_fp(int ab, int64_t K, const void *a, const void *b, uint32_t c_bits, double *abs_out) {
  return tcxref_dot_fp2(ab, K, a, b, REF_F32, c_bits, REF_F32, 0, abs_out);
}

int32_t tcxref_dot_s8(int64_t K, const int8_t *a, const int8_t *b, int32_t c) {
  int64_t s = c, t;
  for (t = 0; t < K; t++) s += (int64_t)a[t] * (int64_t)b[t];
  return (int32_t)(uint32_t)(uint64_t)s;    /* two's-complement wrap */
}

/* exact sum of arbitrary FP32 addends, rounded once (RNE or RZ) into out_fmt.
   Used by the probe-model family (oracle/models.c) and by tests. */
uint32_t tcxref_sum_round(int n, const int *signs, const uint64_t *mants, const int *exps,
                          int out_fmt, int rz) {
  kacc k;
  int i;
  kacc_init(&k);
  for (i = 0; i < n; i++) {
    refnum r;
    r.cls = mants[i] ? CLS_FINITE : CLS_ZERO; r.sign = signs[i]; r.mant = mants[i]; r.exp = exps[i];
    kacc_add_value(&k, r);
  }
  return kacc_round(&k, out_fmt, rz, NULL);
}

/* ------------------------------------------------------------------------------------ */
/* GEMM on a list of sampled output coordinates, multi-threaded.                          */
/* A: M x K (lda), B: N x K (ldb), C: M x N (ldc) or NULL (zeros).                         */
/* out[s] = D[rows[s], cols[s]] bits; abs_out[s] (optional, FP only) = bound magnitude.   */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  int ab; int64_t K; const void *A; int64_t lda; const void *B; int64_t ldb;
  const void *C; int64_t ldc; const int64_t *rows, *cols; uint32_t *out; double *abs_out;
  int64_t s0, s1; int cd;   /* cd: REF_F32 (FP32 C/D; INT32 for S8) or REF_F16 (FP16 C/D) */
} job_t;

static void *gemm_worker(void *arg) {
  job_t *j = (job_t *)arg;
  int64_t s;
  size_t es = (j->ab == REF_S8) ? 1 : ((j->ab == REF_F16 || j->ab == REF_BF16) ? 2 : 4);
  for (s = j->s0; s < j->s1; s++) {
    int64_t r = j->rows[s], c = j->cols[s];
    const char *a = (const char *)j->A + (size_t)(r * j->lda) * es;
    const char *b = (const char *)j->B + (size_t)(c * j->ldb) * es;
    uint32_t cb = 0u;
    if (j->C) cb = j->cd == REF_F16 ? ((const uint16_t *)j->C)[r * j->ldc + c] : ((const uint32_t *)j->C)[r * j->ldc + c];
    if (j->ab == REF_S8) {
      j->out[s] = (uint32_t)tcxref_dot_s8(j->K, (const int8_t *)a, (const int8_t *)b, (int32_t)cb);
    } else {
      double ab = 0.0;
      j->out[s] = tcxref_dot_fp2(j->ab, j->K, a, b, j->cd, cb, j->cd, 0, &ab);
      if (j->abs_out) j->abs_out[s] = ab;
    }
  }
  return NULL;
}

int tcxref_gemm_samples2(int ab, int cd, int64_t K, const void *A, int64_t lda, const void *B, int64_t ldb,
                         const void *C, int64_t ldc, int64_t nsamp, const int64_t *rows,
                         const int64_t *cols, uint32_t *out, double *abs_out, int nthreads) {
  pthread_t th[256];
  job_t jobs[256];
  int t;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  for (t = 0; t < nthreads; t++) {
    job_t *j = &jobs[t];
    j->ab = ab; j->K = K; j->A = A; j->lda = lda; j->B = B; j->ldb = ldb; j->C = C; j->ldc = ldc;
    j->rows = rows; j->cols = cols; j->out = out; j->abs_out = abs_out; j->cd = cd == REF_F16 ? REF_F16 : REF_F32;
    j->s0 = nsamp * t / nthreads; j->s1 = nsamp * (t + 1) / nthreads;
    if (nthreads == 1) { gemm_worker(j); return 0; }
    if (pthread_create(&th[t], NULL, gemm_worker, j)) return -1;
  }
  for (t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  return 0;
}

int tcxref_gemm_samples(int ab, int64_t K, const void *A, int64_t lda, const void *B, int64_t ldb,
                        const void *C, int64_t ldc, int64_t nsamp, const int64_t *rows,
                        const int64_t *cols, uint32_t *out, double *abs_out, int nthreads) {
  return tcxref_gemm_samples2(ab, REF_F32, K, A, lda, B, ldb, C, ldc, nsamp, rows, cols, out, abs_out, nthreads);
}

/* ------------------------------------------------------------------------------------ */
/* 2:4 structured sparsity                            */
/* canonical metadata: u32 words, K/32 per row; group g (dense cols 4g..4g+3) is the       */
/* nibble at bits 4*(g%8) of word g/8, nibble = i0 | i1<<2, i0 < i1 ("lowest-order bit-pair */
/* = first kept element").                                      */
/* ------------------------------------------------------------------------------------ */

/* expand: sA (M x K/2, ld_vals) + meta -> dense A (M x K, lda).  esize = element bytes.
   returns -1 on success, else the first (row*G + group) whose nibble has i0 >= i1. */
int64_t tcxref_sp24_expand(int esize, int64_t M, int64_t K, const void *vals, int64_t ld_vals,
                           const uint32_t *meta, void *dense, int64_t lda) {
  int64_t i, g, G = K / 4;
  for (i = 0; i < M; i++) {
    char *drow = (char *)dense + (size_t)(i * lda) * esize;
    const char *vrow = (const char *)vals + (size_t)(i * ld_vals) * esize;
    memset(drow, 0, (size_t)K * esize);
    for (g = 0; g < G; g++) {
      uint32_t nib = (meta[i * (K / 32) + g / 8] >> (4 * (g % 8))) & 0xFu;
      int i0 = nib & 3, i1 = (nib >> 2) & 3;
      if (i0 >= i1) return i * G + g;
      memcpy(drow + (size_t)(4 * g + i0) * esize, vrow + (size_t)(2 * g) * esize, esize);
      memcpy(drow + (size_t)(4 * g + i1) * esize, vrow + (size_t)(2 * g + 1) * esize, esize);
    }
  }
  return -1;
}

static int is_nonzero(int esize, const char *p) {
  /* +-0 is zero; NaN and everything else is nonzero (SURVEY §8(b) error conventions) */
  if (esize == 1) return *(const int8_t *)p != 0;
  if (esize == 2) return ((*(const uint16_t *)p) & 0x7FFFu) != 0;
  return ((*(const uint32_t *)p) & 0x7FFFFFFFu) != 0;
}

/* compress_24: keep the <=2 nonzeros of each group, pad under-full
   groups with the lowest free indices; reject a group with >2 nonzeros.
   returns -1 on success, else first violating row*G + group (row-major order). */
int64_t tcxref_sp24_compress(int esize, int64_t M, int64_t K, const void *dense, int64_t lda,
                             void *vals, int64_t ld_vals, uint32_t *meta) {
  int64_t i, g, G = K / 4;
  memset(meta, 0, (size_t)(M * (K / 32)) * sizeof(uint32_t));
  for (i = 0; i < M; i++) {
    const char *drow = (const char *)dense + (size_t)(i * lda) * esize;
    char *vrow = (char *)vals + (size_t)(i * ld_vals) * esize;
    for (g = 0; g < G; g++) {
      int idx[4], n = 0, p;
      for (p = 0; p < 4; p++) if (is_nonzero(esize, drow + (size_t)(4 * g + p) * esize)) idx[n++] = p;
      if (n > 2) return i * G + g;
      /* pad with the lowest free indices */
      for (p = 0; p < 4 && n < 2; p++) {
        int used = 0, q;
        for (q = 0; q < n; q++) if (idx[q] == p) used = 1;
        if (!used) idx[n++] = p;
      }
      if (idx[0] > idx[1]) { int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
      memcpy(vrow + (size_t)(2 * g) * esize, drow + (size_t)(4 * g + idx[0]) * esize, esize);
      memcpy(vrow + (size_t)(2 * g + 1) * esize, drow + (size_t)(4 * g + idx[1]) * esize, esize);
      meta[i * (K / 32) + g / 8] |= (uint32_t)(idx[0] | (idx[1] << 2)) << (4 * (g % 8));
    }
  }
  return -1;
}

/* TF32 sparsity is 1:2 in hardware (DESIGN.md R-C12: the paper lists TF32 mma.sp shapes,
   PAPER.md:619-620, without the rule): every aligned PAIR along K keeps one element — its nonzero,
   or its lower element when both are zero; a pair with two nonzeros is a violation.  The kept
   pair positions are written in the canonical 2:4 nibble (i0 in {0,1}, i1 in {2,3}).
   returns -1 on success, else the first violating row*G + group (G = K/4, row-major order). */
int64_t tcxref_sp12_compress(int64_t M, int64_t K, const uint32_t *dense, int64_t lda, uint32_t *vals,
                             int64_t ld_vals, uint32_t *meta) {
  int64_t i, g, G = K / 4;
  memset(meta, 0, (size_t)(M * (K / 32)) * sizeof(uint32_t));
  for (i = 0; i < M; i++) {
    const uint32_t *d = dense + i * lda;
    for (g = 0; g < G; g++) {
      int nz[4], p, i0, i1;
      for (p = 0; p < 4; p++) nz[p] = is_nonzero(4, (const char *)&d[4 * g + p]);
      if ((nz[0] && nz[1]) || (nz[2] && nz[3])) return i * G + g;
      i0 = (nz[1] && !nz[0]) ? 1 : 0;
      i1 = (nz[3] && !nz[2]) ? 3 : 2;
      vals[i * ld_vals + 2 * g] = d[4 * g + i0];
      vals[i * ld_vals + 2 * g + 1] = d[4 * g + i1];
      meta[i * (K / 32) + g / 8] |= (uint32_t)(i0 | (i1 << 2)) << (4 * (g % 8));
    }
  }
  return -1;
}

/* ------------------------------------------------------------------------------------ */
/* tile batch (tcx_mma_tiles semantics): D_t = A_t B_t + C_t, t < count.                   */
/* A_t: m x k row-major, B_t: n x k ("col"), C_t/D_t: m x n row-major.                      */
/* ------------------------------------------------------------------------------------ */
/* cd = REF_F32 (C/D FP32 bits; INT32 for S8) or REF_F16 (C/D stored as 16-bit FP16: the
   FP16-accumulate mma variant, D = RNE_fp16(c + sum a*b) exactly, "converts the
   final result to low-precision FP16 in the end"). */
int tcxref_tiles2(int ab, int cd, int m, int n, int k, int64_t count, const void *A, const void *B,
                  const void *C, uint32_t *D, double *abs_out) {
  int64_t t;
  int i, j;
  size_t es = (ab == REF_S8) ? 1 : ((ab == REF_F16 || ab == REF_BF16) ? 2 : 4);
  for (t = 0; t < count; t++) {
    for (i = 0; i < m; i++) for (j = 0; j < n; j++) {
      const char *a = (const char *)A + ((size_t)t * m * k + (size_t)i * k) * es;
      const char *b = (const char *)B + ((size_t)t * n * k + (size_t)j * k) * es;
      int64_t o = t * m * n + i * n + j;
      uint32_t cb = 0u;
      if (C) cb = cd == REF_F16 ? ((const uint16_t *)C)[o] : ((const uint32_t *)C)[o];
      if (ab == REF_S8) D[o] = (uint32_t)tcxref_dot_s8(k, (const int8_t *)a, (const int8_t *)b, (int32_t)cb);
      else {
        double av = 0.0;
        D[o] = tcxref_dot_fp2(ab, k, a, b, cd == REF_F16 ? REF_F16 : REF_F32, cb, cd == REF_F16 ? REF_F16 : REF_F32,
                              0, &av);
        if (abs_out) abs_out[o] = av;
      }
    }
  }
  return 0;
}

int tcxref_tiles(int ab, int m, int n, int k, int64_t count, const void *A, const void *B,
                 const void *C, uint32_t *D, double *abs_out) {
  return tcxref_tiles2(ab, REF_F32, m, n, k, count, A, B, C, D, abs_out);
}

/* ------------------------------------------------------------------------------------ */
/* chain matrix multiplication (Fig. code-chain-matmul)              */
/* ------------------------------------------------------------------------------------ */
/* FP32 bits -> fmt bits, RNE (the chain's conversion of D_{i-1} into the next A_i). */
void tcxref_quantize_f32_bits(int fmt, int64_t n, const uint32_t *in, uint32_t *out) {
  int64_t i;
  for (i = 0; i < n; i++) {
    float f;
    memcpy(&f, &in[i], 4);
    out[i] = tcxref_quantize((double)f, fmt, 0);
  }
}

/* The paper's CPU baseline "D^FP32": the same chain computed on the CPU in
   binary32 — D_i = A_i x B_i with each element a sequential binary32 dot (ascending k, no FMA
   contraction: built with -ffp-contract=off), and A_{i+1} = D_i with no conversion.
   A0: count x 16 x 8 floats; Bs: count x n_steps x 8 x 8 (n x k); Ds: count x n_steps x 16 x 8. */
void tcxref_chain_fp32(int64_t count, int n_steps, const float *A0, const float *Bs, float *Ds) {
  int64_t c;
  for (c = 0; c < count; c++) {
    float a[16 * 8];
    int s, i, j, k;
    memcpy(a, A0 + c * 128, sizeof(a));
    for (s = 0; s < n_steps; s++) {
      const float *b = Bs + (c * n_steps + s) * 64;
      float *d = Ds + (c * n_steps + s) * 128;
      for (i = 0; i < 16; i++)
        for (j = 0; j < 8; j++) {
          float acc = 0.0f;
          for (k = 0; k < 8; k++) {
            volatile float p = a[i * 8 + k] * b[j * 8 + k];
            acc = acc + p;
          }
          d[i * 8 + j] = acc;
        }
      memcpy(a, d, sizeof(a));
    }
  }
}
