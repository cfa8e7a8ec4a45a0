/*
 * tcxref models — TEST INFRASTRUCTURE ONLY (see tcxref.c header).
 *
 * The numeric-probe (config 2) hypothesis family.  The paper profiles the three operations
 * inside one tensor-core MMA — multiplication, inner-product addition, accumulation
 * addition (Figs. mul/addInnerProduct/addAccum) — and reads its tables
 * as "products and inner sums in high precision, accumulation in relatively low precision"
 * and "computation in high precision, converted only at the end"
 * (PAPER.md:982).  It never states the widths or rounding modes, so B200 behaviour is not
 * assumed: each GPU output element is classified against the bit-exact CPU models below
 * (SURVEY §8(c) "Model family for the C2 classifier"; reading R-C3).
 *
 *   M(g, p, R, t, o):
 *     the k products of one instruction (Ki of them) are processed in blocks of g;
 *     o = c-in-block: a block's addends are {acc, p_k .. p_{k+g-1}}, acc starts at c;
 *       e_max = exponent of the leading bit of the largest-magnitude addend;
 *       every addend is truncated to a multiple of 2^(e_max - 23 - p)
 *       (t = toward zero, or floor); p = -1 means no truncation (infinite precision);
 *       the truncated addends are summed exactly and rounded once to FP32 with R
 *       (RNE or RZ) -> the new acc.
 *     o = c-after: the block's products alone are aligned/truncated/summed exactly to S,
 *       then acc = R(acc + S) (a separate accumulation stage).
 *     Across chained instructions (K > Ki) acc is carried as FP32.
 *   Special cases: exact oracle = M(Ki, inf, RNE, -, c-in-block) for one instruction.
 *
 *   seq32: the paper's CPU FP32 baseline ("FP32 result on CPU"), read as
 *   sequential binary32 in ascending k, c first or c last.
 */
#include <stdint.h>
#include <string.h>

enum { REF_F16 = 0, REF_BF16 = 1, REF_TF32 = 2, REF_F32 = 3 };

/* from tcxref.c */
uint32_t tcxref_sum_round(int n, const int *signs, const uint64_t *mants, const int *exps,
                          int out_fmt, int rz);

typedef struct { int zero; int sign; uint64_t mant; int exp; int eu; int nlead; int fe; } term;
/* eu: unbiased exponent of an input (emin for subnormals); 1000 marks the accumulator term.
   nlead: 'nominal' leading-bit exponent used by the exponent-sum alignment variants:
   emode 1: product = eu_a + eu_b + 1 (a product of two [1,2) significands lies in [1,4)),
            accumulator / c = its actual leading bit;
   emode 2: as 1, but the accumulator / c is also placed in the 2-integer-bit frame (lead + 1).
   emode 3: as 2, but the accumulator's exponent is read from its exponent FIELD, like the inputs':
            a subnormal accumulator / c counts as emin (fe), not as its actual leading bit. */

static term dec(int fmt, uint32_t b) {
  term t = {1, 0, 0, 0, 0, 0, 0};
  int ebits, fbits, bias;
  uint32_t e, f;
  if (fmt == REF_F16) { ebits = 5; fbits = 10; bias = 15; b &= 0xFFFF; }
  else if (fmt == REF_BF16) { ebits = 8; fbits = 7; bias = 127; b &= 0xFFFF; }
  else { ebits = 8; fbits = 23; bias = 127; }
  t.sign = (b >> (ebits + fbits)) & 1;
  e = (b >> fbits) & ((1u << ebits) - 1);
  f = b & ((1u << fbits) - 1);
  t.eu = e == 0 ? 1 - bias : (int)e - bias;
  t.fe = t.eu;
  if (e == 0 && f == 0) return t;
  t.zero = 0;
  if (e == 0) { t.mant = f; t.exp = 1 - bias - fbits; }
  else { t.mant = f | (1u << fbits); t.exp = (int)e - bias - fbits; }
  /* inf/nan are not part of the probe classes (generators keep everything finite) */
  return t;
}

static int lead_exp(term t) { return t.exp + 63 - __builtin_clzll(t.mant); }

/* truncate t to a multiple of 2^L (toward zero, or floor) */
static term trunc_to(term t, int L, int floor_mode) {
  int sh;
  uint64_t m, dropped;
  if (t.zero || t.exp >= L) return t;
  sh = L - t.exp;
  if (sh >= 64) { m = 0; dropped = t.mant; }
  else { m = t.mant >> sh; dropped = t.mant & ((1ull << sh) - 1ull); }
  if (floor_mode && t.sign && dropped) m += 1;
  t.mant = m; t.exp = L;
  if (m == 0) t.zero = 1;
  return t;
}

static uint32_t sum_terms(int n, const term *ts, int rz, int out_fmt) {
  int s[72], e[72], i, k = 0;
  uint64_t m[72];
  for (i = 0; i < n; i++) {
    if (ts[i].zero) continue;
    s[k] = ts[i].sign; m[k] = ts[i].mant; e[k] = ts[i].exp; k++;
  }
  return tcxref_sum_round(k, s, m, e, out_fmt, rz);
}

/* the accumulator term, held in acc_fmt (FP32, or FP16 for the FP16-accumulate variant) */
static term from_acc(uint32_t b, int acc_fmt) {
  term t = dec(acc_fmt, b);
  if (!t.zero) t.nlead = lead_exp(t);
  t.eu = 1000;                                               /* marks the accumulator term */
  return t;
}

/* align + truncate a set of terms relative to their largest addend */
static void align_trunc(int n, term *ts, int p, int floor_mode, int emode, int frac_bits) {
  int i, emax = -100000, L;
  if (p < 0) return;
  for (i = 0; i < n; i++)
    if (!ts[i].zero) {
      int le = emode ? ts[i].nlead : lead_exp(ts[i]);
      if (emode == 3 && ts[i].eu == 1000 && ts[i].fe > le) le = ts[i].fe;   /* field exponent (subnormal: emin) */
      if (emode >= 2 && ts[i].eu == 1000) le += 1;          /* accumulator / c: 2-integer-bit format */
      if (le > emax) emax = le;
    }
  if (emax == -100000) return;
  L = emax - frac_bits - p;
  for (i = 0; i < n; i++) ts[i] = trunc_to(ts[i], L, floor_mode);
}

/* M(g, p, R, t, o) with the accumulator (c in, D out) held in acc_fmt: FP32 or FP16 (the
   FP16-accumulate mma variant).  The truncation window is p bits below win_fmt's significand
   (FP32: 23 fraction bits, FP16: 10) at the block's leading exponent; each block's truncated
   addends are summed exactly and rounded ONCE into acc_fmt.  win_fmt = acc_fmt is the plain
   family; win_fmt = FP32 with acc_fmt = FP16 is "aligned like the FP32 datapath, rounded once
   into FP16" (no intermediate FP32 rounding — the alternative to the two-stage M32 -> RNE16). */
uint32_t tcxref_model_dot4(int ab, int K, const void *a, const void *b, uint32_t c_bits,
                           int Ki, int g, int p, int rz, int floor_mode, int c_after, int emode, int acc_fmt,
                           int win_fmt) {
  uint32_t acc = c_bits;
  int k0, j;
  const int frac_bits = win_fmt == REF_F16 ? 10 : 23;
  for (k0 = 0; k0 < K; k0 += Ki) {           /* one instruction */
    int kk;
    for (kk = 0; kk < Ki && k0 + kk < K; kk += g) {   /* one block */
      term ts[72];
      int n = 0;
      if (!c_after) ts[n++] = from_acc(acc, acc_fmt);
      for (j = 0; j < g && kk + j < Ki && k0 + kk + j < K; j++) {
        int idx = k0 + kk + j;
        uint32_t ab_bits = (ab == REF_F16 || ab == REF_BF16) ? ((const uint16_t *)a)[idx] : ((const uint32_t *)a)[idx];
        uint32_t bb_bits = (ab == REF_F16 || ab == REF_BF16) ? ((const uint16_t *)b)[idx] : ((const uint32_t *)b)[idx];
        term x = dec(ab, ab_bits), y = dec(ab, bb_bits), pr;
        pr.zero = x.zero || y.zero; pr.sign = x.sign ^ y.sign;
        pr.mant = pr.zero ? 0 : x.mant * y.mant; pr.exp = x.exp + y.exp;
        pr.eu = 0; pr.nlead = x.eu + y.eu + 1; pr.fe = 0;
        ts[n++] = pr;
      }
      align_trunc(n, ts, p, floor_mode, emode, frac_bits);
      if (!c_after) {
        acc = sum_terms(n, ts, rz, acc_fmt);
      } else {
        /* products summed exactly among themselves, then one rounding of acc + S */
        term all[73];
        memcpy(all, ts, sizeof(term) * n);
        all[n] = from_acc(acc, acc_fmt);
        acc = sum_terms(n + 1, all, rz, acc_fmt);
      }
    }
  }
  return acc;
}

uint32_t tcxref_model_dot3(int ab, int K, const void *a, const void *b, uint32_t c_bits,
                           int Ki, int g, int p, int rz, int floor_mode, int c_after, int emode, int acc_fmt) {
  return tcxref_model_dot4(ab, K, a, b, c_bits, Ki, g, p, rz, floor_mode, c_after, emode, acc_fmt, acc_fmt);
}

uint32_t tcxref_model_dot2(int ab, int K, const void *a, const void *b, uint32_t c_bits,
                           int Ki, int g, int p, int rz, int floor_mode, int c_after, int emode) {
  return tcxref_model_dot3(ab, K, a, b, c_bits, Ki, g, p, rz, floor_mode, c_after, emode, REF_F32);
}

uint32_t tcxref_model_dot(int ab, int K, const void *a, const void *b, uint32_t c_bits,
                          int Ki, int g, int p, int rz, int floor_mode, int c_after) {
  return tcxref_model_dot2(ab, K, a, b, c_bits, Ki, g, p, rz, floor_mode, c_after, 0);
}

/* the paper's CPU FP32 baseline: sequential binary32 (no FMA contraction; built with
   -ffp-contract=off), ascending k, c first (c_last=0) or last (c_last=1). */
float tcxref_seq32(int K, const float *a, const float *b, float c, int c_last) {
  float acc = c_last ? 0.0f : c;
  int k;
  for (k = 0; k < K; k++) {
    volatile float prod = a[k] * b[k];
    acc = acc + prod;
  }
  if (c_last) acc = acc + c;
  return acc;
}

/* batched model evaluation over n dot products (rows of a and b: n x K element bits), threaded. */
#include <pthread.h>
typedef struct {
  int ab, K; const void *a, *b; const uint32_t *c; int Ki, g, p, rz, floor_mode, c_after, emode, acc_fmt, win_fmt;
  uint32_t *out; long s0, s1;
} mjob;

static void *mworker(void *arg) {
  mjob *j = (mjob *)arg;
  long i;
  size_t es = (j->ab == REF_F16 || j->ab == REF_BF16) ? 2 : 4;
  for (i = j->s0; i < j->s1; i++)
    j->out[i] = tcxref_model_dot4(j->ab, j->K, (const char *)j->a + (size_t)i * j->K * es,
                                  (const char *)j->b + (size_t)i * j->K * es, j->c[i], j->Ki, j->g, j->p,
                                  j->rz, j->floor_mode, j->c_after, j->emode, j->acc_fmt, j->win_fmt);
  return NULL;
}

int tcxref_model_batch3(int ab, long n, int K, const void *a, const void *b, const uint32_t *c, int Ki, int g,
                        int p, int rz, int floor_mode, int c_after, int emode, int acc_fmt, int win_fmt,
                        uint32_t *out, int nthreads) {
  pthread_t th[256];
  mjob jobs[256];
  int t;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  for (t = 0; t < nthreads; t++) {
    mjob *j = &jobs[t];
    j->ab = ab; j->K = K; j->a = a; j->b = b; j->c = c; j->Ki = Ki; j->g = g; j->p = p; j->rz = rz;
    j->floor_mode = floor_mode; j->c_after = c_after; j->emode = emode; j->acc_fmt = acc_fmt;
    j->win_fmt = win_fmt; j->out = out;
    j->s0 = n * t / nthreads; j->s1 = n * (t + 1) / nthreads;
    if (pthread_create(&th[t], NULL, mworker, j)) return -1;
  }
  for (t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  return 0;
}

int tcxref_model_batch2(int ab, long n, int K, const void *a, const void *b, const uint32_t *c, int Ki, int g,
                        int p, int rz, int floor_mode, int c_after, int emode, int acc_fmt, uint32_t *out,
                        int nthreads) {
  return tcxref_model_batch3(ab, n, K, a, b, c, Ki, g, p, rz, floor_mode, c_after, emode, acc_fmt, acc_fmt, out,
                             nthreads);
}

int tcxref_model_batch(int ab, long n, int K, const void *a, const void *b, const uint32_t *c, int Ki, int g,
                       int p, int rz, int floor_mode, int c_after, int emode, uint32_t *out, int nthreads) {
  return tcxref_model_batch2(ab, n, K, a, b, c, Ki, g, p, rz, floor_mode, c_after, emode, REF_F32, out, nthreads);
}
