/*
 * twofold_oracle.c — TEST INFRASTRUCTURE, not product code.
 *
 * A plain-C restatement of the reference's twofold arithmetic on the hot path,
 * used only as the CPU checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg.  The product (libtwofold_b200.so) never
 * links or calls it.
 *
 * Parity pin: every function here is checked bit-exact against golden vectors
 * produced by the reference package itself (numba cores imported from
 * /root/reference, script tests/golden/make_golden.py) — see
 * tests/test_oracle_golden.py.
 *
 * Build flags are part of the algorithm (fp_core.py:29-32: no fastmath):
 *   -ffp-contract=off -fno-fast-math   (no a*b+c contraction, IEEE RN)
 * fma() is the correctly rounded C99 fma (glibc; hardware VFMADD under -mfma),
 * the analogue of the llvm.fma intrinsic (fp_core.py:83-101).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/twofold_b200.h"

#if defined(__FP_FAST_FMA) || defined(__FMA__)
#define HW_FMA 1
#endif

/* ------------------------------------------------------------------------ */
/* exact transforms (fp_core.py:134-185) and twofold cores (arith.py:61-218),
   generic over float/double through a macro "template".                      */

#define DEFINE_CORES(T, S, FMA, SQRT)                                          \
  typedef struct { T a, b; } pair_##S;                                         \
  static inline pair_##S mk_##S(T a, T b) { pair_##S p = {a, b}; return p; }   \
  /* fp_core.py:134-139 */                                                     \
  static inline pair_##S fast_two_sum_##S(T a, T b) {                          \
    T s = a + b; T bv = s - a; return mk_##S(s, b - bv); }                     \
  /* fp_core.py:142-149 */                                                     \
  static inline pair_##S two_sum_##S(T a, T b) {                               \
    T s = a + b; T bv = s - a; T av = s - bv; T br = b - bv; T ar = a - av;    \
    return mk_##S(s, ar + br); }                                               \
  /* fp_core.py:160-167 */                                                     \
  static inline pair_##S two_diff_##S(T a, T b) {                              \
    T d = a - b; T bv = a - d; T av = d + bv; T br = bv - b; T ar = a - av;    \
    return mk_##S(d, ar + br); }                                               \
  /* fp_core.py:170-173 */                                                     \
  static inline pair_##S two_prod_##S(T a, T b) {                              \
    T p = a * b; return mk_##S(p, FMA(a, b, -p)); }                            \
  /* fp_core.py:176-179 */                                                     \
  static inline pair_##S div_rem_##S(T a, T b) {                               \
    T q = a / b; return mk_##S(q, FMA(-q, b, a)); }                            \
  /* fp_core.py:182-185 */                                                     \
  static inline pair_##S sqrt_resid_##S(T a) {                                 \
    T c = SQRT(a); return mk_##S(c, FMA(-c, c, a)); }                          \
  /* arith.py:61-64 */                                                         \
  static inline pair_##S tadd_##S(T x0, T x1, T y0, T y1) {                    \
    pair_##S e = two_sum_##S(x0, y0); return mk_##S(e.a, (x1 + y1) + e.b); }   \
  /* arith.py:67-71 */                                                         \
  static inline pair_##S tadd1_##S(T x0, T x1, T y) {                          \
    pair_##S e = two_sum_##S(x0, y); return mk_##S(e.a, x1 + e.b); }           \
  /* arith.py:74-77 */                                                         \
  static inline pair_##S tsub_##S(T x0, T x1, T y0, T y1) {                    \
    pair_##S e = two_diff_##S(x0, y0); return mk_##S(e.a, (x1 - y1) + e.b); }  \
  /* arith.py:80-83 */                                                         \
  static inline pair_##S tsub1_##S(T x0, T x1, T y) {                          \
    pair_##S e = two_diff_##S(x0, y); return mk_##S(e.a, x1 + e.b); }          \
  /* arith.py:86-94 */                                                         \
  static inline pair_##S tmul_##S(T x0, T x1, T y0, T y1) {                    \
    pair_##S p = two_prod_##S(x0, y0);                                         \
    T p01 = x0 * y1; T p10 = x1 * y0; T p11 = x1 * y1;                         \
    return mk_##S(p.a, (p.b + p11) + (p01 + p10)); }                           \
  /* arith.py:97-101 */                                                        \
  static inline pair_##S tmul1_##S(T x0, T x1, T y) {                          \
    pair_##S p = two_prod_##S(x0, y); T p10 = x1 * y;                          \
    return mk_##S(p.a, p.b + p10); }                                           \
  /* arith.py:104-110 */                                                       \
  static inline pair_##S pmul_##S(T x0, T x1, T y0, T y1) {                    \
    pair_##S p = two_prod_##S(x0, y0); T p01 = x0 * y1; T p10 = x1 * y0;       \
    return mk_##S(p.a, p.b + (p01 + p10)); }                                   \
  /* arith.py:113-117 */                                                       \
  static inline pair_##S tdiv0_##S(T x, T y) {                                 \
    T q = x / y; T r = FMA(-q, y, x); return mk_##S(q, r / y); }               \
  /* arith.py:120-124 */                                                       \
  static inline pair_##S tdiv1_##S(T x0, T x1, T y) {                          \
    T q = x0 / y; T r = FMA(-q, y, x0); return mk_##S(q, (r + x1) / y); }      \
  /* arith.py:127-132 */                                                       \
  static inline pair_##S tdiv_##S(T x0, T x1, T y0, T y1) {                    \
    T q = x0 / y0; T r0 = FMA(-q, y0, x0); T r1 = FMA(-q, y1, x1);             \
    return mk_##S(q, (r0 + r1) / (y0 + y1)); }                                 \
  /* arith.py:135-142 */                                                       \
  static inline pair_##S pdiv_##S(T x0, T x1, T y0, T y1) {                    \
    T q = x0 / y0; T r0 = FMA(-q, y0, x0); T r1 = FMA(-q, y1, x1);             \
    return mk_##S(q, (r0 + r1) / y0); }                                        \
  /* arith.py:145-149 */                                                       \
  static inline pair_##S tsqrt0_##S(T x) {                                     \
    T c = SQRT(x); T d = FMA(-c, c, x); return mk_##S(c, d / (c + c)); }       \
  /* arith.py:152-157 */                                                       \
  static inline pair_##S psqrt_##S(T x0, T x1) {                               \
    T c = SQRT(x0); T d = FMA(-c, c, x0); return mk_##S(c, (x1 + d) / (c + c)); } \
  /* arith.py:160-168 */                                                       \
  static inline pair_##S tsqrt_##S(T x0, T x1) {                               \
    T z0 = SQRT(x0); pair_##S u = two_sum_##S(x0, x1);                         \
    pair_##S v = psqrt_##S(u.a, u.b); pair_##S w = tsub1_##S(v.a, v.b, z0);    \
    return mk_##S(z0, w.a + w.b); }                                            \
  /* arith.py:171-192 */                                                       \
  static inline pair_##S padd_##S(T x0, T x1, T y0, T y1) {                    \
    pair_##S z = tadd_##S(x0, x1, y0, y1); return fast_two_sum_##S(z.a, z.b); } \
  static inline pair_##S padd1_##S(T x0, T x1, T y) {                          \
    pair_##S z = tadd1_##S(x0, x1, y); return fast_two_sum_##S(z.a, z.b); }    \
  static inline pair_##S psub_##S(T x0, T x1, T y0, T y1) {                    \
    pair_##S z = tsub_##S(x0, x1, y0, y1); return fast_two_sum_##S(z.a, z.b); } \
  static inline pair_##S psub1_##S(T x0, T x1, T y) {                          \
    pair_##S z = tsub1_##S(x0, x1, y); return fast_two_sum_##S(z.a, z.b); }    \
  /* arith.py:195-206 */                                                       \
  static inline pair_##S pmul_coupled_##S(T x0, T x1, T y0, T y1) {            \
    pair_##S z = pmul_##S(x0, x1, y0, y1); return two_sum_##S(z.a, z.b); }     \
  static inline pair_##S pmul1_##S(T x0, T x1, T y) {                          \
    pair_##S z = tmul1_##S(x0, x1, y); return two_sum_##S(z.a, z.b); }         \
  /* arith.py:209-218 */                                                       \
  static inline pair_##S pdiv_coupled_##S(T x0, T x1, T y0, T y1) {            \
    pair_##S z = pdiv_##S(x0, x1, y0, y1); return fast_two_sum_##S(z.a, z.b); } \
  static inline pair_##S pdiv1_##S(T x0, T x1, T y) {                          \
    pair_##S z = tdiv1_##S(x0, x1, y); return fast_two_sum_##S(z.a, z.b); }

DEFINE_CORES(double, d, fma, sqrt)
DEFINE_CORES(float, f, fmaf, sqrtf)

/* ------------------------------------------------------------------------ */
/* loop drivers (kernels.py:79-113), one per arity, OpenMP-sharded            */

#define LOOP22(S, T, CORE)                                                     \
  { const T *x0 = in[0], *x1 = in[1], *y0 = in[2], *y1 = in[3];                \
    T *r0 = out[0], *r1 = out[1];                                              \
    _Pragma("omp parallel for schedule(static) num_threads(nt)")              \
    for (int64_t i = 0; i < n; i++) {                                          \
      pair_##S z = CORE##_##S(x0[i], x1[i], y0[i], y1[i]); r0[i] = z.a; r1[i] = z.b; } \
    return 0; }
#define LOOP21(S, T, CORE)                                                     \
  { const T *x0 = in[0], *x1 = in[1], *y = in[2];                              \
    T *r0 = out[0], *r1 = out[1];                                              \
    _Pragma("omp parallel for schedule(static) num_threads(nt)")              \
    for (int64_t i = 0; i < n; i++) {                                          \
      pair_##S z = CORE##_##S(x0[i], x1[i], y[i]); r0[i] = z.a; r1[i] = z.b; } \
    return 0; }
#define LOOP11(S, T, CORE)                                                     \
  { const T *x = in[0], *y = in[1];                                            \
    T *r0 = out[0], *r1 = out[1];                                              \
    _Pragma("omp parallel for schedule(static) num_threads(nt)")              \
    for (int64_t i = 0; i < n; i++) {                                          \
      pair_##S z = CORE##_##S(x[i], y[i]); r0[i] = z.a; r1[i] = z.b; }         \
    return 0; }
#define LOOP1U(S, T, CORE)                                                     \
  { const T *x = in[0];                                                        \
    T *r0 = out[0], *r1 = out[1];                                              \
    _Pragma("omp parallel for schedule(static) num_threads(nt)")              \
    for (int64_t i = 0; i < n; i++) {                                          \
      pair_##S z = CORE##_##S(x[i]); r0[i] = z.a; r1[i] = z.b; }               \
    return 0; }

#define DEFINE_ELEMENTWISE(S, T)                                               \
  static int elementwise_##S(int op, int64_t n, const void* const* in_,        \
                             void* const* out_, int nt) {                      \
    const T* const* in = (const T* const*)in_; T* const* out = (T* const*)out_; \
    switch (op) {                                                              \
      case TF_VTADD2: LOOP22(S, T, tadd)                                       \
      case TF_VTSUB2: LOOP22(S, T, tsub)                                       \
      case TF_VTMUL2: LOOP22(S, T, tmul)                                       \
      case TF_VTDIV2: LOOP22(S, T, tdiv)                                       \
      case TF_VTADD1: LOOP21(S, T, tadd1)                                      \
      case TF_VTSUB1: LOOP21(S, T, tsub1)                                      \
      case TF_VTMUL1: LOOP21(S, T, tmul1)                                      \
      case TF_VTDIV1: LOOP21(S, T, tdiv1)                                      \
      case TF_VTADD: LOOP11(S, T, two_sum)                                     \
      case TF_VTSUB: LOOP11(S, T, two_diff)                                    \
      case TF_VTMUL: LOOP11(S, T, two_prod)                                    \
      case TF_VTDIV: LOOP11(S, T, tdiv0)                                       \
      case TF_VTSQRT1: LOOP11(S, T, tsqrt)                                     \
      case TF_VTSQRT: LOOP1U(S, T, tsqrt0)                                     \
      case TF_VPADD2: LOOP22(S, T, padd)                                       \
      case TF_VPSUB2: LOOP22(S, T, psub)                                       \
      case TF_VPMUL2: LOOP22(S, T, pmul_coupled)                               \
      case TF_VPDIV2: LOOP22(S, T, pdiv_coupled)                               \
      case TF_VPADD1: LOOP21(S, T, padd1)                                      \
      case TF_VPSUB1: LOOP21(S, T, psub1)                                      \
      case TF_VPMUL1: LOOP21(S, T, pmul1)                                      \
      case TF_VPDIV1: LOOP21(S, T, pdiv1)                                      \
      case TF_DIVREM: LOOP11(S, T, div_rem)                                    \
      case TF_SQRTRESID: LOOP1U(S, T, sqrt_resid)                              \
      default: return -1;                                                      \
    }                                                                          \
  }

DEFINE_ELEMENTWISE(d, double)
DEFINE_ELEMENTWISE(f, float)

static int clamp_threads(int nt) {
#ifdef _OPENMP
  if (nt <= 0) nt = omp_get_max_threads();
#else
  nt = 1;
#endif
  return nt < 1 ? 1 : nt;
}

int tfo_elementwise(int op, int dtype, int64_t n, const void* const* in,
                    void* const* out, int nthreads) {
  if (n < 0) return -1;
  int nt = clamp_threads(nthreads);
  if (dtype == TF_F64) return elementwise_d(op, n, in, out, nt);
  if (dtype == TF_F32) return elementwise_f(op, n, in, out, nt);
  return -1;
}

/* dotted baselines vadd/vmul/vdiv/vsqrt/vmem (bench.py:56-87) */
int tfo_dotted(int base, int dtype, int64_t n, const void* x_, const void* y_,
               void* r_, int nthreads) {
  int nt = clamp_threads(nthreads);
#define DOTTED(T, SQ)                                                          \
  { const T *x = x_, *y = y_; T* r = r_;                                       \
    switch (base) {                                                            \
      case 0: _Pragma("omp parallel for num_threads(nt)") for (int64_t i = 0; i < n; i++) r[i] = x[i] + y[i]; return 0; \
      case 1: _Pragma("omp parallel for num_threads(nt)") for (int64_t i = 0; i < n; i++) r[i] = x[i] * y[i]; return 0; \
      case 2: _Pragma("omp parallel for num_threads(nt)") for (int64_t i = 0; i < n; i++) r[i] = x[i] / y[i]; return 0; \
      case 3: _Pragma("omp parallel for num_threads(nt)") for (int64_t i = 0; i < n; i++) r[i] = SQ(x[i]); return 0; \
      case 4: _Pragma("omp parallel for num_threads(nt)") for (int64_t i = 0; i < n; i++) r[i] = x[i]; return 0; \
      default: return -1; } }
  if (dtype == TF_F64) DOTTED(double, sqrt)
  if (dtype == TF_F32) DOTTED(float, sqrtf)
#undef DOTTED
  return -1;
}

/* ------------------------------------------------------------------------ */
/* canonical-order reductions (fold precedent demos.py:107-113)    */

/* adjacent-pair (stride-doubling) tree over m present items, lower index on
   the left, an item without a partner passes through unchanged */
#define DEFINE_TREE(S, T)                                                      \
  static pair_##S tree_##S(pair_##S* a, int64_t m) {                           \
    for (int64_t stride = 1; stride < m; stride *= 2)                          \
      for (int64_t i = 0; i + stride < m; i += 2 * stride)                     \
        a[i] = tadd_##S(a[i].a, a[i].b, a[i + stride].a, a[i + stride].b);     \
    return a[0];                                                               \
  }
DEFINE_TREE(d, double)
DEFINE_TREE(f, float)

/* one tile: lanes fold their elements (k-major, v-minor), then the lane tree */
#define DEFINE_TILE(S, T)                                                      \
  static pair_##S tile_##S(int rop, int64_t n, const T* a, const T* b,         \
                           int64_t base, int V, int W, int K, pair_##S* lanes) { \
    int64_t m = 0;                                                             \
    for (int w = 0; w < W; w++) {                                              \
      int have = 0; pair_##S acc = mk_##S(0, 0);                               \
      for (int k = 0; k < K; k++) {                                            \
        for (int v = 0; v < V; v++) {                                          \
          int64_t i = base + (int64_t)V * (w + (int64_t)W * k) + v;            \
          if (i >= n) continue;                                                \
          pair_##S t;                                                          \
          if (rop == TF_RSUM) {                                                \
            if (!have) { acc = mk_##S(a[i], (T)0); have = 1; continue; }       \
            acc = tadd1_##S(acc.a, acc.b, a[i]); continue;                     \
          }                                                                    \
          t = (rop == TF_RSUM2) ? mk_##S(a[i], b[i]) : two_prod_##S(a[i], b[i]); \
          if (!have) { acc = t; have = 1; continue; }                          \
          acc = tadd_##S(acc.a, acc.b, t.a, t.b);                              \
        }                                                                      \
      }                                                                        \
      if (!have) break; /* lanes past the end are empty (a suffix) */          \
      lanes[m++] = acc;                                                        \
    }                                                                          \
    return tree_##S(lanes, m);                                                 \
  }
DEFINE_TILE(d, double)
DEFINE_TILE(f, float)

#define DEFINE_REDUCE(S, T)                                                    \
  static int reduce_##S(int rop, int64_t n, const T* a, const T* b, int V,     \
                        int W, int K, T* out, T* tiles_out, int nt) {          \
    int64_t L = (int64_t)V * W * K;                                            \
    if (n == 0) { out[0] = (T)0; out[1] = (T)0; return 0; }                    \
    int64_t nt_tiles = (n + L - 1) / L;                                        \
    pair_##S* tiles = malloc(sizeof(pair_##S) * nt_tiles);                     \
    if (!tiles) return -3;                                                     \
    _Pragma("omp parallel num_threads(nt)")                                    \
    {                                                                          \
      pair_##S* lanes = malloc(sizeof(pair_##S) * W);                          \
      _Pragma("omp for schedule(static)")                                      \
      for (int64_t t = 0; t < nt_tiles; t++)                                   \
        tiles[t] = tile_##S(rop, n, a, b, t * L, V, W, K, lanes);              \
      free(lanes);                                                             \
    }                                                                          \
    if (tiles_out)                                                             \
      for (int64_t t = 0; t < nt_tiles; t++) {                                 \
        tiles_out[2 * t] = tiles[t].a; tiles_out[2 * t + 1] = tiles[t].b; }    \
    pair_##S r = tree_##S(tiles, nt_tiles);                                    \
    out[0] = r.a; out[1] = r.b;                                                \
    free(tiles);                                                               \
    return 0;                                                                  \
  }
DEFINE_REDUCE(d, double)
DEFINE_REDUCE(f, float)

int tfo_reduce(int rop, int dtype, int64_t n, const void* a, const void* b,
               int V, int W, int K, void* out, void* tiles_out, int nthreads) {
  if (n < 0 || V < 1 || W < 1 || K < 1 || rop < 0 || rop >= TF_NUM_ROPS) return -1;
  int nt = clamp_threads(nthreads);
  if (dtype == TF_F64) return reduce_d(rop, n, a, b, V, W, K, out, tiles_out, nt);
  if (dtype == TF_F32) return reduce_f(rop, n, a, b, V, W, K, out, tiles_out, nt);
  return -1;
}

/* cross-shard combine: the same tree over shards, empty shards skipped */
int tfo_combine(int dtype, int g, const void* partials, const int64_t* counts,
                void* out) {
  if (g < 0) return -1;
#define COMBINE(S, T)                                                          \
  { const T* p = partials; pair_##S* a = malloc(sizeof(pair_##S) * (g + 1));   \
    int64_t m = 0;                                                             \
    for (int r = 0; r < g; r++) if (counts[r] > 0) a[m++] = mk_##S(p[2 * r], p[2 * r + 1]); \
    pair_##S z = m ? tree_##S(a, m) : mk_##S(0, 0);                            \
    ((T*)out)[0] = z.a; ((T*)out)[1] = z.b; free(a); return 0; }
  if (dtype == TF_F64) COMBINE(d, double)
  if (dtype == TF_F32) COMBINE(f, float)
#undef COMBINE
  return -1;
}

/* ------------------------------------------------------------------------ */
/* fused expression chains (demos.py:153-238), one instance per element       */

#define DEFINE_FUSED(S, T)                                                     \
  static int fused_##S(int fop, int64_t n, const T* const* in, T* const* out, int nt) { \
    if (fop == 0 || fop == 1) {                                                \
      _Pragma("omp parallel for schedule(static) num_threads(nt)")            \
      for (int64_t i = 0; i < n; i++) {                                        \
        pair_##S z;                                                            \
        if (fop == 0) { /* tadd(tmul(a, x), y) */                              \
          pair_##S m = tmul_##S(in[0][i], in[1][i], in[2][i], in[3][i]);       \
          z = tadd_##S(m.a, m.b, in[4][i], in[5][i]);                          \
        } else { /* tsub(c, tmul(a, b)) */                                     \
          pair_##S m = tmul_##S(in[2][i], in[3][i], in[4][i], in[5][i]);       \
          z = tsub_##S(in[0][i], in[1][i], m.a, m.b);                          \
        }                                                                      \
        out[0][i] = z.a; out[1][i] = z.b;                                      \
      }                                                                        \
      return 0;                                                                \
    }                                                                          \
    if (fop == 2) { /* demos.py:222-229 */                                     \
      _Pragma("omp parallel for schedule(static) num_threads(nt)")            \
      for (int64_t i = 0; i < n; i++) {                                        \
        T a0 = in[0][i], a1 = in[1][i], b0 = in[2][i], b1 = in[3][i];          \
        T c0 = in[4][i], c1 = in[5][i];                                        \
        pair_##S bb = tmul_##S(b0, b1, b0, b1);                                \
        pair_##S fa = tmul_##S((T)4, (T)0, a0, a1);                            \
        pair_##S fac = tmul_##S(fa.a, fa.b, c0, c1);                           \
        pair_##S disc = tsub_##S(bb.a, bb.b, fac.a, fac.b);                    \
        pair_##S d = tsqrt_##S(disc.a, disc.b);                                \
        T nb0 = -b0, nb1 = -b1;                                                \
        pair_##S ta = tmul_##S((T)2, (T)0, a0, a1);                            \
        pair_##S s0 = tsub_##S(nb0, nb1, d.a, d.b);                            \
        pair_##S x0 = tdiv_##S(s0.a, s0.b, ta.a, ta.b);                        \
        pair_##S s1 = tadd_##S(nb0, nb1, d.a, d.b);                            \
        pair_##S x1 = tdiv_##S(s1.a, s1.b, ta.a, ta.b);                        \
        out[0][i] = d.a; out[1][i] = d.b; out[2][i] = x0.a; out[3][i] = x0.b;  \
        out[4][i] = x1.a; out[5][i] = x1.b;                                    \
      }                                                                        \
      return 0;                                                                \
    }                                                                          \
    if (fop == 3) { /* demos.py:175-192 */                                     \
      _Pragma("omp parallel for schedule(static) num_threads(nt)")            \
      for (int64_t s = 0; s < n; s++) {                                        \
        pair_##S a[3][3], f[3], x[3];                                          \
        for (int r = 0; r < 3; r++) {                                          \
          for (int c = 0; c < 3; c++)                                          \
            a[r][c] = mk_##S(in[0][(3 * r + c) * n + s], in[1][(3 * r + c) * n + s]); \
          f[r] = mk_##S(in[2][r * n + s], in[3][r * n + s]);                   \
        }                                                                      \
        for (int k = 0; k < 3; k++)                                            \
          for (int i = k + 1; i < 3; i++) {                                    \
            pair_##S m = tdiv_##S(a[i][k].a, a[i][k].b, a[k][k].a, a[k][k].b); \
            for (int j = k; j < 3; j++) {                                      \
              pair_##S t = tmul_##S(m.a, m.b, a[k][j].a, a[k][j].b);           \
              a[i][j] = tsub_##S(a[i][j].a, a[i][j].b, t.a, t.b);              \
            }                                                                  \
            pair_##S t = tmul_##S(m.a, m.b, f[k].a, f[k].b);                   \
            f[i] = tsub_##S(f[i].a, f[i].b, t.a, t.b);                         \
          }                                                                    \
        for (int i = 2; i >= 0; i--) {                                         \
          pair_##S acc = f[i];                                                 \
          for (int j = i + 1; j < 3; j++) {                                    \
            pair_##S t = tmul_##S(a[i][j].a, a[i][j].b, x[j].a, x[j].b);       \
            acc = tsub_##S(acc.a, acc.b, t.a, t.b);                            \
          }                                                                    \
          x[i] = tdiv_##S(acc.a, acc.b, a[i][i].a, a[i][i].b);                 \
        }                                                                      \
        for (int r = 0; r < 3; r++) { out[0][r * n + s] = x[r].a; out[1][r * n + s] = x[r].b; } \
      }                                                                        \
      return 0;                                                                \
    }                                                                          \
    return -1;                                                                 \
  }
DEFINE_FUSED(d, double)
DEFINE_FUSED(f, float)

int tfo_fused(int fop, int dtype, int64_t n, const void* const* in, void* const* out,
              int nthreads) {
  if (n < 0) return -1;
  int nt = clamp_threads(nthreads);
  if (dtype == TF_F64) return fused_d(fop, n, (const double* const*)in, (double* const*)out, nt);
  if (dtype == TF_F32) return fused_f(fop, n, (const float* const*)in, (float* const*)out, nt);
  return -1;
}

/* ------------------------------------------------------------------------ */
/* twofold Horner: r = (c_d, +0); r = _tadd1(_tmul1(r, x), c_k), k = d-1..0     */

int tfo_horner(int dtype, int64_t n, const void* x_, const double* c, int degree,
               void* o0_, void* o1_, int nthreads) {
  if (n < 0 || degree < 0) return -1;
  int nt = clamp_threads(nthreads);
  /* Points are independent: blocks of HB points run the same per-point chain
     side by side (lane loop innermost, so it vectorises); every point still
     sees exactly the scalar sequence of operations, hence the same bits. */
#define HB 16
#define HORNER(S, T)                                                           \
  { const T* x = x_; T *o0 = o0_, *o1 = o1_;                                   \
    const int64_t nb = n / HB;                                                 \
    _Pragma("omp parallel for schedule(static) num_threads(nt)")              \
    for (int64_t blk = 0; blk < nb; blk++) {                                   \
      const int64_t i0 = blk * HB;                                             \
      T a[HB], b[HB];                                                          \
      for (int j = 0; j < HB; j++) { a[j] = (T)c[degree]; b[j] = (T)0; }       \
      for (int k = degree - 1; k >= 0; k--) {                                  \
        const T ck = (T)c[k];                                                  \
        for (int j = 0; j < HB; j++) {                                         \
          pair_##S r = tmul1_##S(a[j], b[j], x[i0 + j]);                       \
          r = tadd1_##S(r.a, r.b, ck);                                         \
          a[j] = r.a; b[j] = r.b;                                              \
        }                                                                      \
      }                                                                        \
      for (int j = 0; j < HB; j++) { o0[i0 + j] = a[j]; o1[i0 + j] = b[j]; }   \
    }                                                                          \
    for (int64_t i = nb * HB; i < n; i++) {                                    \
      pair_##S r = mk_##S((T)c[degree], (T)0);                                 \
      for (int k = degree - 1; k >= 0; k--) {                                  \
        r = tmul1_##S(r.a, r.b, x[i]);                                         \
        r = tadd1_##S(r.a, r.b, (T)c[k]);                                      \
      }                                                                        \
      o0[i] = r.a; o1[i] = r.b;                                                \
    }                                                                          \
    return 0; }
  if (dtype == TF_F64) HORNER(d, double)
  if (dtype == TF_F32) HORNER(f, float)
#undef HORNER
#undef HB
  return -1;
}

/* ------------------------------------------------------------------------ */
/* exact accumulator: Σ of integer*2^e terms in 32-bit limbs (int64 storage).
   limb j weighs 2^(32*j + EXACT_BASE).  Covers every f64 product exactly.     */

#define EXACT_BASE (-2240)
#define EXACT_LIMBS 144

typedef struct { int64_t l[EXACT_LIMBS]; int64_t adds; int nonfinite; } exact_acc;

static void exact_norm(exact_acc* A) {
  /* carry-propagate so limbs 0..N-2 are in [0, 2^32); top limb keeps the sign */
  for (int j = 0; j < EXACT_LIMBS - 1; j++) {
    int64_t c = A->l[j] >> 32; /* arithmetic shift: floor division */
    A->l[j] -= c * ((int64_t)1 << 32);
    A->l[j + 1] += c;
  }
  A->adds = 0;
}

/* add sign * M * 2^E, M < 2^120 */
static void exact_add_int(exact_acc* A, int neg, unsigned __int128 M, int E) {
  if (M == 0) return;
  int p = E - EXACT_BASE; /* >= 0 by construction */
  int j = p >> 5, s = p & 31;
  /* M << s may need 152 bits: split M into low 64 / high 64 */
  uint64_t lo = (uint64_t)M, hi = (uint64_t)(M >> 64);
  uint32_t chunk[6] = {0};
  /* build 192-bit (lo,hi) << s as 32-bit chunks */
  unsigned __int128 a = ((unsigned __int128)lo) << s;       /* up to 96 bits */
  unsigned __int128 b = ((unsigned __int128)hi) << s;       /* weight 2^64 */
  chunk[0] = (uint32_t)a; chunk[1] = (uint32_t)(a >> 32); chunk[2] = (uint32_t)(a >> 64);
  unsigned __int128 c2 = (unsigned __int128)chunk[2] + (uint32_t)b;
  chunk[2] = (uint32_t)c2;
  unsigned __int128 c3 = (c2 >> 32) + (uint32_t)(b >> 32);
  chunk[3] = (uint32_t)c3;
  unsigned __int128 c4 = (c3 >> 32) + (uint32_t)(b >> 64);
  chunk[4] = (uint32_t)c4;
  chunk[5] = (uint32_t)(c4 >> 32);
  for (int q = 0; q < 6; q++) {
    if (!chunk[q]) continue;
    if (neg) A->l[j + q] -= chunk[q]; else A->l[j + q] += chunk[q];
  }
  if (++A->adds >= ((int64_t)1 << 28)) exact_norm(A);
}

static int decompose_d(double x, int* neg, uint64_t* M, int* E) {
  uint64_t u; memcpy(&u, &x, 8);
  *neg = (int)(u >> 63);
  int ex = (int)((u >> 52) & 0x7ff);
  uint64_t fr = u & ((1ull << 52) - 1);
  if (ex == 0x7ff) return -1;
  if (ex == 0) { *M = fr; *E = -1074; }
  else { *M = fr | (1ull << 52); *E = ex - 1075; }
  return 0;
}

static int decompose_f(float x, int* neg, uint64_t* M, int* E) {
  uint32_t u; memcpy(&u, &x, 4);
  *neg = (int)(u >> 31);
  int ex = (int)((u >> 23) & 0xff);
  uint32_t fr = u & ((1u << 23) - 1);
  if (ex == 0xff) return -1;
  if (ex == 0) { *M = fr; *E = -149; }
  else { *M = fr | (1u << 23); *E = ex - 150; }
  return 0;
}

static void exact_add_val(exact_acc* A, exact_acc* Aabs, int dtype, const void* p, int64_t i) {
  int neg, E; uint64_t M;
  int bad = dtype == TF_F64 ? decompose_d(((const double*)p)[i], &neg, &M, &E)
                            : decompose_f(((const float*)p)[i], &neg, &M, &E);
  if (bad) { A->nonfinite = 1; return; }
  exact_add_int(A, neg, M, E);
  if (Aabs) exact_add_int(Aabs, 0, M, E);
}

static void exact_add_prod(exact_acc* A, exact_acc* Aabs, int dtype, const void* x,
                           const void* y, int64_t i) {
  int n1, n2, e1, e2; uint64_t m1, m2;
  int bad = dtype == TF_F64
                ? (decompose_d(((const double*)x)[i], &n1, &m1, &e1) |
                   decompose_d(((const double*)y)[i], &n2, &m2, &e2))
                : (decompose_f(((const float*)x)[i], &n1, &m1, &e1) |
                   decompose_f(((const float*)y)[i], &n2, &m2, &e2));
  if (bad) { A->nonfinite = 1; return; }
  unsigned __int128 M = (unsigned __int128)m1 * m2;
  exact_add_int(A, n1 ^ n2, M, e1 + e2);
  if (Aabs) exact_add_int(Aabs, 0, M, e1 + e2);
}

static void exact_merge(exact_acc* A, const exact_acc* B) {
  for (int j = 0; j < EXACT_LIMBS; j++) A->l[j] += B->l[j];
  A->nonfinite |= B->nonfinite;
}

int tfo_exact_base(void) { return EXACT_BASE; }
int tfo_exact_limbs(void) { return EXACT_LIMBS; }

/*
 * Exact Σ terms and Σ|terms| for rop RSUM (terms x_i), RSUM2 (terms x0_i and
 * x1_i), RDOT (terms x_i*y_i, exact 106-bit products).  Normalized limbs are
 * written to sum_limbs / abs_limbs (EXACT_LIMBS int64 each); returns 1 if a
 * non-finite input was seen, 0 otherwise.
 */
int tfo_exact(int rop, int dtype, int64_t n, const void* a, const void* b,
              int64_t* sum_limbs, int64_t* abs_limbs, int nthreads) {
  int nt = clamp_threads(nthreads);
  exact_acc tot, tabs;
  memset(&tot, 0, sizeof tot); memset(&tabs, 0, sizeof tabs);
#pragma omp parallel num_threads(nt)
  {
    exact_acc* A = calloc(1, sizeof(exact_acc));
    exact_acc* B = calloc(1, sizeof(exact_acc));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; i++) {
      if (rop == TF_RDOT) exact_add_prod(A, B, dtype, a, b, i);
      else {
        exact_add_val(A, B, dtype, a, i);
        if (rop == TF_RSUM2) exact_add_val(A, B, dtype, b, i);
      }
    }
    exact_norm(A); exact_norm(B);
#pragma omp critical
    { exact_merge(&tot, A); exact_merge(&tabs, B); }
    free(A); free(B);
  }
  exact_norm(&tot); exact_norm(&tabs);
  memcpy(sum_limbs, tot.l, sizeof tot.l);
  memcpy(abs_limbs, tabs.l, sizeof tabs.l);
  return tot.nonfinite;
}

int tfo_has_hw_fma(void) {
#ifdef HW_FMA
  return 1;
#else
  return 0;
#endif
}
