/*
 * mpsylv_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker (or the timed CPU baseline), never as the product
 * path.  The product is the sm_100a CUDA library in paper_2503_03456_b200/.
 *
 * What it restates (reference = /root/reference, read-only, Python+numpy):
 *   gemm                    pkg/src/mpsylv/linalg.py:125-154
 *   _vec_norm2_ctx, _dot    pkg/src/mpsylv/linalg.py:198-222
 *   mgs_qr (+fix diag/rank) pkg/src/mpsylv/linalg.py:228-273
 *   _make_reflector, _apply_reflector_left/right  linalg.py:276-312
 *   lu, lu_solve            pkg/src/mpsylv/linalg.py:349-440
 *   _hessenberg             pkg/src/mpsylv/linalg.py:446-464
 *   _givens, _rot_rows, _rot_cols, _wilkinson_shift, schur  linalg.py:467-577
 *   solve_sylv_tri          pkg/src/mpsylv/sylvester.py:111-157
 *   residual                pkg/src/mpsylv/sylvester.py:199-209
 *   solve_pert_sylv_tri_stat pkg/src/mpsylv/refinement.py:95-141
 *   mp_orth / mp_inv        pkg/src/mpsylv/refinement.py:185-297
 * Scalar arithmetic follows pkg/src/mpsylv/precision.py: simulated binary32
 * (correctly rounded +,-,*,/,sqrt on float-representable operands, complex
 * multiply = 4 rounded products + 2 rounded sums, Smith division) is exactly
 * IEEE binary32 arithmetic without FMA (precision.py:322-520, checked against
 * native float32 in pkg/tests/test_precision.py:208-220), so the binary32
 * paths are computed with C `float` operations under -ffp-contract=off and
 * reproduce the reference bit for bit.  binary64 paths use `double`; the
 * reference there calls numpy/OpenBLAS (vdot, norm, SIMD complex multiply)
 * whose summation order is not reproducible, so binary64 results agree to a
 * few ulps, not bitwise.
 *
 * Storage mirrors the reference: every matrix is complex128, row major
 * (numpy C order), and in binary32 mode every stored value is exactly
 * representable in binary32.
 *
 * Parity pinning: tests/test_oracle_golden.py compares every function above
 * with fixtures produced by running the reference itself
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <complex.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double re, im; } zc;

enum {
  OR_OK = 0,
  OR_SINGULAR_EQUATION = 1,
  OR_NUMERIC_BREAKDOWN = 2,
  OR_ITERATION_LIMIT = 3,
  OR_RANK_DEFICIENT = 4,
  OR_SINGULAR_MATRIX = 5,
  OR_FORMAT_OVERFLOW = 6,
  OR_DIMENSION = 7,
};

/* error side channel (row/col of a singular pair) */
static __thread int g_err_row = -1, g_err_col = -1;

/* ---------------------------------------------------------------------- */
/* scalar arithmetic, precision.py:322-520                                 */

typedef struct { int f32; } fmt_t;

static inline double r_add(fmt_t f, double a, double b) { return f.f32 ? (double)((float)a + (float)b) : a + b; }
static inline double r_sub(fmt_t f, double a, double b) { return f.f32 ? (double)((float)a - (float)b) : a - b; }
static inline double r_mul(fmt_t f, double a, double b) { return f.f32 ? (double)((float)a * (float)b) : a * b; }
static inline double r_div(fmt_t f, double a, double b) { return f.f32 ? (double)((float)a / (float)b) : a / b; }
static inline double r_sqrt(fmt_t f, double a) { return f.f32 ? (double)sqrtf((float)a) : sqrt(a); }

static inline zc Z(double re, double im) { zc z = {re, im}; return z; }
static inline zc conjz(zc a) { return Z(a.re, -a.im); }
static inline int zero(zc a) { return a.re == 0.0 && a.im == 0.0; }
static inline int zfinite(zc a) { return isfinite(a.re) && isfinite(a.im); }

static inline zc c_add(fmt_t f, zc a, zc b) { return Z(r_add(f, a.re, b.re), r_add(f, a.im, b.im)); }
static inline zc c_sub(fmt_t f, zc a, zc b) { return Z(r_sub(f, a.re, b.re), r_sub(f, a.im, b.im)); }
/* fl_mul / _smul: rr, ii, ri, ir rounded, then re = rr - ii, im = ri + ir */
static inline zc c_mul(fmt_t f, zc a, zc b) {
  double rr = r_mul(f, a.re, b.re), ii = r_mul(f, a.im, b.im);
  double ri = r_mul(f, a.re, b.im), ir = r_mul(f, a.im, b.re);
  return Z(r_sub(f, rr, ii), r_add(f, ri, ir));
}
/* fl_div / _sdiv: Smith's algorithm with every step rounded (precision.py:462-479) */
static zc c_div(fmt_t f, zc a, zc b) {
  double ar = a.re, ai = a.im, br = b.re, bi = b.im;
  if (br == 0.0 && bi == 0.0) {
    double complex q = (ar + I * ai) / (br + I * bi);
    return Z(creal(q), cimag(q));
  }
  if (fabs(br) >= fabs(bi)) {
    double t = r_div(f, bi, br);
    double d = r_add(f, br, r_mul(f, bi, t));
    return Z(r_div(f, r_add(f, ar, r_mul(f, ai, t)), d),
             r_div(f, r_sub(f, ai, r_mul(f, ar, t)), d));
  }
  double t = r_div(f, br, bi);
  double d = r_add(f, bi, r_mul(f, br, t));
  return Z(r_div(f, r_add(f, ai, r_mul(f, ar, t)), d),
           -r_div(f, r_sub(f, ar, r_mul(f, ai, t)), d));
}
/* _sabs: |z| from rounded square, add, sqrt (binary64: abs() = hypot) */
static inline double c_abs_s(fmt_t f, zc z) {
  if (!f.f32) return hypot(z.re, z.im);
  float s = (float)z.re * (float)z.re + (float)z.im * (float)z.im;
  if (!isfinite(s)) return INFINITY;
  return (double)sqrtf(s);
}
/* _csqrt: principal square root from rounded real steps */
static zc c_sqrt_s(fmt_t f, zc z) {
  if (!f.f32) {
    double complex c = csqrt(z.re + I * z.im);
    return Z(creal(c), cimag(c));
  }
  if (zero(z)) return Z(0.0, 0.0);
  double a = z.re, b = z.im;
  double mag = c_abs_s(f, z);
  if (a >= 0.0) {
    double u = r_sqrt(f, r_div(f, r_add(f, mag, a), 2.0));
    if (u == 0.0) return Z(0.0, b);
    double v = r_div(f, b, r_mul(f, 2.0, u));
    return Z(u, v);
  }
  double v = r_sqrt(f, r_div(f, r_sub(f, mag, a), 2.0));
  v = copysign(v, b != 0.0 ? b : 1.0);
  if (v == 0.0) return Z(0.0, 0.0);
  double u = r_div(f, b, r_mul(f, 2.0, v));
  return Z(u, v);
}

/* _round_real_scalar(x, fmt, err) for binary32: nearest-even with a 2Sum
 * residual breaking exact midpoints (precision.py:242-261). */
static double round32_err(double x, double err) {
  if (x == 0.0 || !isfinite(x)) return x;
  int e;
  frexp(x, &e);
  if (e - 1 > 127 + 1) return copysign(INFINITY, x);
  int q = e - 1 > -126 ? e - 1 : -126;
  int shift = q - 23;
  double scaled = ldexp(x, -shift);
  double r = nearbyint(scaled);
  if (err != 0.0 && isfinite(err)) {
    double lo = floor(scaled);
    if (scaled - lo == 0.5) r = lo + (err > 0.0 ? 1.0 : 0.0);
  }
  double y = ldexp(r, shift);
  if (fabs(y) > 3.4028234663852886e38) return copysign(INFINITY, x);
  if (y == 0.0) return copysign(0.0, x);
  return y;
}
/* _ssub(a, b) for a float-representable a and an arbitrary double b */
static zc c_sub_exact(fmt_t f, zc a, zc b) {
  if (!f.f32) return Z(a.re - b.re, a.im - b.im);
  double out[2];
  double av[2] = {a.re, a.im}, bv[2] = {-b.re, -b.im};
  for (int k = 0; k < 2; k++) {
    double s = av[k] + bv[k];
    double e = 0.0;
    if (isfinite(s)) { double bb = s - av[k]; e = (av[k] - (s - bb)) + (bv[k] - bb); }
    out[k] = round32_err(s, e);
  }
  return Z(out[0], out[1]);
}

static inline double round_in(fmt_t f, double x) { return f.f32 ? (double)(float)x : x; }

/* ---------------------------------------------------------------------- */
/* matrices (row-major complex128)                                         */

#define AT(M, ld, i, j) (M)[(size_t)(i) * (ld) + (j)]

static zc* zalloc(size_t n) { return (zc*)calloc(n ? n : 1, sizeof(zc)); }

/* _enter: round into the format; finite -> non-finite is FormatOverflowError */
static int enter(fmt_t f, const zc* A, zc* out, size_t n) {
  for (size_t i = 0; i < n; i++) {
    out[i] = Z(round_in(f, A[i].re), round_in(f, A[i].im));
    if (!zfinite(out[i]) && zfinite(A[i])) return OR_FORMAT_OVERFLOW;
  }
  return OR_OK;
}

static double fro(const zc* M, size_t n) {
  /* binary64 Frobenius norm (numpy norm); summation order differs from BLAS */
  double s = 0.0;
  for (size_t i = 0; i < n; i++) s += M[i].re * M[i].re + M[i].im * M[i].im;
  return sqrt(s);
}

/* gemm: fl(alpha*A@B + beta*C), ascending-k rank-1 accumulation (linalg.py:125-154).
 * A (m x k, lda), B (k x n, ldb), C (m x n, ldc) or NULL when beta == 0.
 * opA/opB: 'N' or 'C' (conjugate transpose of the stored matrix). */
static void gemm_core(fmt_t f, zc alpha, char opA, const zc* A, int lda, char opB,
                      const zc* B, int ldb, zc beta, const zc* C, int ldc,
                      zc* out, int ldo, int m, int n, int k) {
  /* Parallel restatement: every output element accumulates its k products in
   * ascending order starting from 0, exactly as the reference's rank-1 loop;
   * only the order in which DIFFERENT elements are visited changes (row/column
   * blocks per thread), so the result is bit-identical.  Operands are first
   * copied into row-major op(A) (m x k) and op(B) (k x n); conjugation is exact. */
  zc* Ao = zalloc((size_t)m * k);
  zc* Bo = zalloc((size_t)k * n);
#pragma omp parallel for schedule(static) if ((size_t)m * k > 4096)
  for (int i = 0; i < m; i++)
    for (int p = 0; p < k; p++) Ao[(size_t)i * k + p] = opA == 'N' ? AT(A, lda, i, p) : conjz(AT(A, lda, p, i));
#pragma omp parallel for schedule(static) if ((size_t)n * k > 4096)
  for (int p = 0; p < k; p++)
    for (int j = 0; j < n; j++) Bo[(size_t)p * n + j] = opB == 'N' ? AT(B, ldb, p, j) : conjz(AT(B, ldb, j, p));
  int a1 = alpha.re == 1.0 && alpha.im == 0.0;
  int b0 = beta.re == 0.0 && beta.im == 0.0;
  int b1 = beta.re == 1.0 && beta.im == 0.0;
  enum { IB = 16, JB = 128 };
  int nib = (m + IB - 1) / IB, njb = (n + JB - 1) / JB;
#pragma omp parallel for collapse(2) schedule(dynamic) if ((double)m * n * k > 1e6)
  for (int ib = 0; ib < nib; ib++)
    for (int jb = 0; jb < njb; jb++) {
      zc acc[IB][JB];
      int i0 = ib * IB, i1 = i0 + IB < m ? i0 + IB : m;
      int j0 = jb * JB, j1 = j0 + JB < n ? j0 + JB : n;
      for (int i = i0; i < i1; i++)
        for (int j = j0; j < j1; j++) acc[i - i0][j - j0] = Z(0.0, 0.0);
      for (int p = 0; p < k; p++) {
        const zc* brow = Bo + (size_t)p * n;
        for (int i = i0; i < i1; i++) {
          zc a = Ao[(size_t)i * k + p];
          zc* ar = acc[i - i0];
          for (int j = j0; j < j1; j++) ar[j - j0] = c_add(f, ar[j - j0], c_mul(f, a, brow[j]));
        }
      }
      for (int i = i0; i < i1; i++)
        for (int j = j0; j < j1; j++) {
          zc v = acc[i - i0][j - j0];
          if (!a1) v = c_mul(f, alpha, v);
          if (!b0) v = c_add(f, v, b1 ? AT(C, ldc, i, j) : c_mul(f, beta, AT(C, ldc, i, j)));
          AT(out, ldo, i, j) = v;
        }
    }
  free(Ao); free(Bo);
}

int oracle_gemm(int f32, double ar, double ai, const zc* A, const zc* B, double br,
                double bi, const zc* C, zc* out, int m, int n, int k) {
  fmt_t f = {f32};
  gemm_core(f, Z(ar, ai), 'N', A, k, 'N', B, n, Z(br, bi), C, n, out, n, m, n, k);
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* vector helpers (linalg.py:198-222)                                      */

static double vec_norm2(fmt_t f, const zc* x, int n, int stride) {
  if (!f.f32) {
    double s = 0.0;
    for (int i = 0; i < n; i++) { zc v = x[(size_t)i * stride]; s += v.re * v.re + v.im * v.im; }
    return sqrt(s);
  }
  /* acc = round(acc + |x_i|^2) with |x_i| rounded and its square exact: fmaf */
  float acc = 0.0f;
  for (int i = 0; i < n; i++) {
    float a = (float)c_abs_s(f, x[(size_t)i * stride]);
    acc = fmaf(a, a, acc);
  }
  return (double)sqrtf(acc);
}

/* ---------------------------------------------------------------------- */
/* Householder helpers (linalg.py:276-312)                                 */

/* returns 0 when x == 0 (no reflector); w overwrites x-copy in wout */
static int make_reflector(fmt_t f, const zc* x, int n, int stride, zc* w, double* beta, zc* head) {
  double nx = vec_norm2(f, x, n, stride);
  if (nx == 0.0) return 0;
  zc x0 = x[0];
  double a0 = c_abs_s(f, x0);
  zc phase = a0 != 0.0 ? c_div(f, x0, Z(a0, 0.0)) : Z(1.0, 0.0);
  for (int i = 0; i < n; i++) w[i] = x[(size_t)i * stride];
  w[0] = c_add(f, x0, c_mul(f, phase, Z(nx, 0.0)));
  double ww = c_mul(f, Z(2.0, 0.0), c_mul(f, Z(nx, 0.0), c_add(f, Z(nx, 0.0), Z(a0, 0.0)))).re;
  *beta = c_div(f, Z(2.0, 0.0), Z(ww, 0.0)).re;
  *head = c_mul(f, Z(-1.0, 0.0), c_mul(f, phase, Z(nx, 0.0)));
  return 1;
}

/* M[r0:r0+len, c0:c1] <- (I - beta w w*) M  (rows matching w).
 * Parallel over columns: each t[j] accumulates over i ascending, each M entry
 * gets its single update -- the reference's per-element order. */
static void refl_left(fmt_t f, zc* M, int ld, int r0, int c0, int c1, const zc* w, int len, double beta, zc* t) {
  zc* bw = zalloc(len);
  for (int i = 0; i < len; i++) bw[i] = c_mul(f, Z(beta, 0.0), w[i]);
  enum { CB = 32 };
  int nb = (c1 - c0 + CB - 1) / CB;
#pragma omp parallel for schedule(static) if ((size_t)len * (c1 - c0) > 32768)
  for (int b = 0; b < nb; b++) {
    int j0 = c0 + b * CB, j1 = j0 + CB < c1 ? j0 + CB : c1;
    for (int j = j0; j < j1; j++) t[j - c0] = Z(0.0, 0.0);
    for (int i = 0; i < len; i++) {
      zc wc = conjz(w[i]);
      const zc* row = &AT(M, ld, r0 + i, 0);
      for (int j = j0; j < j1; j++) t[j - c0] = c_add(f, t[j - c0], c_mul(f, wc, row[j]));
    }
    for (int i = 0; i < len; i++) {
      zc* row = &AT(M, ld, r0 + i, 0);
      for (int j = j0; j < j1; j++) row[j] = c_sub(f, row[j], c_mul(f, bw[i], t[j - c0]));
    }
  }
  free(bw);
}

/* M[r0:r1, c0:c0+len] <- M (I - beta w w*)  (columns matching w); parallel over rows */
static void refl_right(fmt_t f, zc* M, int ld, int r0, int r1, int c0, const zc* w, int len, double beta, zc* t) {
  zc* bw = zalloc(len);
  for (int i = 0; i < len; i++) bw[i] = c_mul(f, Z(beta, 0.0), conjz(w[i]));
#pragma omp parallel for schedule(static) if ((size_t)len * (r1 - r0) > 32768)
  for (int r = r0; r < r1; r++) {
    zc* row = &AT(M, ld, r, c0);
    zc s = Z(0.0, 0.0);
    for (int i = 0; i < len; i++) s = c_add(f, s, c_mul(f, row[i], w[i]));
    t[r - r0] = s;
    for (int i = 0; i < len; i++) row[i] = c_sub(f, row[i], c_mul(f, s, bw[i]));
  }
  free(bw);
}

/* ---------------------------------------------------------------------- */
/* Hessenberg + Schur (linalg.py:446-577)                                  */

static void hessenberg(fmt_t f, zc* H, zc* U, int m) {
  zc* w = zalloc(m);
  zc* t = zalloc(m);
  for (int i = 0; i < m; i++)
    for (int j = 0; j < m; j++) AT(U, m, i, j) = Z(i == j ? 1.0 : 0.0, 0.0);
  for (int k = 0; k < m - 2; k++) {
    int any = 0;
    for (int i = k + 2; i < m; i++) if (!zero(AT(H, m, i, k))) { any = 1; break; }
    if (!any) continue;
    double beta; zc head;
    int len = m - k - 1;
    if (!make_reflector(f, &AT(H, m, k + 1, k), len, m, w, &beta, &head)) continue;
    /* left: rows k+1.., columns k.. (column k is overwritten right after) */
    refl_left(f, H, m, k + 1, k + 1, m, w, len, beta, t);
    for (int i = k + 1; i < m; i++) AT(H, m, i, k) = Z(0.0, 0.0);
    AT(H, m, k + 1, k) = head;
    refl_right(f, H, m, 0, m, k + 1, w, len, beta, t);
    refl_right(f, U, m, 0, m, k + 1, w, len, beta, t);
  }
  if (m > 2)
    for (int i = 0; i < m; i++)
      for (int j = 0; j < i - 1; j++) AT(H, m, i, j) = Z(0.0, 0.0);
  free(w); free(t);
}

int oracle_hessenberg(int f32, const zc* A, zc* H, zc* U, int m) {
  fmt_t f = {f32};
  int rc = enter(f, A, H, (size_t)m * m);
  if (rc) return rc;
  hessenberg(f, H, U, m);
  return OR_OK;
}

static void givens(fmt_t f, zc fv, zc g, double* c, zc* s) {
  if (zero(g)) { *c = 1.0; *s = Z(0.0, 0.0); return; }
  if (zero(fv)) {
    double ag = c_abs_s(f, g);
    *c = 0.0; *s = c_div(f, conjz(g), Z(ag, 0.0)); return;
  }
  double af = c_abs_s(f, fv);
  double ag = c_abs_s(f, g);
  double d2 = c_add(f, c_mul(f, Z(af, 0.0), Z(af, 0.0)), c_mul(f, Z(ag, 0.0), Z(ag, 0.0))).re;
  double d = r_sqrt(f, d2);
  *c = c_div(f, Z(af, 0.0), Z(d, 0.0)).re;
  *s = c_div(f, c_mul(f, c_div(f, fv, Z(af, 0.0)), conjz(g)), Z(d, 0.0));
}

static zc wilkinson_shift(fmt_t f, const zc* H, int m, int hi) {
  zc a = AT(H, m, hi - 1, hi - 1), b = AT(H, m, hi - 1, hi);
  zc c = AT(H, m, hi, hi - 1), d = AT(H, m, hi, hi);
  zc delta = c_mul(f, Z(0.5, 0.0), c_sub(f, a, d));
  zc disc = c_sqrt_s(f, c_add(f, c_mul(f, delta, delta), c_mul(f, b, c)));
  if (delta.re * disc.re + delta.im * disc.im < 0) disc = Z(-disc.re, -disc.im);
  zc denom = c_add(f, delta, disc);
  if (zero(denom)) return d;
  return c_sub(f, d, c_div(f, c_mul(f, b, c), denom));
}

/* One QR sweep's rotations, applied in batches of SWEEP_BATCH chase steps.
 *
 * The reference (linalg.py:518-577) applies, at each step k of a sweep, the
 * Givens rotation G_k to rows k, k+1 (columns max(lo,k-1)..m-1), then to
 * columns k, k+1 of H (rows 0..min(k+3,hi+1)-1) and of U (all rows).  Each
 * matrix entry therefore sees a fixed sequence of updates.  This restatement
 * keeps that per-entry sequence exactly (so the result is bit-identical) but
 * lets independent entries be updated by different threads:
 *   phase A (sequential, the chase): steps K..K+S-1 on the columns < K+S+3
 *     and the rows >= K-2 -- everything the next Givens rotations read;
 *   phase B (parallel over columns >= K+S+3): the batch's row rotations, in
 *     ascending k (those columns receive no column rotation in the batch);
 *   phase C (parallel over rows, at the end of the sweep): the column
 *     rotations deferred from rows < K-2 (which no later step reads) and all
 *     rotations of U, each row in ascending k. */
enum { SWEEP_BATCH = 32 };

/* rows != 0: the rot_rows pair update; rows == 0: the rot_cols pair update */
static inline void rot_pair(fmt_t f, zc* a, zc* b, double c, zc s, int rows) {
  zc cc = Z(c, 0.0), sc = conjz(s);
  zc v1 = *a, v2 = *b;
  if (rows) {
    *a = c_add(f, c_mul(f, cc, v1), c_mul(f, s, v2));
    *b = c_sub(f, c_mul(f, cc, v2), c_mul(f, sc, v1));
  } else {
    *a = c_add(f, c_mul(f, cc, v1), c_mul(f, sc, v2));
    *b = c_sub(f, c_mul(f, cc, v2), c_mul(f, s, v1));
  }
}

/* schur: returns OR_ITERATION_LIMIT after 30*m sweeps; *sweeps_out optional */
static int schur_core(fmt_t f, zc* H, zc* U, int m, int* sweeps_out) {
  if (m == 1) { U[0] = Z(1.0, 0.0); return OR_OK; }
  hessenberg(f, H, U, m);
  double u = f.f32 ? ldexp(1.0, -24) : ldexp(1.0, -53);
  int limit = 30 * m, sweeps = 0, stuck = 0, hi = m - 1;
  double* cs = (double*)malloc(sizeof(double) * m);
  zc* ss = zalloc(m);
  int rc = OR_OK;
  while (hi > 0) {
    for (int k = 1; k <= hi; k++) {
      zc h = AT(H, m, k, k - 1);
      if (!zero(h) && hypot(h.re, h.im) <= u * (hypot(AT(H, m, k - 1, k - 1).re, AT(H, m, k - 1, k - 1).im) +
                                                 hypot(AT(H, m, k, k).re, AT(H, m, k, k).im)))
        AT(H, m, k, k - 1) = Z(0.0, 0.0);
    }
    if (zero(AT(H, m, hi, hi - 1))) { hi--; stuck = 0; continue; }
    int lo = hi;
    while (lo > 0 && !zero(AT(H, m, lo, lo - 1))) lo--;
    if (sweeps >= limit) { rc = OR_ITERATION_LIMIT; break; }
    zc shift;
    if (stuck > 0 && stuck % 10 == 0) {
      zc h1 = AT(H, m, hi, hi - 1), h2 = AT(H, m, hi, hi);
      shift = Z(hypot(h1.re, h1.im) + 0.75 * hypot(h2.re, h2.im), 0.0);
    } else {
      shift = wilkinson_shift(f, H, m, hi);
    }
    zc x = c_sub_exact(f, AT(H, m, lo, lo), shift);
    zc y = AT(H, m, lo + 1, lo);
    for (int K = lo; K < hi; K += SWEEP_BATCH) {
      int Ke = K + SWEEP_BATCH < hi ? K + SWEEP_BATCH : hi;
      int cnear = Ke + 3 < m ? Ke + 3 : m;
      int rfar = K - 2 > 0 ? K - 2 : 0;
      /* phase A */
      for (int k = K; k < Ke; k++) {
        double c; zc s;
        givens(f, x, y, &c, &s);
        cs[k] = c; ss[k] = s;
        int j0 = lo > k - 1 ? lo : k - 1;
        for (int j = j0; j < cnear; j++) rot_pair(f, &AT(H, m, k, j), &AT(H, m, k + 1, j), c, s, 1);
        int i1 = (k + 3 < hi + 1) ? k + 3 : hi + 1;
        for (int i = rfar; i < i1; i++) rot_pair(f, &AT(H, m, i, k), &AT(H, m, i, k + 1), c, s, 0);
        if (k > lo) AT(H, m, k + 1, k - 1) = Z(0.0, 0.0);
        if (k < hi - 1) { x = AT(H, m, k + 1, k); y = AT(H, m, k + 2, k); }
      }
      /* phase B */
      enum { CB = 8 };
      int nb = (m - cnear + CB - 1) / CB;
#pragma omp parallel for schedule(static) if (nb * (Ke - K) > 512)
      for (int b = 0; b < nb; b++) {
        int c0 = cnear + b * CB, c1 = c0 + CB < m ? c0 + CB : m;
        for (int k = K; k < Ke; k++) {
          zc* r0 = &AT(H, m, k, 0);
          zc* r1 = &AT(H, m, k + 1, 0);
          for (int j = c0; j < c1; j++) rot_pair(f, r0 + j, r1 + j, cs[k], ss[k], 1);
        }
      }
    }
    /* phase C: deferred column rotations of H (rows < K-2 of each batch) and all of U */
#pragma omp parallel for schedule(static) if ((size_t)m * (hi - lo) > 16384)
    for (int r = 0; r < 2 * m; r++) {
      if (r < m) {
        zc* row = &AT(H, m, r, 0);
        for (int K = lo; K < hi; K += SWEEP_BATCH) {
          if (!(r < K - 2)) continue;
          int Ke = K + SWEEP_BATCH < hi ? K + SWEEP_BATCH : hi;
          for (int k = K; k < Ke; k++) rot_pair(f, row + k, row + k + 1, cs[k], ss[k], 0);
        }
      } else {
        zc* row = &AT(U, m, r - m, 0);
        for (int k = lo; k < hi; k++) rot_pair(f, row + k, row + k + 1, cs[k], ss[k], 0);
      }
    }
    sweeps++; stuck++;
  }
  free(cs); free(ss);
  if (sweeps_out) *sweeps_out = sweeps;
  if (rc) return rc;
  for (int i = 0; i < m; i++)
    for (int j = 0; j < i; j++) AT(H, m, i, j) = Z(0.0, 0.0);
  return OR_OK;
}

int oracle_schur(int f32, const zc* A, zc* T, zc* U, int m, int* sweeps) {
  fmt_t f = {f32};
  int rc = enter(f, A, T, (size_t)m * m);
  if (rc) return rc;
  return schur_core(f, T, U, m, sweeps);
}

/* ---------------------------------------------------------------------- */
/* MGS QR with positive diagonal (linalg.py:228-273), binary64 or binary32  */

static int mgs_qr_core(fmt_t f, const zc* A_in, zc* Q, zc* R, int m, int n) {
  /* Right-looking restatement: once q_i is final, every later column j
   * projects against it (in parallel over j).  Column j still sees the
   * projections i = 0, 1, ..., j-1 in that order with the reference's
   * arithmetic, so Q and R are bit-identical to the column-by-column loop. */
  int rc = enter(f, A_in, Q, (size_t)m * n);
  if (rc) return rc;
  double nrmA = fro(Q, (size_t)m * n);
  memset(R, 0, sizeof(zc) * (size_t)n * n);
  zc* V = zalloc((size_t)n * m); /* row j = column j */
  for (int i = 0; i < m; i++)
    for (int j = 0; j < n; j++) V[(size_t)j * m + i] = AT(Q, n, i, j);
  for (int i = 0; i < n; i++) {
    zc* q = V + (size_t)i * m;
    double nv = vec_norm2(f, q, m, 1);
    AT(R, n, i, i) = Z(nv, 0.0);
    if (nv == 0.0) { free(V); return OR_RANK_DEFICIENT; }
    for (int p = 0; p < m; p++) q[p] = c_div(f, q[p], Z(nv, 0.0));
#pragma omp parallel for schedule(static) if ((size_t)(n - i - 1) * m > 16384)
    for (int j = i + 1; j < n; j++) {
      zc* v = V + (size_t)j * m;
      zc r = Z(0.0, 0.0);
      if (!f.f32) {
        for (int p = 0; p < m; p++) {
          zc qq = q[p];
          r.re += qq.re * v[p].re + qq.im * v[p].im;
          r.im += qq.re * v[p].im - qq.im * v[p].re;
        }
      } else {
        for (int p = 0; p < m; p++) r = c_add(f, r, c_mul(f, conjz(q[p]), v[p]));
      }
      AT(R, n, i, j) = r;
      for (int p = 0; p < m; p++) v[p] = c_sub(f, v[p], c_mul(f, r, q[p]));
    }
  }
  for (int i = 0; i < m; i++)
    for (int j = 0; j < n; j++) AT(Q, n, i, j) = V[(size_t)j * m + i];
  free(V);
  /* _fix_r_diagonal: R[j,j] = nv is real positive already (phase == 1) */
  double u = f.f32 ? ldexp(1.0, -24) : ldexp(1.0, -53);
  double dmin = INFINITY;
  for (int j = 0; j < n; j++) { double a = hypot(AT(R, n, j, j).re, AT(R, n, j, j).im); if (a < dmin) dmin = a; }
  if (dmin <= n * u * nrmA) return OR_RANK_DEFICIENT;
  return OR_OK;
}

int oracle_mgs_qr(int f32, const zc* A, zc* Q, zc* R, int m, int n) {
  fmt_t f = {f32};
  return mgs_qr_core(f, A, Q, R, m, n);
}

/* ---------------------------------------------------------------------- */
/* LU with partial pivoting and solves (linalg.py:349-440)                 */

static int lu_core(fmt_t f, const zc* A_in, zc* W, long long* piv, int n) {
  int rc = enter(f, A_in, W, (size_t)n * n);
  if (rc) return rc;
  for (int k = 0; k < n; k++) {
    int p = k; double best = -1.0;
    for (int i = k; i < n; i++) {
      double a = hypot(AT(W, n, i, k).re, AT(W, n, i, k).im);
      if (a > best) { best = a; p = i; }
    }
    if (zero(AT(W, n, p, k))) return OR_SINGULAR_MATRIX;
    piv[k] = p;
    if (p != k)
      for (int j = 0; j < n; j++) { zc tmp = AT(W, n, k, j); AT(W, n, k, j) = AT(W, n, p, j); AT(W, n, p, j) = tmp; }
    for (int i = k + 1; i < n; i++) AT(W, n, i, k) = c_div(f, AT(W, n, i, k), AT(W, n, k, k));
#pragma omp parallel for schedule(static) if ((size_t)(n - k) * (n - k) > 16384)
    for (int i = k + 1; i < n; i++) {
      zc l = AT(W, n, i, k);
      for (int j = k + 1; j < n; j++) AT(W, n, i, j) = c_sub(f, AT(W, n, i, j), c_mul(f, l, AT(W, n, k, j)));
    }
  }
  return OR_OK;
}

int oracle_lu(int f32, const zc* A, zc* LU, long long* piv, int n) {
  fmt_t f = {f32};
  return lu_core(f, A, LU, piv, n);
}

static void apply_pivots(zc* B, int nrhs, const long long* piv, int n, int inverse) {
  for (int t = 0; t < n; t++) {
    int k = inverse ? n - 1 - t : t;
    int p = (int)piv[k];
    if (p != k)
      for (int j = 0; j < nrhs; j++) { zc tmp = AT(B, nrhs, k, j); AT(B, nrhs, k, j) = AT(B, nrhs, p, j); AT(B, nrhs, p, j) = tmp; }
  }
}

/* _solve_lower / _solve_upper on X (n x nrhs) in place.  Restated in row
 * (dot-product) order: row r receives the updates from rows i = 0..r-1
 * (lower) or i = n-1..r+1 (upper) in the same order as the reference's
 * column sweep, then its diagonal division -- identical per-entry arithmetic.
 * Right-hand-side columns are independent and split across threads. */
static int solve_tri(fmt_t f, const zc* L, int n, zc* X, int nrhs, int unit, int cj, int upper) {
  if (!unit)
    for (int t = 0; t < n; t++) {
      int i = upper ? n - 1 - t : t;
      if (zero(AT(L, n, i, i))) return OR_SINGULAR_MATRIX;
    }
  /* op(L)[r][i] row-contiguous */
  zc* Lo = zalloc((size_t)n * n);
#pragma omp parallel for schedule(static) if ((size_t)n * n > 16384)
  for (int r = 0; r < n; r++)
    for (int i = 0; i < n; i++) Lo[(size_t)r * n + i] = cj ? conjz(AT(L, n, i, r)) : AT(L, n, r, i);
  enum { JC = 16 };
  int nch = (nrhs + JC - 1) / JC;
#pragma omp parallel for schedule(dynamic) if ((size_t)n * n * nrhs > 100000)
  for (int c = 0; c < nch; c++) {
    int j0 = c * JC, j1 = j0 + JC < nrhs ? j0 + JC : nrhs;
    for (int t = 0; t < n; t++) {
      int r = upper ? n - 1 - t : t;
      zc* xr = &AT(X, nrhs, r, 0);
      const zc* lr = Lo + (size_t)r * n;
      if (!upper) {
        for (int i = 0; i < r; i++) {
          const zc* xi = &AT(X, nrhs, i, 0);
          for (int j = j0; j < j1; j++) xr[j] = c_sub(f, xr[j], c_mul(f, lr[i], xi[j]));
        }
      } else {
        for (int i = n - 1; i > r; i--) {
          const zc* xi = &AT(X, nrhs, i, 0);
          for (int j = j0; j < j1; j++) xr[j] = c_sub(f, xr[j], c_mul(f, lr[i], xi[j]));
        }
      }
      if (!unit) {
        zc d = lr[r];
        for (int j = j0; j < j1; j++) xr[j] = c_div(f, xr[j], d);
      }
    }
  }
  free(Lo);
  return OR_OK;
}
static int solve_lower(fmt_t f, const zc* L, int n, zc* X, int nrhs, int unit, int cj) {
  return solve_tri(f, L, n, X, nrhs, unit, cj, 0);
}
static int solve_upper(fmt_t f, const zc* Um, int n, zc* X, int nrhs, int unit, int cj) {
  return solve_tri(f, Um, n, X, nrhs, unit, cj, 1);
}

/* lu_solve(F, B, side, transpose); left: B is n x nrhs; right: B is nrows x n */
static int lu_solve_core(fmt_t f, const zc* LU, const long long* piv, int n, const zc* B, int rows, int cols,
                         int right, int cj, zc* X) {
  if (right) {
    /* X A = B <=> A* X* = B*, X A* = B <=> A X* = B* (linalg.py:425-429) */
    zc* Bt = zalloc((size_t)rows * cols);
    for (int i = 0; i < rows; i++)
      for (int j = 0; j < cols; j++) AT(Bt, rows, j, i) = conjz(AT(B, cols, i, j));
    zc* Yt = zalloc((size_t)rows * cols);
    int rc = lu_solve_core(f, LU, piv, n, Bt, cols, rows, 0, !cj, Yt);
    for (int i = 0; i < rows; i++)
      for (int j = 0; j < cols; j++) AT(X, cols, i, j) = conjz(AT(Yt, rows, j, i));
    free(Bt); free(Yt);
    return rc;
  }
  memcpy(X, B, sizeof(zc) * (size_t)rows * cols);
  int rc;
  if (!cj) {
    apply_pivots(X, cols, piv, n, 0);
    solve_lower(f, LU, n, X, cols, 1, 0);
    rc = solve_upper(f, LU, n, X, cols, 0, 0);
    return rc;
  }
  rc = solve_lower(f, LU, n, X, cols, 0, 1);
  if (rc) return rc;
  solve_upper(f, LU, n, X, cols, 1, 1);
  apply_pivots(X, cols, piv, n, 1);
  return OR_OK;
}

int oracle_lu_solve(int f32, const zc* LU, const long long* piv, int n, const zc* B, int rows, int cols,
                    int right, int cj, zc* X) {
  fmt_t f = {f32};
  return lu_solve_core(f, LU, piv, n, B, rows, cols, right, cj, X);
}

/* ---------------------------------------------------------------------- */
/* triangular Sylvester recurrence (sylvester.py:111-157)                  */

static int is_upper(const zc* T, int n) {
  for (int i = 0; i < n; i++) for (int j = 0; j < i; j++) if (!zero(AT(T, n, i, j))) return 0;
  return 1;
}
static int is_lower(const zc* T, int n) {
  for (int i = 0; i < n; i++) for (int j = i + 1; j < n; j++) if (!zero(AT(T, n, i, j))) return 0;
  return 1;
}

static int solve_sylv_tri_core(fmt_t f, const zc* TA, int m, const zc* TB, int n, const zc* C, zc* Y) {
  /* Column recurrence of sylvester.py:111-157.  Restated with (i) the back
   * substitution blocked by row panels -- row r still receives its updates
   * from i = m-1 down to r+1 in that order -- and the updates of the rows
   * above a panel split across threads, (ii) the rank-1 update of the
   * remaining columns split by rows.  Per-entry arithmetic is unchanged. */
  if (!(m == 1 || is_upper(TA, m))) return OR_DIMENSION;
  int lower = 0;
  if (n > 1 && !is_upper(TB, n)) {
    if (is_lower(TB, n)) lower = 1; else return OR_DIMENSION;
  }
  zc* W = zalloc((size_t)m * n);
  memcpy(W, C, sizeof(zc) * (size_t)m * n);
  zc* col = zalloc(m);
  zc* y = zalloc(m);
  int rc = OR_OK;
  enum { PB = 128 };
  for (int t = 0; t < n && !rc; t++) {
    int j = lower ? n - 1 - t : t;
    zc shift = AT(TB, n, j, j);
    for (int i = 0; i < m; i++) { col[i] = AT(W, n, i, j); y[i] = Z(0.0, 0.0); }
    for (int r1 = m; r1 > 0 && !rc; r1 -= PB) {
      int r0 = r1 - PB > 0 ? r1 - PB : 0;
      for (int i = r1 - 1; i >= r0; i--) {
        zc d = c_add(f, AT(TA, m, i, i), shift);
        if (zero(d)) { g_err_row = i; g_err_col = j; rc = OR_SINGULAR_EQUATION; break; }
        y[i] = c_div(f, col[i], d);
        for (int r = r0; r < i; r++) col[r] = c_sub(f, col[r], c_mul(f, AT(TA, m, r, i), y[i]));
      }
      if (rc) break;
#pragma omp parallel for schedule(static) if ((size_t)r0 * (r1 - r0) > 32768)
      for (int r = 0; r < r0; r++) {
        const zc* tr = &AT(TA, m, r, 0);
        zc v = col[r];
        for (int i = r1 - 1; i >= r0; i--) v = c_sub(f, v, c_mul(f, tr[i], y[i]));
        col[r] = v;
      }
    }
    if (rc) break;
    for (int i = 0; i < m; i++) if (!zfinite(y[i])) { rc = OR_NUMERIC_BREAKDOWN; g_err_col = j; break; }
    if (rc) break;
    for (int i = 0; i < m; i++) AT(Y, n, i, j) = y[i];
    int c0 = lower ? 0 : j + 1, c1 = lower ? j : n;
#pragma omp parallel for schedule(static) if ((size_t)m * (c1 - c0) > 32768)
    for (int i = 0; i < m; i++) {
      zc yi = y[i];
      zc* wr = &AT(W, n, i, 0);
      const zc* tb = &AT(TB, n, j, 0);
      for (int jj = c0; jj < c1; jj++) wr[jj] = c_sub(f, wr[jj], c_mul(f, yi, tb[jj]));
    }
  }
  free(W); free(col); free(y);
  return rc;
}

int oracle_solve_sylv_tri(int f32, const zc* TA, int m, const zc* TB, int n, const zc* C, zc* Y,
                          int* err_row, int* err_col) {
  fmt_t f = {f32};
  g_err_row = g_err_col = -1;
  int rc = solve_sylv_tri_core(f, TA, m, TB, n, C, Y);
  if (err_row) *err_row = g_err_row;
  if (err_col) *err_col = g_err_col;
  return rc;
}

/* ---------------------------------------------------------------------- */
/* residual metric (sylvester.py:199-209), binary64                         */

double oracle_residual(const zc* A, const zc* B, const zc* C, const zc* X, int m, int n) {
  /* ||A X + X B - C||_F / (||C||_F + ||X||_F (||A||_F + ||B||_F)) in binary64.
   * The reference evaluates the products with numpy/OpenBLAS, so only the
   * value (to a few ulps), not the summation order, is restated. */
  fmt_t fh = {0};
  zc* AX = zalloc((size_t)m * n);
  zc* XB = zalloc((size_t)m * n);
  gemm_core(fh, Z(1.0, 0.0), 'N', A, m, 'N', X, n, Z(0.0, 0.0), NULL, 0, AX, n, m, n, m);
  gemm_core(fh, Z(1.0, 0.0), 'N', X, n, 'N', B, n, Z(0.0, 0.0), NULL, 0, XB, n, m, n, n);
  double num = 0.0;
  for (size_t e = 0; e < (size_t)m * n; e++) {
    double sr = AX[e].re + XB[e].re - C[e].re, si = AX[e].im + XB[e].im - C[e].im;
    num += sr * sr + si * si;
  }
  free(AX); free(XB);
  num = sqrt(num);
  double den = fro(C, (size_t)m * n) + fro(X, (size_t)m * n) * (fro(A, (size_t)m * m) + fro(B, (size_t)n * n));
  if (den == 0.0) return 0.0;
  return num / den;
}

int oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

/* ---------------------------------------------------------------------- */
/* Alg. 1: stationary refinement (refinement.py:95-141), binary64           */

typedef struct {
  int status;        /* OR_* of a raised error, else 0 */
  int iterations;
  int converged;
  int failure;       /* 0 none, 1 singular_equation, 2 nan_breakdown, 3 non_convergence */
  int fail_stage;    /* 0 refinement, 1 initial triangular solve */
  int fail_row, fail_col;
  double residual;
  int n_norms;
  double norms[256];
} oracle_report;

static int stat_core(const zc* TA, const zc* dTA, const zc* TB, const zc* dTB, const zc* C, const zc* Y0,
                     int m, int n, double eps, int max_iter, zc* Y, oracle_report* rep) {
  fmt_t f = {0};
  zc* SA = zalloc((size_t)m * m);
  zc* SB = zalloc((size_t)n * n);
  zc* R = zalloc((size_t)m * n);
  zc* R2 = zalloc((size_t)m * n);
  zc* D = zalloc((size_t)m * n);
  for (size_t i = 0; i < (size_t)m * m; i++) SA[i] = c_add(f, TA[i], dTA[i]);
  for (size_t i = 0; i < (size_t)n * n; i++) SB[i] = c_add(f, TB[i], dTB[i]);
  memcpy(Y, Y0, sizeof(zc) * (size_t)m * n);
  int i = 0, rc = OR_OK;
  rep->converged = 0; rep->failure = 0; rep->n_norms = 0;
  while (i < max_iter) {
    gemm_core(f, Z(-1.0, 0.0), 'N', SA, m, 'N', Y, n, Z(1.0, 0.0), C, n, R, n, m, n, m);
    gemm_core(f, Z(-1.0, 0.0), 'N', Y, n, 'N', SB, n, Z(1.0, 0.0), R, n, R2, n, m, n, n);
    g_err_row = g_err_col = -1;
    int trc = solve_sylv_tri_core(f, TA, m, TB, n, R2, D);
    if (trc == OR_NUMERIC_BREAKDOWN) { rep->failure = 2; break; }
    if (trc == OR_SINGULAR_EQUATION) { rc = trc; rep->fail_row = g_err_row; rep->fail_col = g_err_col; break; }
    if (trc) { rc = trc; break; }
    for (size_t e = 0; e < (size_t)m * n; e++) Y[e] = c_add(f, Y[e], D[e]);
    i++;
    double nD = fro(D, (size_t)m * n), nY = fro(Y, (size_t)m * n);
    if (rep->n_norms < 256) rep->norms[rep->n_norms++] = nD;
    if (!(isfinite(nD) && isfinite(nY))) { rep->failure = 2; break; }
    if (nD <= eps * nY) { rep->converged = 1; break; }
  }
  if (!rc && rep->failure == 0 && !rep->converged) rep->failure = 3;
  rep->iterations = i;
  rep->status = rc;
  if (!rc) rep->residual = oracle_residual(SA, SB, C, Y, m, n);
  free(SA); free(SB); free(R); free(R2); free(D);
  return rc;
}

int oracle_stat(const zc* TA, const zc* dTA, const zc* TB, const zc* dTB, const zc* C, const zc* Y0,
                int m, int n, double eps, int max_iter, zc* Y, oracle_report* rep) {
  memset(rep, 0, sizeof(*rep));
  return stat_core(TA, dTA, TB, dTB, C, Y0, m, n, eps, max_iter, Y, rep);
}

/* ---------------------------------------------------------------------- */
/* mp_orth / mp_inv (refinement.py:185-297)                                */

static void conj_transpose(const zc* A, int rows, int cols, zc* out) {
  for (int i = 0; i < rows; i++)
    for (int j = 0; j < cols; j++) AT(out, rows, j, i) = conjz(AT(A, cols, i, j));
}

/* variant 0 = mp_orth, 1 = mp_inv; kind 0 general, 1 lyapunov.
 * Raised errors return their OR_* code (rep->status); typed failures are
 * reported in rep->failure with X all-NaN when the initial solve failed. */
int oracle_mp_solve(int variant, int f32_low, int kind, const zc* A, const zc* B, const zc* C, int m, int n,
                    double eps, int max_iter, int y0_zero, zc* X, oracle_report* rep) {
  memset(rep, 0, sizeof(*rep));
  fmt_t fl = {f32_low}, fh = {0};
  int rc;
  size_t mm = (size_t)m * m, nn = (size_t)n * n, mn = (size_t)m * n;
  zc *TA = zalloc(mm), *UA = zalloc(mm), *TB = zalloc(nn), *UB = zalloc(nn);
  zc *QA = zalloc(mm), *RA = zalloc(mm), *QB = zalloc(nn), *RB = zalloc(nn);
  zc *F = zalloc(mn), *tmp = zalloc(mm > mn ? (mm > nn ? mm : nn) : (mn > nn ? mn : nn));
  zc *LA = zalloc(mm), *LB = zalloc(nn), *Y0 = zalloc(mn), *Fl = zalloc(mn), *Y = zalloc(mn);
  zc *UAh = zalloc(mm), *Wm = zalloc(mm), *Wn = zalloc(nn), *Zm = zalloc(mn);
  long long *pivA = calloc(m, sizeof(long long)), *pivB = calloc(n, sizeof(long long));

  /* _low_precision_schur_pair (refinement.py:190-197) */
  rc = enter(fl, A, TA, mm);
  if (!rc) rc = schur_core(fl, TA, UA, m, NULL);
  if (!rc) {
    if (kind == 1) { memcpy(UB, UA, sizeof(zc) * mm); conj_transpose(TA, m, m, TB); }
    else { rc = enter(fl, B, TB, nn); if (!rc) rc = schur_core(fl, TB, UB, n, NULL); }
  }
  if (rc) goto done;

  if (variant == 0) {
    rc = mgs_qr_core(fh, UA, QA, RA, m, m);
    if (!rc) {
      if (kind == 1) memcpy(QB, QA, sizeof(zc) * mm);
      else rc = mgs_qr_core(fh, UB, QB, RB, n, n);
    }
    if (rc) goto done;
    /* F = (Q_A^H C) Q_B ; L_A = (Q_A^H A) Q_A - T_A */
    gemm_core(fh, Z(1, 0), 'C', QA, m, 'N', C, n, Z(0, 0), NULL, 0, tmp, n, m, n, m);
    gemm_core(fh, Z(1, 0), 'N', tmp, n, 'N', QB, n, Z(0, 0), NULL, 0, F, n, m, n, n);
    gemm_core(fh, Z(1, 0), 'C', QA, m, 'N', A, m, Z(0, 0), NULL, 0, tmp, m, m, m, m);
    gemm_core(fh, Z(1, 0), 'N', tmp, m, 'N', QA, m, Z(0, 0), NULL, 0, LA, m, m, m, m);
    for (size_t e = 0; e < mm; e++) LA[e] = c_sub(fh, LA[e], TA[e]);
    if (kind == 1) conj_transpose(LA, m, m, LB);
    else {
      gemm_core(fh, Z(1, 0), 'C', QB, n, 'N', B, n, Z(0, 0), NULL, 0, tmp, n, n, n, n);
      gemm_core(fh, Z(1, 0), 'N', tmp, n, 'N', QB, n, Z(0, 0), NULL, 0, LB, n, n, n, n);
      for (size_t e = 0; e < nn; e++) LB[e] = c_sub(fh, LB[e], TB[e]);
    }
  } else {
    conj_transpose(UA, m, m, UAh);
    rc = lu_core(fh, UAh, QA, pivA, m);              /* QA holds LU(U_A^H) */
    if (!rc && kind != 1) rc = lu_core(fh, UB, QB, pivB, n);
    if (rc) goto done;
    gemm_core(fh, Z(1, 0), 'C', UA, m, 'N', C, n, Z(0, 0), NULL, 0, tmp, n, m, n, m);
    gemm_core(fh, Z(1, 0), 'N', tmp, n, 'N', UB, n, Z(0, 0), NULL, 0, F, n, m, n, n);
    gemm_core(fh, Z(1, 0), 'C', UA, m, 'N', A, m, Z(0, 0), NULL, 0, Wm, m, m, m, m);
    lu_solve_core(fh, QA, pivA, m, Wm, m, m, 1, 0, LA);
    for (size_t e = 0; e < mm; e++) LA[e] = c_sub(fh, LA[e], TA[e]);
    if (kind == 1) conj_transpose(LA, m, m, LB);
    else {
      gemm_core(fh, Z(1, 0), 'N', B, n, 'N', UB, n, Z(0, 0), NULL, 0, Wn, n, n, n, n);
      lu_solve_core(fh, QB, pivB, n, Wn, n, n, 0, 0, LB);
      for (size_t e = 0; e < nn; e++) LB[e] = c_sub(fh, LB[e], TB[e]);
    }
  }

  /* Y0 = solve_sylv_tri(T_A, T_B, round_l(F)) in u_l (refinement.py:200-202) */
  for (size_t e = 0; e < mn; e++) Fl[e] = Z(round_in(fl, F[e].re), round_in(fl, F[e].im));
  g_err_row = g_err_col = -1;
  rc = solve_sylv_tri_core(fl, TA, m, TB, n, Fl, Y0);
  if (rc == OR_SINGULAR_EQUATION || rc == OR_NUMERIC_BREAKDOWN) {
    if (!y0_zero) {
      rep->failure = rc == OR_SINGULAR_EQUATION ? 1 : 2;
      rep->fail_stage = 1; rep->fail_row = g_err_row; rep->fail_col = g_err_col;
      for (size_t e = 0; e < mn; e++) X[e] = Z(NAN, NAN);
      rep->residual = NAN; rep->iterations = 0;
      rc = OR_OK;
      goto done;
    }
    memset(Y0, 0, sizeof(zc) * mn);
    rc = OR_OK;
  } else if (rc) goto done;

  {
    double e_ = eps > 0 ? eps : 1e-12 * (m > n ? m : n);
    int src = stat_core(TA, LA, TB, LB, F, Y0, m, n, e_, max_iter, Y, rep);
    if (src == OR_SINGULAR_EQUATION) {
      rep->failure = 1; rep->fail_stage = 0; rep->status = 0; rep->iterations = 0; rep->converged = 0;
      rep->n_norms = 0;
      for (size_t e = 0; e < mn; e++) X[e] = Z(NAN, NAN);
      rep->residual = NAN;
      rc = OR_OK;
      goto done;
    }
    if (src) { rc = src; goto done; }
  }
  if (variant == 0) {
    gemm_core(fh, Z(1, 0), 'N', QA, m, 'N', Y, n, Z(0, 0), NULL, 0, tmp, n, m, n, m);
    gemm_core(fh, Z(1, 0), 'N', tmp, n, 'C', QB, n, Z(0, 0), NULL, 0, X, n, m, n, n);
  } else {
    lu_solve_core(fh, QA, pivA, m, Y, m, n, 0, 0, Zm);
    if (kind == 1) lu_solve_core(fh, QA, pivA, m, Zm, m, n, 1, 1, X);
    else lu_solve_core(fh, QB, pivB, n, Zm, m, n, 1, 0, X);
  }
  rep->residual = oracle_residual(A, B, C, X, m, n);

done:
  rep->status = rc;
  free(TA); free(UA); free(TB); free(UB); free(QA); free(RA); free(QB); free(RB);
  free(F); free(tmp); free(LA); free(LB); free(Y0); free(Fl); free(Y);
  free(UAh); free(Wm); free(Wn); free(Zm); free(pivA); free(pivB);
  return rc;
}

int oracle_report_size(void) { return (int)sizeof(oracle_report); }
