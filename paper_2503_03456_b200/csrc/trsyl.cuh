// trsyl.cuh -- T_A Y + Y T_B = W for (quasi-)triangular T_A (upper) and T_B (upper, or
// lower for the Lyapunov adjoint), in place on W.
//
// Replaces the reference's column recurrence `solve_sylv_tri` (pkg/src/mpsylv/sylvester.py:111-157):
// same equation, same ascending (T_B upper) / descending (T_B lower) column order,
// same typed failures -- an exactly singular diagonal pair -> SINGULAR_EQUATION
// at (row, col) (sylvester.py:141-143), non-finite values -> NUMERIC_BREAKDOWN
// (sylvester.py:147-149).  Real Schur factors may carry 2x2 diagonal blocks;
// they are solved as coupled 2x2/4x4 systems and never split across tiles.
//
// B200 design: the m x n unknown is tiled into NB x NB blocks (boundaries nudged
// so no 2x2 block straddles a tile edge).  Block (I,J) depends on the blocks below
// it in its column and before it in its row, so blocks on one anti-diagonal are
// independent.  One kernel launch per anti-diagonal d: every pending block applies
// the two rank-NB GEMM updates coming from diagonal d-1 (in registers, smem-tiled),
// and blocks on diagonal d then solve themselves in shared memory with an
// element-level wavefront over 1x1/2x2 units.  (m/NB + n/NB - 1) launches total.
#pragma once
#include "common.cuh"
#include "gemm_dmma.cuh"

namespace msy {

// LEAF2: two-level leaf (sub-tile wavefront); measured faster for the 64-wide leaves,
// slower for the 32-wide complex128 leaves, which keep the single-level wavefront
// LEAF: 3 = lazy single-warp element wavefront (each unit gathers its row / column dot
// products when it becomes ready: ~nru + ncu warp-synchronous steps, no block barriers);
// 2 = two-level sub-tile wavefront; 1 = eager single-level wavefront (block barriers)
#ifndef MSY_TRS_LEAF
#define MSY_TRS_LEAF 3
#endif
template <class S> struct TrsylCfg { static constexpr int NB = 64; static constexpr int LEAF = MSY_TRS_LEAF; };
template <> struct TrsylCfg<cdouble> { static constexpr int NB = 32; static constexpr int LEAF = 3; };

enum { TRS_OK = 0, TRS_SINGULAR = 1, TRS_BREAKDOWN = 2 };

// Reciprocal for the unit solves on the leaf's critical path: the hardware approximation
// refined by Newton steps (two for fp64, one for fp32) -- a few dependent FMAs instead of
// the IEEE division routine.  Callers handle exact zeros before calling.
__device__ __forceinline__ float trs_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return fmaf(r, fmaf(-x, r, 1.0f), r);
}
__device__ __forceinline__ double trs_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}
template <class R> __device__ __forceinline__ cplx<R> trs_rcp(cplx<R> x) { return cplx<R>(R(1)) / x; }

// Inverse of the p x q unit's Kronecker matrix  I (x) TA_RR + TB_CC^T (x) I  (unknowns ordered
// r + PP c, as in unit_solve), by Gauss-Jordan with partial pivoting, written row-major into
// out[0 .. (PP QQ)^2).  Returns false on an exactly zero pivot (the singular diagonal pair of
// sylvester.py:141-143).  Precomputed for every unit pair of a leaf before its wavefront, so
// the wavefront's per-unit solve is a small mat-vec.
template <class S, int PP, int QQ>
__device__ __forceinline__ bool unit_inverse(const S* As, const S* Bs, int P, int i, int j, S* out) {
  typedef typename tr<S>::R R;
  constexpr int NS = PP * QQ;
  S M[NS][2 * NS];
#pragma unroll
  for (int c = 0; c < QQ; c++)
#pragma unroll
    for (int r = 0; r < PP; r++) {
      const int u = r + PP * c;
#pragma unroll
      for (int v = 0; v < 2 * NS; v++) M[u][v] = (v == NS + u) ? S(1) : S(0);
#pragma unroll
      for (int r2 = 0; r2 < PP; r2++) M[u][r2 + PP * c] = M[u][r2 + PP * c] + As[(i + r) + (i + r2) * P];
#pragma unroll
      for (int c2 = 0; c2 < QQ; c2++) M[u][r + PP * c2] = M[u][r + PP * c2] + Bs[(j + c2) + (j + c) * P];
    }
  bool ok = true;
#pragma unroll
  for (int c = 0; c < NS; c++) {
#pragma unroll
    for (int r = c + 1; r < NS; r++)
      if (abs1(M[r][c]) > abs1(M[c][c]))
#pragma unroll
        for (int v = 0; v < 2 * NS; v++) { S t = M[c][v]; M[c][v] = M[r][v]; M[r][v] = t; }
    if (abs1(M[c][c]) == R(0)) ok = false;
    const S inv = ok ? S(1) / M[c][c] : S(0);
#pragma unroll
    for (int v = 0; v < 2 * NS; v++) M[c][v] = M[c][v] * inv;
#pragma unroll
    for (int r = 0; r < NS; r++) {
      if (r == c) continue;
      const S f = M[r][c];
#pragma unroll
      for (int v = 0; v < 2 * NS; v++) M[r][v] = M[r][v] - f * M[c][v];
    }
  }
#pragma unroll
  for (int r = 0; r < NS; r++)
#pragma unroll
    for (int v = 0; v < NS; v++) out[r * NS + v] = M[r][NS + v];
  return ok;
}

// leaf wavefront with 4 threads per unit (real types); complex keeps one thread per unit
template <class S> constexpr bool kLeafGroups = std::is_same<S, float>::value || std::is_same<S, double>::value;

// status: [0] = min key (crank*m + m-1-row) of a singular unit, INT_MAX if none
__global__ void trsyl_status_init(int* status) {
  status[0] = 0x7fffffff; status[1] = -1; status[2] = -1; status[3] = 0;
}

// boundaries: rb[0..nbi], cb[0..nbj]; nominal k*NB moved by +1 if it would split a 2x2 block
template <class S>
__global__ void trsyl_partition_kernel(int m, const S* TA, int lda, int n, const S* TB, int ldb, int lowerB, int NB,
                                       int* rb, int nbi, int* cb, int nbj) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k <= nbi) {
    int b = k == nbi ? m : k * NB;
    if (k > 0 && k < nbi && !iszero(TA[b + (size_t)(b - 1) * lda])) b++;
    rb[k] = b;
  }
  if (k <= nbj) {
    int b = k == nbj ? n : k * NB;
    if (k > 0 && k < nbj) {
      S c = lowerB ? TB[(b - 1) + (size_t)b * ldb] : TB[b + (size_t)(b - 1) * ldb];
      if (!iszero(c)) b++;
    }
    cb[k] = b;
  }
}

// solve the pq x pq Kronecker system in place (Gaussian elimination, partial pivoting);
// returns false on an exactly zero pivot
template <class S>
__device__ bool small_solve(int nsys, S M[4][4], S rhs[4]) {
  typedef typename tr<S>::R R;
  for (int c = 0; c < nsys; c++) {
    int p = c;
    R best = abs1(M[c][c]);
    for (int r = c + 1; r < nsys; r++)
      if (abs1(M[r][c]) > best) { best = abs1(M[r][c]); p = r; }
    if (best == R(0)) return false;
    if (p != c) {
      for (int q = 0; q < nsys; q++) { S t = M[c][q]; M[c][q] = M[p][q]; M[p][q] = t; }
      S t = rhs[c]; rhs[c] = rhs[p]; rhs[p] = t;
    }
    for (int r = c + 1; r < nsys; r++) {
      S f = M[r][c] / M[c][c];
      for (int q = c; q < nsys; q++) M[r][q] = M[r][q] - f * M[c][q];
      rhs[r] = rhs[r] - f * rhs[c];
    }
  }
  for (int c = nsys - 1; c >= 0; c--) {
    S s = rhs[c];
    for (int q = c + 1; q < nsys; q++) s = s - M[c][q] * rhs[q];
    rhs[c] = s / M[c][c];
  }
  return true;
}

// Solve the p x q unit system  TA_RR Y + Y TB_CC = W_RC  in registers (compile-time
// sizes: fully unrolled Gaussian elimination with partial pivoting on the pq x pq
// Kronecker matrix I (x) TA_RR + TB_CC^T (x) I).  Writes Y over W; false on an
// exactly zero pivot (then Y = NaN).
template <class S, int PP, int QQ>
__device__ __forceinline__ bool unit_solve(const S* As, const S* Bs, S* Ws, int P, int i, int j) {
  typedef typename tr<S>::R R;
  constexpr int NS = PP * QQ;
  S M[NS][NS], x[NS];
#pragma unroll
  for (int c = 0; c < QQ; c++)
#pragma unroll
    for (int r = 0; r < PP; r++) {
      const int u = r + PP * c;
      x[u] = Ws[(i + r) + (j + c) * P];
#pragma unroll
      for (int v = 0; v < NS; v++) M[u][v] = S(0);
#pragma unroll
      for (int r2 = 0; r2 < PP; r2++) M[u][r2 + PP * c] = M[u][r2 + PP * c] + As[(i + r) + (i + r2) * P];
#pragma unroll
      for (int c2 = 0; c2 < QQ; c2++) M[u][r + PP * c2] = M[u][r + PP * c2] + Bs[(j + c2) + (j + c) * P];
    }
  bool ok = true;
  S dinv[NS];  // reciprocal pivots: the back substitution multiplies (no divisions on the chain)
#pragma unroll
  for (int c = 0; c < NS; c++) {
    // partial pivoting by swapping values (indices stay compile-time constants)
#pragma unroll
    for (int r = c + 1; r < NS; r++) {
      if (abs1(M[r][c]) > abs1(M[c][c])) {
#pragma unroll
        for (int v = 0; v < NS; v++) { S t = M[c][v]; M[c][v] = M[r][v]; M[r][v] = t; }
        S t = x[c]; x[c] = x[r]; x[r] = t;
      }
    }
    if (abs1(M[c][c]) == R(0)) ok = false;
    const S inv = ok ? trs_rcp(M[c][c]) : S(0);
    dinv[c] = inv;
#pragma unroll
    for (int r = c + 1; r < NS; r++) {
      const S f = M[r][c] * inv;
#pragma unroll
      for (int v = c + 1; v < NS; v++) M[r][v] = M[r][v] - f * M[c][v];
      x[r] = x[r] - f * x[c];
    }
  }
#pragma unroll
  for (int c = NS - 1; c >= 0; c--) {
    S s = x[c];
#pragma unroll
    for (int v = c + 1; v < NS; v++) s = s - M[c][v] * x[v];
    x[c] = s * dinv[c];
  }
#pragma unroll
  for (int c = 0; c < QQ; c++)
#pragma unroll
    for (int r = 0; r < PP; r++) Ws[(i + r) + (j + c) * P] = ok ? x[r + PP * c] : mk<S>(NAN, NAN);
  return ok;
}

#ifndef MSY_TRS_MINB
#define MSY_TRS_MINB 2
#endif
constexpr int TRS_TPB = 256;  // 2 CTAs per SM: the update of one block overlaps another's loads
// ---------------------------------------------------------------------------
// Left-looking schedule (real types).  Tiles are at most TL_LD = 64 on a side (nominal
// spacing 63, nudged +1 at a 2x2 block).  When tile (I, J) is due (anti-diagonal d) its
// right-hand side is
//   R = W[I, J] - T_A[I, i1:m] Y[i1:m, J] - Y[I, K_B] T_B[K_B, J],
// K_B = [0, j0) for an upper T_B, [j1, n) for the lower (Lyapunov adjoint) one: all of
// it already solved.  Both products are cut into K chunks of TL_KC; one CTA computes one
// chunk of one tile into a private partial (trsyl_lpart_*), and the tile's leaf solve
// subtracts the partials in chunk order (deterministic) before its wavefront.  Work per
// solve is the same mn(m+n) flops as the eager schedule, but it runs as ~100 waves of
// independent 64 x 64 x TL_KC GEMM tiles (fp64 on DMMA) instead of SIMT rank-64 updates,
// and W is written once per tile.
constexpr int TL_LD = 64, TL_TILE = TL_LD * TL_LD, TL_SPACING = TL_LD - 1, TL_KC = 256;

// Chunks of a leaf, in the fixed summation order: [0] the tile just below (A part, solved on
// the previous diagonal), [1] the tile just before in solve order (B part, previous diagonal),
// then the older A-part range in TL_KC pieces, then the older B-part range.  The two "new"
// chunks may be empty (zero partials).  The older chunks only read tiles solved two or more
// diagonals back, so they are computed on a side stream while the previous diagonal solves.
struct LeafK {
  int na0, na1, nb0, nb1;   // new ranges [na0, na1) (A) and [nb0, nb1) (B)
  int oa0, oa1, ob0, ob1;   // older ranges
};
__host__ __device__ __forceinline__ LeafK lleaf_ranges(int m, int n, int lowerB, int nbi, int nbj, const int* rb,
                                                       const int* cb, int I, int J) {
  LeafK k;
  const int i1 = rb[I + 1];
  k.na0 = i1;
  k.na1 = I + 1 < nbi ? rb[I + 2] : m;
  k.oa0 = k.na1;
  k.oa1 = m;
  if (!lowerB) {
    const int j0 = cb[J];
    k.nb1 = j0;
    k.nb0 = J >= 1 ? cb[J - 1] : 0;
    k.ob0 = 0;
    k.ob1 = k.nb0;
  } else {
    const int j1 = cb[J + 1];
    k.nb0 = j1;
    k.nb1 = J + 1 < nbj ? cb[J + 2] : n;
    k.ob0 = k.nb1;
    k.ob1 = n;
  }
  return k;
}
__host__ __device__ __forceinline__ int lleaf_old_chunks(const LeafK& k) {
  return (k.oa1 - k.oa0 + TL_KC - 1) / TL_KC + (k.ob1 - k.ob0 + TL_KC - 1) / TL_KC;
}
__host__ __device__ __forceinline__ int lleaf_chunks(const LeafK& k) { return 2 + lleaf_old_chunks(k); }

// decode (leaf b of anti-diagonal d, chunk c) -> operand pointers and K range; false if idle
template <class S>
__device__ __forceinline__ bool lleaf_operands(int m, int n, const S* TA, int lda, const S* TB, int ldb, int lowerB,
                                               const S* W, int ldw, const int* rb, const int* cb, int nbi, int nbj,
                                               int d, int b, int c, int& bi, int& bj, const S*& Ap, int& ldA,
                                               const S*& Bp, int& ldB, int& klen) {
  const int llo = max(0, d - nbj + 1);
  const int rI = llo + b, cJ = d - rI;
  const int I = nbi - 1 - rI, J = lowerB ? nbj - 1 - cJ : cJ;
  const int i0 = rb[I], i1 = rb[I + 1], j0 = cb[J], j1 = cb[J + 1];
  bi = i1 - i0;
  bj = j1 - j0;
  if (bi <= 0 || bj <= 0) return false;
  const LeafK k = lleaf_ranges(m, n, lowerB, nbi, nbj, rb, cb, I, J);
  int a0, a1, isA;
  if (c == 0) { a0 = k.na0; a1 = k.na1; isA = 1; }
  else if (c == 1) { a0 = k.nb0; a1 = k.nb1; isA = 0; }
  else {
    c -= 2;
    const int noa = (k.oa1 - k.oa0 + TL_KC - 1) / TL_KC, nob = (k.ob1 - k.ob0 + TL_KC - 1) / TL_KC;
    if (c < noa) { a0 = k.oa0 + c * TL_KC; a1 = min(k.oa1, a0 + TL_KC); isA = 1; }
    else if (c - noa < nob) { a0 = k.ob0 + (c - noa) * TL_KC; a1 = min(k.ob1, a0 + TL_KC); isA = 0; }
    else return false;
  }
  klen = max(0, a1 - a0);
  if (isA) {  // T_A[i0:i1, k] Y[k, j0:j1]
    Ap = TA + i0 + (size_t)a0 * lda; ldA = lda;
    Bp = W + a0 + (size_t)j0 * ldw; ldB = ldw;
  } else {    // Y[i0:i1, k] T_B[k, j0:j1]
    Ap = W + i0 + (size_t)a0 * ldw; ldA = ldw;
    Bp = TB + a0 + (size_t)j0 * ldb; ldB = ldb;
  }
  return true;
}

// fp64 partial: 64 x 64 x klen on DMMA (4 warps, 32 x 32 per warp), staged like gemm_dmma_kernel
__global__ void __launch_bounds__(128) trsyl_lpart_dmma_kernel(int m, int n, const double* __restrict__ TA, int lda,
                                                               const double* __restrict__ TB, int ldb, int lowerB,
                                                               const double* W, int ldw, const int* __restrict__ rb,
                                                               const int* __restrict__ cb, int nbi, int nbj, int d,
                                                               int maxch, int coff, double* __restrict__ part) {
  int bi, bj, ldA, ldB, klen;
  const double *Ap, *Bp;
  const int chunk = blockIdx.y + coff;
  if (!lleaf_operands<double>(m, n, TA, lda, TB, ldb, lowerB, W, ldw, rb, cb, nbi, nbj, d, blockIdx.x, chunk, bi,
                              bj, Ap, ldA, Bp, ldB, klen))
    return;
  __shared__ __align__(16) double As[2][DM_BK][DM_LD];
  __shared__ __align__(16) double Bs[2][DM_BK][DM_LD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[8], rbv[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int idx = tid + e * 128;
      const int i = idx & 63, k = idx >> 6;            // A: 64 x 16, i fastest
      ra[e] = (i < bi && k0 + k < klen) ? Ap[i + (size_t)(k0 + k) * ldA] : 0.0;
      const int kk = idx & 15, j = idx >> 4;           // B: 16 x 64, k fastest
      rbv[e] = (j < bj && k0 + kk < klen) ? Bp[(k0 + kk) + (size_t)j * ldB] : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int idx = tid + e * 128;
      As[buf][idx >> 6][idx & 63] = ra[e];
      Bs[buf][idx & 15][idx >> 4] = rbv[e];
    }
  };
  const int nk = (klen + DM_BK - 1) / DM_BK;
  load(0);
  store(0);
  __syncthreads();
  const int fr = lane >> 2, fc = lane & 3;
  for (int t = 0; t < nk; t++) {
    const int cur = t & 1;
    if (t + 1 < nk) load((t + 1) * DM_BK);
#pragma unroll
    for (int kk = 0; kk < DM_BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[cur][kk + fc][wm + i * 8 + fr];
#pragma unroll
      for (int j = 0; j < 4; j++) b[j] = Bs[cur][kk + fc][wn + j * 8 + fr];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (t + 1 < nk) store(cur ^ 1);
    __syncthreads();
  }
  double* out = part + ((size_t)blockIdx.x * maxch + chunk) * TL_TILE;
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) out[(wm + i * 8 + fr) + (size_t)(wn + j * 8 + fc * 2 + h) * TL_LD] = acc[i][j][h];
}

// fp32 (and generic) partial: SIMT, 256 threads, 4 x 4 register tile each, K staged by 16
template <class S>
__global__ void __launch_bounds__(256) trsyl_lpart_simt_kernel(int m, int n, const S* __restrict__ TA, int lda,
                                                               const S* __restrict__ TB, int ldb, int lowerB,
                                                               const S* W, int ldw, const int* __restrict__ rb,
                                                               const int* __restrict__ cb, int nbi, int nbj, int d,
                                                               int maxch, int coff, S* __restrict__ part) {
  int bi, bj, ldA, ldB, klen;
  const S *Ap, *Bp;
  const int chunk = blockIdx.y + coff;
  if (!lleaf_operands<S>(m, n, TA, lda, TB, ldb, lowerB, W, ldw, rb, cb, nbi, nbj, d, blockIdx.x, chunk, bi, bj,
                         Ap, ldA, Bp, ldB, klen))
    return;
  constexpr int KS = 16;
  __shared__ __align__(16) S As[2][KS][TL_LD + 4];
  __shared__ __align__(16) S Bs[2][KS][TL_LD + 4];
  const int tid = threadIdx.x, tr_ = tid & 15, tc = tid >> 4;
  S acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b] = S(0);
  S ra[4], rbv[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int idx = tid + e * 256;
      const int i = idx & 63, k = idx >> 6;
      ra[e] = (i < bi && k0 + k < klen) ? Ap[i + (size_t)(k0 + k) * ldA] : S(0);
      const int kk = idx & 15, j = idx >> 4;
      rbv[e] = (j < bj && k0 + kk < klen) ? Bp[(k0 + kk) + (size_t)j * ldB] : S(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int idx = tid + e * 256;
      As[buf][idx >> 6][idx & 63] = ra[e];
      Bs[buf][idx & 15][idx >> 4] = rbv[e];
    }
  };
  const int nk = (klen + KS - 1) / KS;
  load(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; t++) {
    const int cur = t & 1;
    if (t + 1 < nk) load((t + 1) * KS);
#pragma unroll
    for (int k = 0; k < KS; k++) {
      S a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        a[q] = As[cur][k][tr_ + 16 * q];
        b[q] = Bs[cur][k][tc + 16 * q];
      }
#pragma unroll
      for (int x = 0; x < 4; x++)
#pragma unroll
        for (int y = 0; y < 4; y++) acc[x][y] = fmac(a[x], b[y], acc[x][y]);
    }
    if (t + 1 < nk) store(cur ^ 1);
    __syncthreads();
  }
  S* out = part + ((size_t)blockIdx.x * maxch + chunk) * TL_TILE;
#pragma unroll
  for (int x = 0; x < 4; x++)
#pragma unroll
    for (int y = 0; y < 4; y++) out[(tr_ + 16 * x) + (size_t)(tc + 16 * y) * TL_LD] = acc[x][y];
}

// W[tile] -= sum of the tile's partials, in chunk order (deterministic); grid (leaf, 16 slices)
template <class S>
__global__ void __launch_bounds__(256) trsyl_lreduce_kernel(int m, int n, int lowerB, S* W, int ldw,
                                                            const int* __restrict__ rb, const int* __restrict__ cb,
                                                            int nbi, int nbj, int d, int maxch,
                                                            const S* __restrict__ part) {
  const int llo = max(0, d - nbj + 1);
  const int rI = llo + blockIdx.x, cJ = d - rI;
  const int I = nbi - 1 - rI, J = lowerB ? nbj - 1 - cJ : cJ;
  const int i0 = rb[I], i1 = rb[I + 1], j0 = cb[J], j1 = cb[J + 1];
  const int e = blockIdx.y * 256 + threadIdx.x, i = e % TL_LD, j = e / TL_LD;
  if (i >= i1 - i0 || j >= j1 - j0) return;
  const int nch = lleaf_chunks(lleaf_ranges(m, n, lowerB, nbi, nbj, rb, cb, I, J));
  const S* pp = part + (size_t)blockIdx.x * maxch * TL_TILE + e;
  S acc = S(0);
  int c = 0;
  for (; c + 4 <= nch; c += 4) {  // four loads in flight, summed in chunk order
    const S p0 = pp[(size_t)c * TL_TILE], p1 = pp[(size_t)(c + 1) * TL_TILE];
    const S p2 = pp[(size_t)(c + 2) * TL_TILE], p3 = pp[(size_t)(c + 3) * TL_TILE];
    acc = acc + p0; acc = acc + p1; acc = acc + p2; acc = acc + p3;
  }
  for (; c < nch; c++) acc = acc + pp[(size_t)c * TL_TILE];
  S* w = W + (i0 + i) + (size_t)(j0 + j) * ldw;
  *w = *w - acc;
}

template <class S>
__global__ void __launch_bounds__(TRS_TPB, MSY_TRS_MINB) trsyl_step_kernel(int m, int n, const S* __restrict__ TA, int lda,
                                                         const S* __restrict__ TB, int ldb, int lowerB, S* W, int ldw,
                                                         const int* __restrict__ rb, const int* __restrict__ cb, int nbi,
                                                         int nbj, int d, int* status, int dbg, int left = 0,
                                                         S* __restrict__ uinv = nullptr) {
  constexpr int NB = TrsylCfg<S>::NB;
  constexpr int P = 4 * ((NB + 1 + 3) / 4);  // padded tile edge (smem stride)
  constexpr int TG = 16;                     // 16 x 16 threads, RM x RM accumulators each
  constexpr int RM = (NB + 1 + TG - 1) / TG;
  // blockIdx.x enumerates the blocks that change at step d (rank space: rI = row rank from
  // the bottom, cJ = column rank in solve order): rows rI < d with cJ >= d - rI, then
  // columns cJ < d with rI >= d; at d = 0 the single block (0, 0).  Blocks with rI >= d
  // and cJ >= d receive nothing yet and are not launched.
  // The blocks that solve at this step (rank sum d: the leaves, on the critical path) take
  // the lowest block indices so they are scheduled first and their leaf solves overlap the
  // update-only waves; the update-only blocks follow in the original order.
  int rI = 0, cJ = 0;
  {
    int b = blockIdx.x;
    if (d > 0) {
      const int llo = max(0, d - nbj + 1), lhi = min(d, nbi - 1);
      const int nleaf = max(0, lhi - llo + 1);
      if (b < nleaf) {
        rI = llo + b;
        cJ = d - rI;
      } else {
        b -= nleaf;
        const int ra = min(d, nbi);
        rI = -1;
        for (int r = 0; r < ra; r++) {  // row r: blocks cJ in [d - r, nbj), the first is the leaf
          const int st = (d - r < nbj) ? d - r + 1 : d - r;
          const int len = max(0, nbj - st);
          if (b < len) { rI = r; cJ = st + b; break; }
          b -= len;
        }
        if (rI < 0) {  // columns cJ < min(d, nbj), rows rI >= d, without the leaf (d, 0)
          const int h = nbi - d;
          if (b < h - 1) { cJ = 0; rI = d + 1 + b; }
          else { b -= h - 1; cJ = 1 + b / h; rI = d + b % h; }
        }
      }
    }
  }
  const int I = nbi - 1 - rI, J = lowerB ? nbj - 1 - cJ : cJ;
  const int dd = rI + cJ;
  const int i0 = rb[I], i1 = rb[I + 1], j0 = cb[J], j1 = cb[J + 1];
  const int bi = i1 - i0, bj = j1 - j0;
  if (bi <= 0 || bj <= 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* As = (S*)smem_raw;      // [k][i], ld P   (K up to NB+1)
  S* Bs = As + P * P;        // [k][j], ld P
  S* Ws = Bs + P * P;        // W block, [i + j*P]
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int tr_ = tid % TG, tc = tid / TG;
  S acc[RM][RM];
#pragma unroll
  for (int a = 0; a < RM; a++)
#pragma unroll
    for (int b = 0; b < RM; b++) acc[a][b] = S(0);
  // rank-bk update acc += As[:, k] Bs[k, :]; entries past the block edge accumulate
  // garbage in accumulators that are never written back, so the tiles need no zero fill
  auto mm = [&](int bk) {
    for (int k = 0; k < bk; k++) {
      S a[RM], b[RM];
#pragma unroll
      for (int q = 0; q < RM; q++) {
        const int i = min(tr_ + TG * q, P - 1), j = min(tc + TG * q, P - 1);
        a[q] = As[k * P + i];
        b[q] = Bs[k * P + j];
      }
#pragma unroll
      for (int x = 0; x < RM; x++)
#pragma unroll
        for (int y = 0; y < RM; y++) acc[x][y] = fmac(a[x], b[y], acc[x][y]);
    }
  };

  // ---- updates from diagonal d-1 ----
  if (d >= 1 && !(dbg & 2) && !left) {
    // A-part: W -= TA[I, I*] Y[I*, J], with rank(I*) = d-1-cJ
    int ra = d - 1 - cJ;
    if (ra >= 0 && ra < rI) {
      int Is = nbi - 1 - ra;
      int k0 = rb[Is], k1 = rb[Is + 1], bk = k1 - k0;
      for (int e = tid; e < bi * bk; e += nt) {
        int i = e % bi, k = e / bi;
        As[k * P + i] = TA[(i0 + i) + (size_t)(k0 + k) * lda];
      }
      for (int e = tid; e < bk * bj; e += nt) {
        int k = e % bk, j = e / bk;
        Bs[k * P + j] = W[(k0 + k) + (size_t)(j0 + j) * ldw];
      }
      __syncthreads();
      mm(bk);
      __syncthreads();
    }
    // B-part: W -= Y[I, J*] TB[J*, J], with rank(J*) = d-1-rI
    int cr = d - 1 - rI;
    if (cr >= 0 && cr < cJ) {
      int Js = lowerB ? nbj - 1 - cr : cr;
      int k0 = cb[Js], k1 = cb[Js + 1], bk = k1 - k0;
      for (int e = tid; e < bi * bk; e += nt) {
        int i = e % bi, k = e / bi;
        As[k * P + i] = W[(i0 + i) + (size_t)(k0 + k) * ldw];
      }
      for (int e = tid; e < bk * bj; e += nt) {
        int k = e % bk, j = e / bk;
        Bs[k * P + j] = TB[(k0 + k) + (size_t)(j0 + j) * ldb];
      }
      __syncthreads();
      mm(bk);
      __syncthreads();
    }
  }
  // ---- write back the updated W (or stage it for the leaf solve) ----
  const bool solve = (dd == d) && !(dbg & 1);  // dbg: timing experiments only (MSY_TRSYL_DBG)
  {
#pragma unroll
    for (int x = 0; x < RM; x++) {
      int i = tr_ + TG * x;
      if (i >= bi) continue;
#pragma unroll
      for (int y = 0; y < RM; y++) {
        int j = tc + TG * y;
        if (j >= bj) continue;
        S v = W[(i0 + i) + (size_t)(j0 + j) * ldw] - acc[x][y];
        if (solve) Ws[i + j * P] = v;
        else W[(i0 + i) + (size_t)(j0 + j) * ldw] = v;
      }
    }
  }
  if (!solve) return;
  if constexpr (TrsylCfg<S>::LEAF == 3) {
    for (int e = tid; e < bi * bi; e += nt) {
      int i = e % bi, k = e / bi;
      As[i + k * P] = TA[(i0 + i) + (size_t)(i0 + k) * lda];
    }
    for (int e = tid; e < bj * bj; e += nt) {
      int i = e % bj, k = e / bj;
      Bs[i + k * P] = TB[(j0 + i) + (size_t)(j0 + k) * ldb];
    }
    __syncthreads();
    __shared__ int g_rof[NB + 2], g_rln[NB + 2], g_cof[NB + 2], g_cln[NB + 2], g_n[2];
    if (tid == 0) {  // row units from the bottom
      int cnt = 0, i = bi - 1;
      while (i >= 0) {
        const int st2 = (i > 0 && !iszero(As[i + (i - 1) * P])) ? i - 1 : i;
        g_rof[cnt] = st2; g_rln[cnt] = i - st2 + 1; cnt++;
        i = st2 - 1;
      }
      g_n[0] = cnt;
    } else if (tid == 32) {  // column units in solve order
      int cnt = 0;
      if (!lowerB) {
        int j = 0;
        while (j < bj) {
          const int len = (j + 1 < bj && !iszero(Bs[(j + 1) + j * P])) ? 2 : 1;
          g_cof[cnt] = j; g_cln[cnt] = len; cnt++;
          j += len;
        }
      } else {
        int j = bj - 1;
        while (j >= 0) {
          const int st2 = (j > 0 && !iszero(Bs[(j - 1) + j * P])) ? j - 1 : j;
          g_cof[cnt] = st2; g_cln[cnt] = j - st2 + 1; cnt++;
          j = st2 - 1;
        }
      }
      g_n[1] = cnt;
    }
    __syncthreads();
    if constexpr (kLeafGroups<S>) {  // (real types always run the left-looking schedule: uinv is set)
      // Lazy wavefront with GS = 4 threads per 1x1 / 2x2 unit: on step s every ready unit
      // (row unit a, column unit s - a) gathers its two dot products (T_A rows below it x
      // solved Y, solved Y left of it x T_B) split round-robin over its 4 threads, reduces
      // them with two xor-shuffles, and its first thread solves the unit.  One block
      // barrier per step; the dot products are ~4x shorter than with one thread per unit.
      constexpr int GS = 4;
      const int nru = g_n[0], ncu = g_n[1];
      const int slot = tid / GS, sub = tid % GS;
      // unit-pair inverses (16 entries per pair, pair a * ncu + b), all pairs in parallel;
      // a zero pivot is flagged by a NaN first entry
      S* minv = uinv + (size_t)blockIdx.x * TL_TILE * 16;
      for (int e = tid; e < nru * ncu; e += nt) {
        const int a = e / ncu, b = e % ncu;
        const int iu = g_rof[a], p = g_rln[a], ju = g_cof[b], q = g_cln[b];
        S* o = minv + (size_t)e * 16;
        bool ok;
        if (p == 1 && q == 1) {
          const S dd = As[iu + iu * P] + Bs[ju + ju * P];
          ok = !iszero(dd);
          o[0] = ok ? S(1) / dd : S(0);
        } else if (p == 2 && q == 1) ok = unit_inverse<S, 2, 1>(As, Bs, P, iu, ju, o);
        else if (p == 1 && q == 2) ok = unit_inverse<S, 1, 2>(As, Bs, P, iu, ju, o);
        else ok = unit_inverse<S, 2, 2>(As, Bs, P, iu, ju, o);
        if (!ok) o[0] = mk<S>(NAN, NAN);
      }
      __syncthreads();
      // The units' inverses are staged two steps ahead into a 3-slot shared-memory ring with
      // cp.async (the group of unit slot g copies the 16 entries of its unit of step s + 2), so
      // the L2 latency of the table never sits on a step's critical path.
      S* ring = Ws + (size_t)P * P;  // [3][64 slots][16]
      auto stage = [&](int s2) {
        const int a2 = max(0, s2 - ncu + 1) + slot;
        if (s2 < nru + ncu - 1 && a2 <= min(s2, nru - 1)) {
          const char* src = reinterpret_cast<const char*>(minv + (size_t)(a2 * ncu + (s2 - a2)) * 16);
          char* dst = reinterpret_cast<char*>(ring + ((size_t)(s2 % 3) * 64 + slot) * 16);
          constexpr int CH = 16 * (int)sizeof(S) / 16;  // 16-byte chunks per unit
          for (int c = sub; c < CH; c += GS) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(dst + 16 * c);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 16 * c) : "memory");
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      };
      stage(0);
      stage(1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      __syncthreads();
      for (int s = 0; s < nru + ncu - 1; s++) {
        const int a = max(0, s - ncu + 1) + slot;
        const bool act = a <= min(s, nru - 1) && slot < (TRS_TPB / GS);
        stage(s + 2);
        S v00 = S(0), v10 = S(0), v01 = S(0), v11 = S(0);
        int iu = 0, p = 1, ju = 0, q = 1;
        if (act) {
          const int bb = s - a;
          iu = g_rof[a]; p = g_rln[a]; ju = g_cof[bb]; q = g_cln[bb];
        }
        if (act) {
          const int kb = iu + p;
          const int la = lowerB ? ju + q : 0, lb = lowerB ? bj : ju;
          const int nr = bi - kb, nl = lb - la;
          if (p == 1 && q == 1) {
            S w0 = S(0), w1 = S(0);
            int t = sub;
            for (; t + GS < nr; t += 2 * GS) {
              w0 = fmac(As[iu + (size_t)(kb + t) * P], Ws[(kb + t) + (size_t)ju * P], w0);
              w1 = fmac(As[iu + (size_t)(kb + t + GS) * P], Ws[(kb + t + GS) + (size_t)ju * P], w1);
            }
            if (t < nr) w0 = fmac(As[iu + (size_t)(kb + t) * P], Ws[(kb + t) + (size_t)ju * P], w0);
            t = sub;
            for (; t + GS < nl; t += 2 * GS) {
              w0 = fmac(Ws[iu + (size_t)(la + t) * P], Bs[(la + t) + (size_t)ju * P], w0);
              w1 = fmac(Ws[iu + (size_t)(la + t + GS) * P], Bs[(la + t + GS) + (size_t)ju * P], w1);
            }
            if (t < nl) w0 = fmac(Ws[iu + (size_t)(la + t) * P], Bs[(la + t) + (size_t)ju * P], w0);
            v00 = w0 + w1;
          } else {
            const int di = p > 1 ? 1 : 0, dj = q > 1 ? (int)P : 0;  // duplicates are discarded
            // two independent accumulator sets, loads of both iterations issued together
            S u00 = S(0), u10 = S(0), u01 = S(0), u11 = S(0);
            int t = sub;
            for (; t + GS < nr; t += 2 * GS) {
              const S* X = As + iu + (size_t)(kb + t) * P;
              const S* Y = Ws + (kb + t) + (size_t)ju * P;
              const S* X2 = X + (size_t)GS * P;
              const S* Y2 = Y + GS;
              const S a0 = X[0], a1 = X[di], y0 = Y[0], y1 = Y[dj];
              const S b0 = X2[0], b1 = X2[di], z0 = Y2[0], z1 = Y2[dj];
              v00 = fmac(a0, y0, v00); v10 = fmac(a1, y0, v10); v01 = fmac(a0, y1, v01); v11 = fmac(a1, y1, v11);
              u00 = fmac(b0, z0, u00); u10 = fmac(b1, z0, u10); u01 = fmac(b0, z1, u01); u11 = fmac(b1, z1, u11);
            }
            if (t < nr) {
              const S* X = As + iu + (size_t)(kb + t) * P;
              const S* Y = Ws + (kb + t) + (size_t)ju * P;
              const S a0 = X[0], a1 = X[di], y0 = Y[0], y1 = Y[dj];
              v00 = fmac(a0, y0, v00); v10 = fmac(a1, y0, v10); v01 = fmac(a0, y1, v01); v11 = fmac(a1, y1, v11);
            }
            t = sub;
            for (; t + GS < nl; t += 2 * GS) {
              const S* X = Ws + iu + (size_t)(la + t) * P;
              const S* Y = Bs + (la + t) + (size_t)ju * P;
              const S* X2 = X + (size_t)GS * P;
              const S* Y2 = Y + GS;
              const S a0 = X[0], a1 = X[di], y0 = Y[0], y1 = Y[dj];
              const S b0 = X2[0], b1 = X2[di], z0 = Y2[0], z1 = Y2[dj];
              v00 = fmac(a0, y0, v00); v10 = fmac(a1, y0, v10); v01 = fmac(a0, y1, v01); v11 = fmac(a1, y1, v11);
              u00 = fmac(b0, z0, u00); u10 = fmac(b1, z0, u10); u01 = fmac(b0, z1, u01); u11 = fmac(b1, z1, u11);
            }
            if (t < nl) {
              const S* X = Ws + iu + (size_t)(la + t) * P;
              const S* Y = Bs + (la + t) + (size_t)ju * P;
              const S a0 = X[0], a1 = X[di], y0 = Y[0], y1 = Y[dj];
              v00 = fmac(a0, y0, v00); v10 = fmac(a1, y0, v10); v01 = fmac(a0, y1, v01); v11 = fmac(a1, y1, v11);
            }
            v00 = v00 + u00; v10 = v10 + u10; v01 = v01 + u01; v11 = v11 + u11;
          }
        }
#pragma unroll
        for (int o = 1; o < GS; o <<= 1) {
          v00 = v00 + __shfl_xor_sync(0xffffffffu, v00, o);
          v10 = v10 + __shfl_xor_sync(0xffffffffu, v10, o);
          v01 = v01 + __shfl_xor_sync(0xffffffffu, v01, o);
          v11 = v11 + __shfl_xor_sync(0xffffffffu, v11, o);
        }
        if (act) {  // 4-way mat-vec: thread `sub` produces entry sub of the unit
          const S* mi = ring + ((size_t)(s % 3) * 64 + slot) * 16;
          const bool ok = !isnan(re(mi[0]));
          const int ns = p * q;
          S mcur[4];
#pragma unroll
          for (int c = 0; c < 4; c++) mcur[c] = (sub < ns && c < ns) ? mi[sub * ns + c] : S(0);
          S r4[4];
          r4[0] = Ws[iu + ju * P] - v00;
          r4[1] = p == 2 ? Ws[(iu + 1) + ju * P] - v10 : S(0);
          r4[2] = q == 2 ? Ws[iu + (ju + 1) * P] - v01 : S(0);
          r4[3] = (p == 2 && q == 2) ? Ws[(iu + 1) + (ju + 1) * P] - v11 : S(0);
          if (p == 1 && q == 2) r4[1] = r4[2];  // unknowns ordered r + p c
          S y = S(0);
#pragma unroll
          for (int c = 0; c < 4; c++) y = fmac(mcur[c], r4[c], y);
          __syncwarp(0xFu << (lane & ~3));  // the group's reads of W precede its writes
          if (sub < ns) {
            const int r = sub % p, c = sub / p;
            Ws[(iu + r) + (ju + c) * P] = ok ? y : mk<S>(NAN, NAN);
          }
          if (!ok && sub == 0) {  // singular diagonal pair: report the first in reference order (decoded on the host)
            const int jg = j0 + ju, ig = i0 + iu + p - 1;
            const int crank = lowerB ? (n - 1 - jg) : jg;
            atomicMin(&status[0], crank * m + (m - 1 - ig));
          }
        }
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // step s + 1's inverses have landed
        __syncthreads();
      }
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else if (warp < 2) {  // two warps run the wavefront, synchronised by a 64-thread named barrier
      const int nru = g_n[0], ncu = g_n[1];
      for (int s = 0; s < nru + ncu - 1; s++) {
        for (int a = tid; a < nru; a += 64) {
          const int bb = s - a;
          if (bb < 0 || bb >= ncu) continue;
          const int iu = g_rof[a], p = g_rln[a], ju = g_cof[bb], q = g_cln[bb];
          const int kb = iu + p;                                        // rows below the unit
          const int la = lowerB ? ju + q : 0, lb = lowerB ? bj : ju;   // columns solved before it
          // one fused walk over both dot products: x stride P, y stride 1 in both pieces
          const int nr = bi - kb, tot = nr + (lb - la);
          const S* xa = As + iu + (size_t)kb * P;          // t <  nr: As[iu, kb + t]
          const S* xb = Ws + iu + (ptrdiff_t)(la - nr) * P;  // t >= nr: Ws[iu, la + t - nr]
          const S* ya = Ws + kb + (size_t)ju * P;          // t <  nr: Ws[kb + t, ju]
          const S* yb = Bs + (la - nr) + (size_t)ju * P;   // t >= nr: Bs[la + t - nr, ju]
          bool ok = true;
          if (p == 1 && q == 1) {
            S v0 = Ws[iu + ju * P], v1 = S(0), v2 = S(0), v3 = S(0);
            int t = 0;
            for (; t + 3 < tot; t += 4) {
#pragma unroll
              for (int u = 0; u < 4; u++) {
                const int tt = t + u;
                const S* X = tt < nr ? xa : xb;
                const S* Y = tt < nr ? ya : yb;
                const S prod = X[(size_t)tt * P] * Y[tt];
                if (u == 0) v0 = v0 - prod; else if (u == 1) v1 = v1 - prod; else if (u == 2) v2 = v2 - prod; else v3 = v3 - prod;
              }
            }
            for (; t < tot; t++) {
              const S* X = t < nr ? xa : xb;
              const S* Y = t < nr ? ya : yb;
              v0 = v0 - X[(size_t)t * P] * Y[t];
            }
            const S dd = As[iu + iu * P] + Bs[ju + ju * P];
            ok = !iszero(dd);
            Ws[iu + ju * P] = ok ? ((v0 + v1) + (v2 + v3)) * (S(1) / dd) : mk<S>(NAN, NAN);
          } else {
            S v00 = Ws[iu + ju * P];
            S v10 = p > 1 ? Ws[(iu + 1) + ju * P] : S(0);
            S v01 = q > 1 ? Ws[iu + (ju + 1) * P] : S(0);
            S v11 = (p > 1 && q > 1) ? Ws[(iu + 1) + (ju + 1) * P] : S(0);
            const int di = p > 1 ? 1 : 0, dj = q > 1 ? (int)P : 0;  // duplicates are discarded
            for (int t = 0; t < tot; t++) {
              const S* X = t < nr ? xa : xb;
              const S* Y = t < nr ? ya : yb;
              const size_t xo = (size_t)t * P;
              const S a0 = X[xo], a1 = X[xo + di], y0 = Y[t], y1 = Y[t + dj];
              v00 = v00 - a0 * y0; v10 = v10 - a1 * y0; v01 = v01 - a0 * y1; v11 = v11 - a1 * y1;
            }
            Ws[iu + ju * P] = v00;
            if (p > 1) Ws[(iu + 1) + ju * P] = v10;
            if (q > 1) Ws[iu + (ju + 1) * P] = v01;
            if (p > 1 && q > 1) Ws[(iu + 1) + (ju + 1) * P] = v11;
            if (p == 2 && q == 1) ok = unit_solve<S, 2, 1>(As, Bs, Ws, P, iu, ju);
            else if (p == 1 && q == 2) ok = unit_solve<S, 1, 2>(As, Bs, Ws, P, iu, ju);
            else ok = unit_solve<S, 2, 2>(As, Bs, Ws, P, iu, ju);
          }
          if (!ok) {  // singular diagonal pair: report the first in reference order (decoded on the host)
            const int jg = j0 + ju, ig = i0 + iu + p - 1;
            const int crank = lowerB ? (n - 1 - jg) : jg;
            atomicMin(&status[0], crank * m + (m - 1 - ig));
          }
        }
        asm volatile("bar.sync 1, 64;" ::: "memory");
      }
    }
    __syncthreads();
    for (int e = tid; e < bi * bj; e += nt) {
      int i = e % bi, j = e / bi;
      W[(i0 + i) + (size_t)(j0 + j) * ldw] = Ws[i + j * P];
    }
  } else if constexpr (TrsylCfg<S>::LEAF == 2) {
  // ---- leaf: TA_II Y + Y TB_JJ = W_IJ in shared memory ----
  // Two levels: the leaf is cut into sub-tiles of ~LST x LST (edges nudged so no 2x2
  // block is split); sub-tile anti-diagonals are processed in order.  On each, one
  // warp per sub-tile solves it with an element-level wavefront over its 1x1 / 2x2
  // units (warp-synchronous), then every pending sub-tile takes the contributions of
  // the sub-tiles just solved (small shared-memory GEMMs, one warp per sub-tile).
  for (int e = tid; e < bi * bi; e += nt) {
    int i = e % bi, k = e / bi;
    As[i + k * P] = TA[(i0 + i) + (size_t)(i0 + k) * lda];
  }
  for (int e = tid; e < bj * bj; e += nt) {
    int i = e % bj, k = e / bj;
    Bs[i + k * P] = TB[(j0 + i) + (size_t)(j0 + k) * ldb];
  }
  __syncthreads();
  constexpr int LST = 8, LSM = LST + 1, NSUB = (NB + 1 + LST - 1) / LST + 1;
  constexpr int NWARP = TRS_TPB / 32;
  __shared__ int sr[NSUB + 1], sc[NSUB + 1], s_nsr, s_nsc;
  if (tid == 0) {  // sub-tile edges: rows in index order, columns in solve order
    int c = 0, b0 = 0;
    while (b0 < bi) {
      int e1 = min(b0 + LST, bi);
      if (e1 < bi && !iszero(As[e1 + (e1 - 1) * P])) e1++;
      sr[c++] = b0;
      b0 = e1;
    }
    sr[c] = bi;
    s_nsr = c;
    c = 0; b0 = 0;
    while (b0 < bj) {
      int e1 = min(b0 + LST, bj);
      if (e1 < bj && !iszero(lowerB ? Bs[(e1 - 1) + e1 * P] : Bs[e1 + (e1 - 1) * P])) e1++;
      sc[c++] = b0;
      b0 = e1;
    }
    sc[c] = bj;
    s_nsc = c;
  }
  __syncthreads();
  const int nsr = s_nsr, nsc = s_nsc;
  // sub-tile of row rank a (from the bottom) / column rank b (solve order)
  auto rows_of = [&](int a, int& r0, int& r1) { const int I = nsr - 1 - a; r0 = sr[I]; r1 = sr[I + 1]; };
  auto cols_of = [&](int bb, int& c0, int& c1) { const int J = lowerB ? nsc - 1 - bb : bb; c0 = sc[J]; c1 = sc[J + 1]; };
  // unit tables of the whole leaf, built once: row units ranked from the bottom, column
  // units in solve order; a sub-tile's units are a contiguous rank range (edges never
  // split a 2x2 block)
  __shared__ int g_rrk[NB + 2], g_rof[NB + 2], g_rln[NB + 2], g_crk[NB + 2], g_cof[NB + 2], g_cln[NB + 2];
  if (tid == 0) {
    int cnt = 0, i = bi - 1;
    while (i >= 0) {
      const int st2 = (i > 0 && !iszero(As[i + (i - 1) * P])) ? i - 1 : i;
      for (int q = st2; q <= i; q++) g_rrk[q] = cnt;
      g_rof[cnt] = st2; g_rln[cnt] = i - st2 + 1; cnt++;
      i = st2 - 1;
    }
  } else if (tid == 32) {
    int cnt = 0;
    if (!lowerB) {
      int j = 0;
      while (j < bj) {
        const int len = (j + 1 < bj && !iszero(Bs[(j + 1) + j * P])) ? 2 : 1;
        for (int q = j; q < j + len; q++) g_crk[q] = cnt;
        g_cof[cnt] = j; g_cln[cnt] = len; cnt++;
        j += len;
      }
    } else {
      int j = bj - 1;
      while (j >= 0) {
        const int st2 = (j > 0 && !iszero(Bs[(j - 1) + j * P])) ? j - 1 : j;
        for (int q = st2; q <= j; q++) g_crk[q] = cnt;
        g_cof[cnt] = st2; g_cln[cnt] = j - st2 + 1; cnt++;
        j = st2 - 1;
      }
    }
  }
  __syncthreads();
  for (int s = 0; s < nsr + nsc - 1; s++) {
    // ---- solve the sub-tiles on anti-diagonal s (one warp each) ----
    const int alo = max(0, s - (nsc - 1)), ahi = min(s, nsr - 1);
    for (int a = alo + warp; a <= ahi; a += NWARP) {
      const int bb = s - a;
      int r0, r1, c0, c1;
      rows_of(a, r0, r1);
      cols_of(bb, c0, c1);
      const int ri = r1 - r0, cj = c1 - c0;
      const int rbase = g_rrk[r1 - 1], cbase = lowerB ? g_crk[c1 - 1] : g_crk[c0];
      const int* rof = g_rof + rbase; const int* rln = g_rln + rbase;
      const int* cof = g_cof + cbase; const int* cln = g_cln + cbase;
      const int nru = g_rrk[r0] - rbase + 1, ncu = (lowerB ? g_crk[c0] : g_crk[c1 - 1]) - cbase + 1;
      constexpr int EPL = (LSM * LSM + 31) / 32;
      int ei[EPL], ej[EPL], era[EPL], ecr[EPL];
#pragma unroll
      for (int k = 0; k < EPL; k++) {
        const int e = lane + 32 * k;
        if (e < ri * cj) {
          ei[k] = r0 + e % ri; ej[k] = c0 + e / ri;
          era[k] = g_rrk[ei[k]] - rbase; ecr[k] = g_crk[ej[k]] - cbase;
        } else {
          ei[k] = 0; ej[k] = 0; era[k] = -1000000; ecr[k] = -1000000;
        }
      }
      for (int t = 0; t < nru + ncu - 1; t++) {
        if (lane < nru) {  // lane a solves unit (a, t - a)
          const int ua = lane, ub = t - lane;
          if (ub >= 0 && ub < ncu) {
            const int i = rof[ua], p = rln[ua], jst = cof[ub], q = cln[ub];
            bool ok = true;
            if (p == 1 && q == 1) {
              const S dd = As[i + i * P] + Bs[jst + jst * P];
              ok = !iszero(dd);
              Ws[i + jst * P] = ok ? Ws[i + jst * P] / dd : mk<S>(NAN, NAN);
            } else if (p == 2 && q == 1) {
              ok = unit_solve<S, 2, 1>(As, Bs, Ws, P, i, jst);
            } else if (p == 1 && q == 2) {
              ok = unit_solve<S, 1, 2>(As, Bs, Ws, P, i, jst);
            } else {
              ok = unit_solve<S, 2, 2>(As, Bs, Ws, P, i, jst);
            }
            if (!ok) {  // singular diagonal pair: report the first in reference order (decoded on the host)
              const int jg = j0 + jst, ig = i0 + i + p - 1;
              const int crank = lowerB ? (n - 1 - jg) : jg;
              atomicMin(&status[0], crank * m + (m - 1 - ig));
            }
          }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < EPL; k++) {
          const int ra = era[k], cr = ecr[k];
          if (ra + cr > t) {
            const int i = ei[k], j = ej[k];
            S v = Ws[i + j * P];
            const int rs = t - cr;
            if (rs >= 0 && rs < ra) {
              const int st2 = rof[rs];
              v = v - As[i + st2 * P] * Ws[st2 + j * P];
              if (rln[rs] == 2) v = v - As[i + (st2 + 1) * P] * Ws[(st2 + 1) + j * P];
            }
            const int cs = t - ra;
            if (cs >= 0 && cs < cr) {
              const int st2 = cof[cs];
              v = v - Ws[i + st2 * P] * Bs[st2 + j * P];
              if (cln[cs] == 2) v = v - Ws[i + (st2 + 1) * P] * Bs[(st2 + 1) + j * P];
            }
            Ws[i + j * P] = v;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- pending sub-tiles take the contributions of diagonal s ----
    for (int it = warp; it < nsr * nsc; it += NWARP) {
      const int a = it % nsr, bb = it / nsr;
      if (a + bb <= s) continue;
      const int as = s - bb, bs = s - a;  // solved tile in my column (below) / in my row (before)
      const bool pa = as >= 0 && as < a, pb = bs >= 0 && bs < bb;
      if (!pa && !pb) continue;
      int r0, r1, c0, c1;
      rows_of(a, r0, r1);
      cols_of(bb, c0, c1);
      const int ri = r1 - r0, cj = c1 - c0;
      int k0 = 0, k1 = 0, l0 = 0, l1 = 0;
      if (pa) rows_of(as, k0, k1);
      if (pb) cols_of(bs, l0, l1);
      for (int e = lane; e < ri * cj; e += 32) {
        const int i = r0 + e % ri, j = c0 + e / ri;
        S v = Ws[i + j * P];
        for (int k = k0; k < k1; k++) v = v - As[i + k * P] * Ws[k + j * P];
        for (int l = l0; l < l1; l++) v = v - Ws[i + l * P] * Bs[l + j * P];
        Ws[i + j * P] = v;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < bi * bj; e += nt) {
    int i = e % bi, j = e / bi;
    W[(i0 + i) + (size_t)(j0 + j) * ldw] = Ws[i + j * P];
  }
  } else {
  // ---- leaf: TA_II Y + Y TB_JJ = W_IJ in shared memory ----
  // element-level anti-diagonal wavefront over 1x1 / 2x2 units: sub-step s solves the
  // units (a, b) with a + b = s (a = row-unit rank from the bottom, b = column-unit
  // rank in solve order), then every pending entry subtracts the contributions of
  // the units just solved.  Entry ownership and unit ranks are precomputed, so a
  // sub-step costs a few shared-memory FMAs per owned entry plus two barriers.
  for (int e = tid; e < bi * bi; e += nt) {
    int i = e % bi, k = e / bi;
    As[i + k * P] = TA[(i0 + i) + (size_t)(i0 + k) * lda];
  }
  for (int e = tid; e < bj * bj; e += nt) {
    int i = e % bj, k = e / bj;
    Bs[i + k * P] = TB[(j0 + i) + (size_t)(j0 + k) * ldb];
  }
  __syncthreads();
  __shared__ int ru_rank[NB + 2], cu_rank[NB + 2];
  __shared__ int ru_of[NB + 2], cu_of[NB + 2];  // rank -> first row / column of the unit
  __shared__ int nru, ncu;
  __shared__ int ru_len[NB + 2], cu_len[NB + 2];
  if (tid == 0) {
    // row units from the bottom (rank 0 = bottom unit); 2x2 if As[i][i-1] != 0
    int cnt = 0, i = bi - 1;
    while (i >= 0) {
      int st = (i > 0 && !iszero(As[i + (i - 1) * P])) ? i - 1 : i;
      for (int q = st; q <= i; q++) ru_rank[q] = cnt;
      ru_of[cnt] = st;
      ru_len[cnt] = i - st + 1;
      cnt++;
      i = st - 1;
    }
    nru = cnt;
    // column units in solve order (upper: left->right; lower: right->left)
    cnt = 0;
    if (!lowerB) {
      int j = 0;
      while (j < bj) {
        int len = (j + 1 < bj && !iszero(Bs[(j + 1) + j * P])) ? 2 : 1;
        for (int q = j; q < j + len; q++) cu_rank[q] = cnt;
        cu_of[cnt] = j;
        cu_len[cnt] = len;
        cnt++;
        j += len;
      }
    } else {
      int j = bj - 1;
      while (j >= 0) {
        int st = (j > 0 && !iszero(Bs[(j - 1) + j * P])) ? j - 1 : j;
        for (int q = st; q <= j; q++) cu_rank[q] = cnt;
        cu_of[cnt] = st;
        cu_len[cnt] = j - st + 1;
        cnt++;
        j = st - 1;
      }
    }
    ncu = cnt;
  }
  __syncthreads();
  constexpr int EPT = ((NB + 1) * (NB + 1) + TRS_TPB - 1) / TRS_TPB;  // entries per thread
  int ei[EPT], ej[EPT], era[EPT], ecr[EPT];
#pragma unroll
  for (int k = 0; k < EPT; k++) {
    const int e = tid + k * nt;
    if (e < bi * bj) {
      ei[k] = e % bi; ej[k] = e / bi;
      era[k] = ru_rank[ei[k]]; ecr[k] = cu_rank[ej[k]];
    } else {
      ei[k] = 0; ej[k] = 0; era[k] = -1000000; ecr[k] = -1000000;  // never pending
    }
  }
  const int nsteps = nru + ncu - 1;
  for (int s = 0; s < nsteps; s++) {
    // phase 1: thread a solves unit (a, s - a)
    if (tid < nru) {
      const int a = tid, bb = s - a;
      if (bb >= 0 && bb < ncu) {
        const int i = ru_of[a], p = ru_len[a], jst = cu_of[bb], q = cu_len[bb];
        bool ok = true;
        if (p == 1 && q == 1) {
          const S d = As[i + i * P] + Bs[jst + jst * P];
          ok = !iszero(d);
          Ws[i + jst * P] = ok ? Ws[i + jst * P] / d : mk<S>(NAN, NAN);
        } else if (p == 2 && q == 1) {
          ok = unit_solve<S, 2, 1>(As, Bs, Ws, P, i, jst);
        } else if (p == 1 && q == 2) {
          ok = unit_solve<S, 1, 2>(As, Bs, Ws, P, i, jst);
        } else {
          ok = unit_solve<S, 2, 2>(As, Bs, Ws, P, i, jst);
        }
        if (!ok) {  // singular diagonal pair: report the first in reference order (decoded on the host)
          const int jg = j0 + jst, ig = i0 + i + p - 1;
          const int crank = lowerB ? (n - 1 - jg) : jg;
          atomicMin(&status[0], crank * m + (m - 1 - ig));
        }
      }
    }
    __syncthreads();
    // phase 2: owned pending entries take the contributions of the units just solved
#pragma unroll
    for (int k = 0; k < EPT; k++) {
      const int ra = era[k], cr = ecr[k];
      if (ra + cr > s) {
        const int i = ei[k], j = ej[k];
        S v = Ws[i + j * P];
        const int rs = s - cr;  // solved unit in my column unit (below me if rs < ra)
        if (rs >= 0 && rs < ra) {
          const int st = ru_of[rs];
          v = v - As[i + st * P] * Ws[st + j * P];
          if (ru_len[rs] == 2) v = v - As[i + (st + 1) * P] * Ws[(st + 1) + j * P];
        }
        const int cs = s - ra;  // solved unit in my row unit (before me if cs < cr)
        if (cs >= 0 && cs < cr) {
          const int st = cu_of[cs];
          v = v - Ws[i + st * P] * Bs[st + j * P];
          if (cu_len[cs] == 2) v = v - Ws[i + (st + 1) * P] * Bs[(st + 1) + j * P];
        }
        Ws[i + j * P] = v;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < bi * bj; e += nt) {
    int i = e % bi, j = e / bi;
    W[(i0 + i) + (size_t)(j0 + j) * ldw] = Ws[i + j * P];
  }
  }
}

template <class S>
static size_t trsyl_smem() {
  constexpr int P = 4 * ((TrsylCfg<S>::NB + 1 + 3) / 4);
  // + the 3 x 64 x 16 ring of staged unit inverses (grouped leaf, real types)
  return (size_t)3 * P * P * sizeof(S) + (kLeafGroups<S> ? (size_t)3 * 64 * 16 * sizeof(S) : 0);
}

// side stream + events of the left-looking schedule (per host thread, like the sweep contexts)
struct TrsylSide {
  cudaStream_t side = nullptr;
  cudaEvent_t evLeaf = nullptr, evOld = nullptr;
  int dev = -1;
};
inline TrsylSide& trsyl_side() {
  thread_local TrsylSide t;
  int d = 0;
  cudaGetDevice(&d);
  if (t.side == nullptr || t.dev != d) {
    cudaStreamCreateWithFlags(&t.side, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&t.evLeaf, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&t.evOld, cudaEventDisableTiming);
    t.dev = d;
  }
  return t;
}

// left-looking schedule for the real types (fp32 Y0, fp64 corrections); complex keeps the
// eager wavefront
template <class S> constexpr bool kTrsylLeft = std::is_same<S, float>::value || std::is_same<S, double>::value;

template <class S>
struct TrsylWs {
  int* rb;
  int* cb;
  S* part;    // left-looking split-K partials: [leaf][chunk][64 x 64]
  S* uinv;    // per-leaf unit-pair inverses: [leaf][pair][16]
  int maxch;  // chunks per leaf (upper bound)
  static void carve(Arena& ar, int m, int n, TrsylWs& w) {
    w.rb = ar.get<int>(m / 1 + 2);
    w.cb = ar.get<int>(n / 1 + 2);
    w.part = nullptr;
    w.uinv = nullptr;
    w.maxch = 0;
    if constexpr (kTrsylLeft<S>) {
      const int nbi = cdiv(m, TL_SPACING), nbj = cdiv(n, TL_SPACING);
      w.maxch = cdiv(m, TL_KC) + cdiv(n, TL_KC) + 4;  // + the two new chunks and two range tails
      w.part = ar.get<S>((size_t)2 * std::min(nbi, nbj) * w.maxch * TL_TILE);  // x2: diagonal parity
      w.uinv = ar.get<S>((size_t)std::min(nbi, nbj) * TL_TILE * 16);
    }
  }
};

// Solve in place; status (device, 4 ints) must be initialised by the caller with
// trsyl_status_init (several solves may share one status word).
template <class S>
int trsyl(int m, int n, const S* TA, int lda, const S* TB, int ldb, int lowerB, S* W, int ldw, TrsylWs<S>& w,
          int* status, cudaStream_t st) {
  constexpr int NB = TrsylCfg<S>::NB;
  MSY_SMEM_ATTR_ONCE(trsyl_step_kernel<S>, (int)trsyl_smem<S>());
  constexpr int dbg = 0;  // trsyl_step_kernel's timing-experiment bits (MSY_TRSYL_DBG was removed)
  if constexpr (kTrsylLeft<S>) {
    if (w.part != nullptr) {
      const int nbi = cdiv(m, TL_SPACING), nbj = cdiv(n, TL_SPACING);
      trsyl_partition_kernel<S><<<cdiv(max(nbi, nbj) + 1, 128), 128, 0, st>>>(m, TA, lda, n, TB, ldb, lowerB,
                                                                              TL_SPACING, w.rb, nbi, w.cb, nbj);
      MSY_LAUNCH_CK();
      // Per diagonal d on `st`: the leaves' two "new" chunks (K <= 128 each), the fixed-order
      // reduction into W, the leaf solves.  The older chunks of diagonal d + 1 run on the side
      // stream during diagonal d (they read tiles solved by d - 1 at the latest).  Partials are
      // double-buffered by diagonal parity.
      TrsylSide& sd = trsyl_side();
      const size_t half = (size_t)std::min(nbi, nbj) * w.maxch * TL_TILE;
      auto leaves = [&](int d) { return std::min(d, nbi - 1) - std::max(0, d - nbj + 1) + 1; };
      auto launch_part = [&](int d, int coff, int ny, cudaStream_t s2) -> int {
        const int nl = leaves(d);
        if (nl <= 0 || ny <= 0) return 0;
        S* part = w.part + (d & 1) * half;
        KScope ks(KC_TRSYL, 2.0 * TL_SPACING * TL_SPACING * TL_SPACING * (coff == 0 ? 2.0 : (d - 1.0)) * nl, s2);
        if constexpr (std::is_same<S, double>::value)
          trsyl_lpart_dmma_kernel<<<dim3(nl, ny), 128, 0, s2>>>(m, n, TA, lda, TB, ldb, lowerB, W, ldw, w.rb, w.cb,
                                                               nbi, nbj, d, w.maxch, coff, part);
        else
          trsyl_lpart_simt_kernel<S><<<dim3(nl, ny), 256, 0, s2>>>(m, n, TA, lda, TB, ldb, lowerB, W, ldw, w.rb,
                                                                   w.cb, nbi, nbj, d, w.maxch, coff, part);
        MSY_LAUNCH_CK();
        return 0;
      };
      // older chunks of diagonal d: K <= (d - 1) * 64 in TL_KC pieces (+2 for the two ranges' tails)
      auto old_chunks = [&](int d) { return d >= 2 ? std::min(w.maxch - 2, cdiv((d - 1) * TL_LD, TL_KC) + 2) : 0; };
      MSY_CK(cudaEventRecord(sd.evLeaf, st));  // "leaf(-1)": the partition is done
      for (int d = 0; d < nbi + nbj - 1; d++) {
        const int nleaf = leaves(d);
        if (nleaf <= 0) continue;
        if (d > 0) MSY_CK(cudaStreamWaitEvent(st, sd.evOld, 0));   // old chunks of d (issued last iteration)
        // side: old chunks of d + 1 after leaf(d - 1) (recorded at the end of the last iteration)
        cudaStream_t side = sd.side;
        MSY_CK(cudaStreamWaitEvent(side, sd.evLeaf, 0));
        int rc = launch_part(d + 1, 2, d + 1 < nbi + nbj - 1 ? old_chunks(d + 1) : 0, side);
        if (rc) return rc;
        MSY_CK(cudaEventRecord(sd.evOld, side));
        if (d > 0) {
          if (d == 1) {  // diagonal 1 has no older chunks; its new ones
            rc = launch_part(d, 0, 2, st);
          } else {
            rc = launch_part(d, 0, 2, st);
          }
          if (rc) return rc;
          KScope ks(KC_TRSYL, 0, st);
          trsyl_lreduce_kernel<S><<<dim3(nleaf, TL_TILE / 256), 256, 0, st>>>(m, n, lowerB, W, ldw, w.rb, w.cb, nbi,
                                                                              nbj, d, w.maxch,
                                                                              w.part + (d & 1) * half);
          MSY_LAUNCH_CK();
        }
        {
          KScope ks(KC_TRSYL, 0, st);
          trsyl_step_kernel<S><<<(unsigned)nleaf, TRS_TPB, trsyl_smem<S>(), st>>>(
              m, n, TA, lda, TB, ldb, lowerB, W, ldw, w.rb, w.cb, nbi, nbj, d, status, 0, 1, w.uinv);
          MSY_LAUNCH_CK();
        }
        MSY_CK(cudaEventRecord(sd.evLeaf, st));
      }
      MSY_CK(cudaStreamWaitEvent(st, sd.evOld, 0));  // join the side stream
      return 0;
    }
  }
  const int nbi = cdiv(m, NB), nbj = cdiv(n, NB);
  trsyl_partition_kernel<S><<<cdiv(max(nbi, nbj) + 1, 128), 128, 0, st>>>(m, TA, lda, n, TB, ldb, lowerB, NB, w.rb,
                                                                          nbi, w.cb, nbj);
  MSY_LAUNCH_CK();
  for (int d = 0; d < nbi + nbj - 1; d++) {
    // blocks changed at step d (see trsyl_step_kernel)
    long cnt = 0;
    if (d == 0) cnt = 1;
    else {
      for (int r = 0; r < std::min(d, nbi); r++) cnt += std::max(0, nbj - std::max(0, d - r));
      cnt += (long)std::min(d, nbj) * std::max(0, nbi - d);
    }
    if (cnt == 0) continue;
    KScope ks(KC_TRSYL, 0, st);
    trsyl_step_kernel<S><<<(unsigned)cnt, TRS_TPB, trsyl_smem<S>(), st>>>(m, n, TA, lda, TB, ldb, lowerB, W, ldw, w.rb, w.cb,
                                                                      nbi, nbj, d, status, dbg);
    MSY_LAUNCH_CK();
  }
  return 0;
}

}  // namespace msy
