// lu.cuh -- fp64 LU with partial pivoting and the four lu_solve modes (mp_inv path).
//
// Replaces the reference's `lu` (pkg/src/mpsylv/linalg.py:349-369: argmax pivot,
// first occurrence; exact zero pivot -> SingularMatrixError) and `lu_solve`
// (linalg.py:416-440: left/right x no/conj, right solves through the conjugate
// transpose, linalg.py:425-429).  Blocked right-looking factorisation:
//   one-CTA panel (pivot search by block reduction, swaps, rank-1 updates)
//   -> row swaps on the rest (lu_swap_kernel) -> unit-lower TRSM -> trailing GEMM.
// Triangular solves with many right-hand sides are blocked the same way
// (one-thread-per-column substitution on a diagonal block + GEMM updates).
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "util.cuh"
#include "orth.cuh"

namespace msy {

constexpr int LU_NB = 32;


template <class S>
struct LuWs {
  int* ipiv;  // m
  int* flag;  // singular flag
  static void carve(Arena& ar, int m, LuWs& w) {
    w.ipiv = ar.get<int>(m + 1);
    w.flag = ar.get<int>(8);
  }
};

template <class S>
__global__ void __launch_bounds__(1024) lu_panel_kernel(int m, S* A, int lda, int k, int nb, int* ipiv, int* flag) {
  typedef typename tr<S>::R R;
  __shared__ R bv[32];
  __shared__ int bi[32];
  __shared__ int s_p;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int j = 0; j < nb; j++) {
    const int c = k + j;
    // argmax |A[r, c]|, r >= c, first occurrence on ties
    R best = -1;
    int bidx = m;
    for (int r = c + tid; r < m; r += nt) {
      R a = absv(A[r + (size_t)c * lda]);
      if (a > best) { best = a; bidx = r; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      R ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    if (lane == 0) { bv[wid] = best; bi[wid] = bidx; }
    __syncthreads();
    if (tid == 0) {
      R b = bv[0];
      int p = bi[0];
      for (int q = 1; q < nw; q++)
        if (bv[q] > b || (bv[q] == b && bi[q] < p)) { b = bv[q]; p = bi[q]; }
      if (p >= m) p = c;
      if (iszero(A[p + (size_t)c * lda])) { *flag = 1; }
      ipiv[c] = p;
      s_p = p;
    }
    __syncthreads();
    const int p = s_p;
    if (p != c)
      for (int q = k + tid; q < k + nb; q += nt) {
        S t = A[c + (size_t)q * lda];
        A[c + (size_t)q * lda] = A[p + (size_t)q * lda];
        A[p + (size_t)q * lda] = t;
      }
    __syncthreads();
    S piv = A[c + (size_t)c * lda];
    bool ok = !iszero(piv);
    for (int r = c + 1 + tid; r < m; r += nt) {
      S l = ok ? A[r + (size_t)c * lda] / piv : S(0);
      A[r + (size_t)c * lda] = l;
      for (int q = c + 1; q < k + nb; q++) A[r + (size_t)q * lda] = A[r + (size_t)q * lda] - l * A[c + (size_t)q * lda];
    }
    __syncthreads();
  }
}

// apply the swaps ipiv[k..k+nb) to columns outside [k, k+nb)
template <class S>
__global__ void lu_swap_kernel(int m, int ncols, S* A, int lda, int k, int nb, const int* ipiv) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ncols || (q >= k && q < k + nb)) return;
  S* col = A + (size_t)q * lda;
  for (int j = k; j < k + nb; j++) {
    int p = ipiv[j];
    if (p != j) { S t = col[j]; col[j] = col[p]; col[p] = t; }
  }
}

// B (rows x nrhs) row permutation by ipiv[0..n) forward (inverse = reverse order)
template <class S>
__global__ void perm_rows_kernel(int n, int nrhs, S* B, int ldb, const int* ipiv, int inverse) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrhs) return;
  S* col = B + (size_t)q * ldb;
  for (int t = 0; t < n; t++) {
    int j = inverse ? n - 1 - t : t;
    int p = ipiv[j];
    if (p != j) { S x = col[j]; col[j] = col[p]; col[p] = x; }
  }
}

// op(T) X = B on an nb x nb diagonal block, one thread per column of B.
// lower: T lower (or, with cj, T^H where the stored block is upper); unit: skip diagonal.
template <class S>
__global__ void __launch_bounds__(128) trsm_block_kernel(int nb, const S* T, int ldt, int lower_eff, int cj, int unit,
                                                         int nrhs, S* B, int ldb) {
  __shared__ S Ts[ChNb<S>::v][ChNb<S>::v + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    // effective operator entry E[i][j] = cj ? conj(T[j][i]) : T[i][j]
    Ts[i][j] = cj ? conj(T[j + (size_t)i * ldt]) : T[i + (size_t)j * ldt];
  }
  __syncthreads();
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrhs) return;
  S x[ChNb<S>::v];
  for (int i = 0; i < nb; i++) x[i] = B[i + (size_t)q * ldb];
  if (lower_eff) {
    for (int i = 0; i < nb; i++) {
      S s = x[i];
      for (int j = 0; j < i; j++) s = s - Ts[i][j] * x[j];
      x[i] = unit ? s : s / Ts[i][i];
    }
  } else {
    for (int i = nb - 1; i >= 0; i--) {
      S s = x[i];
      for (int j = i + 1; j < nb; j++) s = s - Ts[i][j] * x[j];
      x[i] = unit ? s : s / Ts[i][i];
    }
  }
  for (int i = 0; i < nb; i++) B[i + (size_t)q * ldb] = x[i];
}

// Blocked op(T) X = B in place.  T n x n; lower_eff tells whether op(T) is lower.
template <class S>
int trsm_left(int n, const S* T, int ldt, int lower_eff, int cj, int unit, int nrhs, S* B, int ldb, cudaStream_t st) {
  const int nblk = cdiv(n, ChNb<S>::v);
  for (int t = 0; t < nblk; t++) {
    int b = lower_eff ? t : nblk - 1 - t;
    int k = b * ChNb<S>::v, nb = std::min(ChNb<S>::v, n - k);
    const S* Tkk = T + k + (size_t)k * ldt;
    trsm_block_kernel<S><<<cdiv(nrhs, 128), 128, 0, st>>>(nb, Tkk, ldt, lower_eff, cj, unit, nrhs, B + k, ldb);
    MSY_LAUNCH_CK();
    int rc = 0;
    if (lower_eff && k + nb < n) {
      // B[k+nb:n] -= E[k+nb:n, kb] X[kb], E = T or T^H
      if (!cj) rc = gemm<S>('N', 'N', n - k - nb, nrhs, nb, S(-1), T + (k + nb) + (size_t)k * ldt, ldt, B + k, ldb, S(1),
                            B + k + nb, ldb, st);
      else rc = gemm<S>('C', 'N', n - k - nb, nrhs, nb, S(-1), T + k + (size_t)(k + nb) * ldt, ldt, B + k, ldb, S(1),
                        B + k + nb, ldb, st);
    } else if (!lower_eff && k > 0) {
      if (!cj) rc = gemm<S>('N', 'N', k, nrhs, nb, S(-1), T + (size_t)k * ldt, ldt, B + k, ldb, S(1), B, ldb, st);
      else rc = gemm<S>('C', 'N', k, nrhs, nb, S(-1), T + k, ldt, B + k, ldb, S(1), B, ldb, st);
    }
    if (rc) return rc;
  }
  return 0;
}

// In place LU (PA = LU) of an m x m matrix.
template <class S>
int lu_factor(int m, S* A, int lda, LuWs<S>& w, cudaStream_t st) {
  MSY_CK(cudaMemsetAsync(w.flag, 0, sizeof(int), st));
  for (int k = 0; k < m; k += LU_NB) {
    int nb = std::min(LU_NB, m - k);
    lu_panel_kernel<S><<<1, 1024, 0, st>>>(m, A, lda, k, nb, w.ipiv, w.flag);
    MSY_LAUNCH_CK();
    lu_swap_kernel<S><<<cdiv(m, 128), 128, 0, st>>>(m, m, A, lda, k, nb, w.ipiv);
    MSY_LAUNCH_CK();
    int rest = m - k - nb;
    if (rest > 0) {
      S* Akr = A + k + (size_t)(k + nb) * lda;
      int rc = trsm_left<S>(nb, A + k + (size_t)k * lda, lda, 1, 0, 1, rest, Akr, lda, st);
      if (rc) return rc;
      rc = gemm<S>('N', 'N', rest, rest, nb, S(-1), A + (k + nb) + (size_t)k * lda, lda, Akr, lda, S(1),
                   A + (k + nb) + (size_t)(k + nb) * lda, lda, st);
      if (rc) return rc;
    }
  }
  return 0;
}

template <class S>
int lu_read_status(LuWs<S>& w, int* singular, cudaStream_t st) {
  MSY_CK(d2h(singular, w.flag, sizeof(int), st));
  MSY_CK(host_sync(st));
  return 0;
}

// lu_solve(F, B, side, transpose) in place on B.
//   left:  B is n x nrhs;  right: B is nrhs x n (nrhs rows), solved via B^H.
// tmp: scratch of n * nrhs elements (right side only).
template <class S>
int lu_solve(int n, const S* LU, int ldlu, LuWs<S>& w, int right, int cj, int nrhs, S* B, int ldb, S* tmp,
             cudaStream_t st) {
  if (right) {
    // X A = B <=> A^H X^H = B^H ; X A^H = B <=> A X^H = B^H
    int rc = conj_transpose<S>(nrhs, n, B, ldb, tmp, n, st);
    if (rc) return rc;
    rc = lu_solve<S>(n, LU, ldlu, w, 0, !cj, nrhs, tmp, n, nullptr, st);
    if (rc) return rc;
    return conj_transpose<S>(n, nrhs, tmp, n, B, ldb, st);
  }
  if (!cj) {
    perm_rows_kernel<S><<<cdiv(nrhs, 128), 128, 0, st>>>(n, nrhs, B, ldb, w.ipiv, 0);
    MSY_LAUNCH_CK();
    int rc = trsm_left<S>(n, LU, ldlu, 1, 0, 1, nrhs, B, ldb, st);  // L (unit lower)
    if (rc) return rc;
    return trsm_left<S>(n, LU, ldlu, 0, 0, 0, nrhs, B, ldb, st);     // U
  }
  int rc = trsm_left<S>(n, LU, ldlu, 1, 1, 0, nrhs, B, ldb, st);    // U^H (lower)
  if (rc) return rc;
  rc = trsm_left<S>(n, LU, ldlu, 0, 1, 1, nrhs, B, ldb, st);        // L^H (unit upper)
  if (rc) return rc;
  perm_rows_kernel<S><<<cdiv(nrhs, 128), 128, 0, st>>>(n, nrhs, B, ldb, w.ipiv, 1);
  MSY_LAUNCH_CK();
  return 0;
}

}  // namespace msy
