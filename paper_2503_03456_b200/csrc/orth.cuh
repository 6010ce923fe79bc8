// orth.cuh -- high-precision re-orthonormalisation of the low-precision Schur vectors.
//
// Replaces the reference's modified Gram-Schmidt `mgs_qr` (pkg/src/mpsylv/linalg.py:252-273,
// positive real diagonal `_fix_r_diagonal` :228-241, rank test `_check_rank` :244-249).
// B200 design: Cholesky-QR in fp64, all level-3: G = U^H U (GEMM), G = R^H R
// (blocked Cholesky: one-CTA diagonal factor + TRSM + GEMM update), Q = U R^{-1}
// (blocked right TRSM: GEMM + one-CTA-per-row-slab triangular solve).  Because U
// is orthonormal to u_l (kappa(U) = 1 + O(1e-7)), one Cholesky-QR pass is
// orthonormal to O(u_64); R has a positive real diagonal by construction, the
// factorisation the paper's Alg. 3 footnote asks for.
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace msy {

// diagonal block edge (64; 32 for complex double to stay under 48 KB static smem)
template <class S> struct ChNb { static constexpr int v = sizeof(S) > 8 ? 32 : 64; };

// Cholesky (upper, G = R^H R) of an nb x nb diagonal block, in place; bad pivot -> flag
template <class S>
__global__ void __launch_bounds__(256) potrf_small_kernel(int nb, S* G, int ldg, int* flag, double* diag_min) {
  typedef typename tr<S>::R R;
  __shared__ S A[ChNb<S>::v][ChNb<S>::v + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) A[e % nb][e / nb] = G[(e % nb) + (size_t)(e / nb) * ldg];
  __syncthreads();
  for (int j = 0; j < nb; j++) {
    R d = re(A[j][j]);
    __syncthreads();
    if (!(d > R(0))) {
      if (tid == 0) *flag = 1;
      d = R(1);
    }
    R r = sqrt(d);
    for (int c = j + 1 + tid; c < nb; c += blockDim.x) A[j][c] = A[j][c] / mk<S>(r);
    __syncthreads();
    if (tid == 0) {
      A[j][j] = mk<S>(r);
      atomicMin((unsigned long long*)diag_min, (unsigned long long)__double_as_longlong((double)r));
    }
    // trailing: A[c1][c2] -= conj(A[j][c1]) A[j][c2], c2 >= c1 > j
    const int t = nb - j - 1;
    for (int e = tid; e < t * t; e += blockDim.x) {
      int c1 = j + 1 + e % t, c2 = j + 1 + e / t;
      if (c2 >= c1) A[c1][c2] = A[c1][c2] - conj(A[j][c1]) * A[j][c2];
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    int i = e % nb, c = e / nb;
    G[i + (size_t)c * ldg] = (i <= c) ? A[i][c] : S(0);
  }
}

// Solve R^H X = B in place (R nb x nb upper => R^H lower), B is nb x ncols.  One thread per
// column; the substitution is fully unrolled over the compile-time block edge so the column
// stays in registers, and the pivots are applied as precomputed reciprocals.
template <class S>
__global__ void __launch_bounds__(128) trsm_lhu_kernel(int nb, const S* Rk, int ldr, int ncols, S* B, int ldb) {
  constexpr int NB = ChNb<S>::v;
  __shared__ S Rs[NB][NB + 1];
  __shared__ S rinv[NB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Rs[e % nb][e / nb] = Rk[(e % nb) + (size_t)(e / nb) * ldr];
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) rinv[i] = S(1) / conj(Rs[i][i]);
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  S x[NB];
#pragma unroll
  for (int i = 0; i < NB; i++) x[i] = i < nb ? B[i + (size_t)c * ldb] : S(0);
#pragma unroll
  for (int i = 0; i < NB; i++) {
    if (i < nb) {
      S s = x[i];
#pragma unroll
      for (int q = 0; q < i; q++) s = s - conj(Rs[q][i]) * x[q];
      x[i] = s * rinv[i];
    }
  }
#pragma unroll
  for (int i = 0; i < NB; i++)
    if (i < nb) B[i + (size_t)c * ldb] = x[i];
}

// Solve X R = B in place (R nb x nb upper), B is nrows x nb (one thread per row, unrolled)
template <class S>
__global__ void __launch_bounds__(128) trsm_rup_kernel(int nb, const S* Rk, int ldr, int nrows, S* B, int ldb) {
  constexpr int NB = ChNb<S>::v;
  __shared__ S Rs[NB][NB + 1];
  __shared__ S rinv[NB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Rs[e % nb][e / nb] = Rk[(e % nb) + (size_t)(e / nb) * ldr];
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) rinv[i] = S(1) / Rs[i][i];
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  S x[NB];
#pragma unroll
  for (int j = 0; j < NB; j++) x[j] = j < nb ? B[r + (size_t)j * ldb] : S(0);
#pragma unroll
  for (int j = 0; j < NB; j++) {
    if (j < nb) {
      S s = x[j];
#pragma unroll
      for (int q = 0; q < j; q++) s = s - x[q] * Rs[q][j];
      x[j] = s * rinv[j];
    }
  }
#pragma unroll
  for (int j = 0; j < NB; j++)
    if (j < nb) B[r + (size_t)j * ldb] = x[j];
}

template <class S>
__global__ void clear_lower_kernel(int m, S* G, int ldg) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < m && i > j) G[i + (size_t)j * ldg] = S(0);
}

// Q = U R^{-1} with U^H U = R^H R.  G is an m x m scratch (holds R on return).
// dinfo: device scratch (int flag + double diag_min).
template <class S>
int orth_cholqr(int m, const S* U, int ldu, S* Q, int ldq, S* G, int ldg, int* dflag, double* ddiag, cudaStream_t st) {
  int rc = gemm<S>('C', 'N', m, m, m, S(1), U, ldu, U, ldu, S(0), G, ldg, st);
  if (rc) return rc;
  for (int k = 0; k < m; k += ChNb<S>::v) {
    int nb = std::min(ChNb<S>::v, m - k);
    S* Gkk = G + k + (size_t)k * ldg;
    potrf_small_kernel<S><<<1, 256, 0, st>>>(nb, Gkk, ldg, dflag, ddiag);
    MSY_LAUNCH_CK();
    int rest = m - k - nb;
    if (rest > 0) {
      S* Gkr = G + k + (size_t)(k + nb) * ldg;
      trsm_lhu_kernel<S><<<cdiv(rest, 128), 128, 0, st>>>(nb, Gkk, ldg, rest, Gkr, ldg);
      MSY_LAUNCH_CK();
      rc = gemm<S>('C', 'N', rest, rest, nb, S(-1), Gkr, ldg, Gkr, ldg, S(1), G + (k + nb) + (size_t)(k + nb) * ldg, ldg,
                   st);
      if (rc) return rc;
    }
  }
  // Q = U R^{-1}, column blocks left to right
  for (int k = 0; k < m; k += ChNb<S>::v) {
    int nb = std::min(ChNb<S>::v, m - k);
    S* Qk = Q + (size_t)k * ldq;
    cudaMemcpy2DAsync(Qk, (size_t)ldq * sizeof(S), U + (size_t)k * ldu, (size_t)ldu * sizeof(S), (size_t)m * sizeof(S),
                      nb, cudaMemcpyDeviceToDevice, st);
    if (k > 0) {
      rc = gemm<S>('N', 'N', m, nb, k, S(-1), Q, ldq, G + (size_t)k * ldg, ldg, S(1), Qk, ldq, st);
      if (rc) return rc;
    }
    trsm_rup_kernel<S><<<cdiv(m, 128), 128, 0, st>>>(nb, G + k + (size_t)k * ldg, ldg, m, Qk, ldq);
    MSY_LAUNCH_CK();
  }
  // the trailing GEMM updates also wrote the strictly lower part: clear it so G holds R
  clear_lower_kernel<S><<<dim3(cdiv(m, 256), m), 256, 0, st>>>(m, G, ldg);
  MSY_LAUNCH_CK();
  return 0;
}

}  // namespace msy
