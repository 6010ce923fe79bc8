// gemm.cuh -- C = alpha*op(A)*op(B) + beta*C for float/double/complex.
//
// Replaces the reference's ascending-k rank-1 `gemm` (pkg/src/mpsylv/linalg.py:125-154)
// on every u_h / u_l contraction of the path.  Two engines:
//   * gemm_simt<S>   register-blocked SIMT FFMA/DFMA kernel (all four scalar types),
//                    double-buffered smem tiles, 256 threads;
//   * gemm_dmma      fp64 tensor-pipe kernel (mma.sync m8n8k4 f64 -> DMMA.8x8x4 on
//                    sm_100a) used for the real fp64 GEMM phases (see gemm_dmma.cuh).
// op codes: 'N' (as stored), 'T' (transpose), 'C' (conjugate transpose).
#pragma once
#include "common.cuh"
#include "gemm_dmma.cuh"

namespace msy {

template <class S> struct GemmCfg;
template <> struct GemmCfg<float> { static constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8; };
template <> struct GemmCfg<double> { static constexpr int BM = 64, BN = 64, BK = 8, TM = 4, TN = 4; };
template <> struct GemmCfg<cfloat> { static constexpr int BM = 64, BN = 64, BK = 8, TM = 4, TN = 4; };
template <> struct GemmCfg<cdouble> { static constexpr int BM = 32, BN = 32, BK = 8, TM = 2, TN = 2; };

template <class S, char OP>
__device__ __forceinline__ S opval(S v) {
  if (OP == 'C') return conj(v);
  return v;
}

// op(A) is M x K.  OPA == 'N': A is M x K col-major; else A is K x M.
// Split-K: blockIdx.z handles K-range [z*kchunk, (z+1)*kchunk); with `part` != null the
// unscaled partial product goes to part + z*M*N (ld M) instead of C.
template <class S, char OPA, char OPB>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int M, int N, int K, S alpha, const S* __restrict__ A, int lda,
                                                        const S* __restrict__ B, int ldb, S beta, S* C, int ldc,
                                                        int kchunk, S* part) {
  typedef GemmCfg<S> G;
  constexpr int BM = G::BM, BN = G::BN, BK = G::BK, TM = G::TM, TN = G::TN;
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int LA = BM * BK / NT, LB = BN * BK / NT;  // elements per thread per tile
  __shared__ S As[2][BK][BM + 1];
  __shared__ S Bs[2][BK][BN + 1];
  const int tid = threadIdx.x;
  const int bm = blockIdx.x * BM, bn = blockIdx.y * BN;
  const int tx = tid % (BM / TM), ty = tid / (BM / TM);
  S acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) acc[i][j] = S(0);
  S ra[LA], rb[LB];
  const int kbeg = blockIdx.z * kchunk, kend = min(K, kbeg + kchunk);

  auto loadA = [&](int k0) {
#pragma unroll
    for (int e = 0; e < LA; e++) {
      int idx = tid + e * NT;
      int i, k;
      if (OPA == 'N') { i = idx % BM; k = idx / BM; } else { k = idx % BK; i = idx / BK; }
      int gi = bm + i, gk = k0 + k;
      S v = S(0);
      if (gi < M && gk < kend) v = (OPA == 'N') ? A[gi + (size_t)gk * lda] : opval<S, OPA>(A[gk + (size_t)gi * lda]);
      ra[e] = v;
    }
  };
  auto loadB = [&](int k0) {
#pragma unroll
    for (int e = 0; e < LB; e++) {
      int idx = tid + e * NT;
      int j, k;
      if (OPB == 'N') { k = idx % BK; j = idx / BK; } else { j = idx % BN; k = idx / BN; }
      int gj = bn + j, gk = k0 + k;
      S v = S(0);
      if (gj < N && gk < kend) v = (OPB == 'N') ? B[gk + (size_t)gj * ldb] : opval<S, OPB>(B[gj + (size_t)gk * ldb]);
      rb[e] = v;
    }
  };
  auto storeAB = [&](int buf) {
#pragma unroll
    for (int e = 0; e < LA; e++) {
      int idx = tid + e * NT;
      int i, k;
      if (OPA == 'N') { i = idx % BM; k = idx / BM; } else { k = idx % BK; i = idx / BK; }
      As[buf][k][i] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < LB; e++) {
      int idx = tid + e * NT;
      int j, k;
      if (OPB == 'N') { k = idx % BK; j = idx / BK; } else { j = idx % BN; k = idx / BN; }
      Bs[buf][k][j] = rb[e];
    }
  };

  int nk = (kend - kbeg + BK - 1) / BK;
  if (nk > 0) {
    loadA(kbeg);
    loadB(kbeg);
    storeAB(0);
  }
  __syncthreads();
  for (int t = 0; t < nk; t++) {
    int cur = t & 1;
    if (t + 1 < nk) {
      loadA(kbeg + (t + 1) * BK);
      loadB(kbeg + (t + 1) * BK);
    }
#pragma unroll
    for (int k = 0; k < BK; k++) {
      S a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i++) a[i] = As[cur][k][tx + i * (BM / TM)];
#pragma unroll
      for (int j = 0; j < TN; j++) b[j] = Bs[cur][k][ty + j * (BN / TN)];
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) acc[i][j] = fmac(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < nk) storeAB(cur ^ 1);
    __syncthreads();
  }
  const bool b0 = iszero(beta);
#pragma unroll
  for (int i = 0; i < TM; i++) {
    int gi = bm + tx + i * (BM / TM);
    if (gi >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; j++) {
      int gj = bn + ty + j * (BN / TN);
      if (gj >= N) continue;
      if (part) {
        part[(size_t)blockIdx.z * M * N + gi + (size_t)gj * M] = acc[i][j];
        continue;
      }
      S* c = &C[gi + (size_t)gj * ldc];
      S v = alpha * acc[i][j];
      if (!b0) v = fmac(beta, *c, v);
      *c = v;
    }
  }
}

template <class S> __host__ __device__ inline S scal_mul(S a, S b) { return a * b; }

template <class S, char OPA, char OPB>
static int gemm_simt_launch(int M, int N, int K, S alpha, const S* A, int lda, const S* B, int ldb, S beta, S* C,
                            int ldc, cudaStream_t st) {
  typedef GemmCfg<S> G;
  dim3 grid(cdiv(M, G::BM), cdiv(N, G::BN));
  KScope ks(KC_SIMT, (tr<S>::cx ? 8.0 : 2.0) * M * N * K, st);
  gemm_simt_kernel<S, OPA, OPB><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, K, nullptr);
  MSY_LAUNCH_CK();
  return 0;
}

// C = alpha * sum_z part[z] + beta * C (fixed order: deterministic)
template <class S>
__global__ void splitk_reduce_kernel(int M, int N, int splits, const S* part, S alpha, S beta, S* C, int ldc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= M) return;
  S s = S(0);
  for (int z = 0; z < splits; z++) s += part[(size_t)z * M * N + i + (size_t)j * M];
  S* c = &C[i + (size_t)j * ldc];
  S v = alpha * s;
  if (!iszero(beta)) v = fmac(beta, *c, v);
  *c = v;
}

template <class S, char OPA, char OPB>
static int gemm_splitk_launch(int M, int N, int K, S alpha, const S* A, int lda, const S* B, int ldb, S beta, S* C,
                              int ldc, S* ws, int splits, cudaStream_t st) {
  typedef GemmCfg<S> G;
  const int kchunk = cdiv(cdiv(K, splits), G::BK) * G::BK;
  splits = cdiv(K, kchunk);
  dim3 grid(cdiv(M, G::BM), cdiv(N, G::BN), splits);
  KScope ks(KC_SIMT, (tr<S>::cx ? 8.0 : 2.0) * M * N * K, st);
  gemm_simt_kernel<S, OPA, OPB><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, ws);
  MSY_LAUNCH_CK();
  splitk_reduce_kernel<S><<<dim3(cdiv(M, 128), N), 128, 0, st>>>(M, N, splits, ws, alpha, beta, C, ldc);
  MSY_LAUNCH_CK();
  return 0;
}

// Skinny GEMMs (few output tiles, long K): split K over blockIdx.z into `ws`
// (splits * M * N elements) and reduce in a fixed order.
template <class S>
int gemm_splitk(char opa, char opb, int M, int N, int K, S alpha, const S* A, int lda, const S* B, int ldb, S beta,
                S* C, int ldc, S* ws, int splits, cudaStream_t st) {
  if (!tr<S>::cx) {
    if (opa == 'C') opa = 'T';
    if (opb == 'C') opb = 'T';
  }
#define MSY_G(a, b) \
  if (opa == a && opb == b) return gemm_splitk_launch<S, a, b>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, splits, st);
  MSY_G('N', 'N') MSY_G('N', 'T') MSY_G('T', 'N') MSY_G('T', 'T')
  if (tr<S>::cx) { MSY_G('C', 'N') MSY_G('N', 'C') MSY_G('C', 'C') MSY_G('C', 'T') MSY_G('T', 'C') }
#undef MSY_G
  return -2;
}

// scale C by beta (used when K == 0)
template <class S>
__global__ void scale_kernel(int M, int N, S beta, S* C, int ldc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < M) C[i + (size_t)j * ldc] = iszero(beta) ? S(0) : beta * C[i + (size_t)j * ldc];
}

// Generic dispatcher.
template <class S>
int gemm(char opa, char opb, int M, int N, int K, S alpha, const S* A, int lda, const S* B, int ldb, S beta, S* C,
         int ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0) {
    scale_kernel<S><<<dim3(cdiv(M, 256), N), 256, 0, st>>>(M, N, beta, C, ldc);
    MSY_LAUNCH_CK();
    return 0;
  }
  int h = gemm_dmma_try<S>(opa, opb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  if (h <= 0) return h;
  if (!tr<S>::cx) {
    if (opa == 'C') opa = 'T';
    if (opb == 'C') opb = 'T';
  }
#define MSY_G(a, b) \
  if (opa == a && opb == b) return gemm_simt_launch<S, a, b>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  MSY_G('N', 'N') MSY_G('N', 'T') MSY_G('T', 'N') MSY_G('T', 'T')
  if (tr<S>::cx) { MSY_G('C', 'N') MSY_G('N', 'C') MSY_G('C', 'C') MSY_G('C', 'T') MSY_G('T', 'C') }
#undef MSY_G
  return -2;
}

}  // namespace msy
