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

// Skinny projection  P_z (Q x N) = V[rows_z, :]^T C[rows_z, :]  (Q <= 32 columns of V, real fp32):
// the W1 = V^T A products of the Hessenberg panels and the Q0 accumulation read the trailing
// matrix once.  One CTA = 64 columns of C x a slice of VT_RS rows; the rows are walked in chunks
// of 32 staged in shared memory (C chunk 32 x 64, V chunk 32 x Q); thread (q = tid % 32,
// column group tid / 32) accumulates out[q, 8 g .. 8 g + 7].  Partials per row slice go to
// `part` and are reduced in slice order by splitk_reduce_kernel (deterministic).
constexpr int VT_RS = 512, VT_BN = 64, VT_CH = 32;
__global__ void __launch_bounds__(256) vtc_partial_kernel(int Krows, int N, int Q, const float* __restrict__ V, int ldv,
                                                          const float* __restrict__ C, int ldc,
                                                          float* __restrict__ part) {
  __shared__ float Cs[VT_CH][VT_BN + 1];
  __shared__ float Vs[VT_CH][33];
  const int tid = threadIdx.x, q = tid & 31, g = tid >> 5;
  const int bn = blockIdx.x * VT_BN, r0 = blockIdx.y * VT_RS, r1 = min(Krows, r0 + VT_RS);
  float acc[8];
#pragma unroll
  for (int c = 0; c < 8; c++) acc[c] = 0.f;
  for (int rc = r0; rc < r1; rc += VT_CH) {
    // stage: C rows rc..rc+31 x 64 columns (coalesced down the rows), V rows x Q
#pragma unroll
    for (int e = tid; e < VT_CH * VT_BN; e += 256) {
      const int i = e % VT_CH, j = e / VT_CH;
      Cs[i][j] = (rc + i < r1 && bn + j < N) ? C[(rc + i) + (size_t)(bn + j) * ldc] : 0.f;
    }
#pragma unroll
    for (int e = tid; e < VT_CH * 32; e += 256) {
      const int i = e % VT_CH, qq = e / VT_CH;
      Vs[i][qq] = (rc + i < r1 && qq < Q) ? V[(rc + i) + (size_t)qq * ldv] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int i = 0; i < VT_CH; i++) {
      const float v = Vs[i][q];
#pragma unroll
      for (int c = 0; c < 8; c++) acc[c] = fmaf(v, Cs[i][8 * g + c], acc[c]);
    }
    __syncthreads();
  }
  if (q < Q) {
    float* out = part + (size_t)blockIdx.y * Q * N;
#pragma unroll
    for (int c = 0; c < 8; c++)
      if (bn + 8 * g + c < N) out[q + (size_t)(bn + 8 * g + c) * Q] = acc[c];
  }
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
  if constexpr (std::is_same<S, float>::value) {
    // skinny V^T C (M <= 32 rows of output): the row-slice projection kernel; its slices must
    // fit the caller's split-K workspace (splits * M * N)
    const int nsl = cdiv(K, VT_RS);
    if (opa == 'T' && opb == 'N' && M <= 32 && nsl <= splits && K > 0) {
      KScope ks(KC_SIMT, 2.0 * M * N * K, st);
      vtc_partial_kernel<<<dim3(cdiv(N, VT_BN), nsl), 256, 0, st>>>(K, N, M, A, lda, B, ldb, ws);
      MSY_LAUNCH_CK();
      splitk_reduce_kernel<S><<<dim3(cdiv(M, 128), N), 128, 0, st>>>(M, N, nsl, ws, alpha, beta, C, ldc);
      MSY_LAUNCH_CK();
      return 0;
    }
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

// ---------------------------------------------------------------------------
// Rank-k update  C (M x N) += alpha * A (M x K) op(B),  K <= RK_KMAX, real fp32.
// The Hessenberg trailing updates and the Q0 accumulation are rank-32 updates of a large C:
// memory-bound (8 flop per C byte), so the kernel reads and writes each C element exactly once
// with warp-coalesced accesses, stages the whole A panel (128 x K) and B panel (K x 64) in
// shared memory once per tile, and keeps 4 x 8 outputs per thread (rows tr + 32 r, columns
// 8 tc + c; the 8 B columns come as two float4 broadcasts).  C is prefetched into registers
// before the K loop so its load latency overlaps the FMAs.
constexpr int RK_BM = 128, RK_BN = 64, RK_KMAX = 64;
template <char OPB>
__global__ void __launch_bounds__(256, 2) rankk_update_kernel(int M, int N, int K, float alpha, const float* __restrict__ A,
                                                           int lda, const float* __restrict__ B, int ldb, float* C,
                                                           int ldc) {
  __shared__ __align__(16) float As[RK_KMAX][RK_BM];
  __shared__ __align__(16) float Bs[RK_KMAX][RK_BN];
  const int tid = threadIdx.x, tr = tid & 31, tc = tid >> 5;
  const int bm = blockIdx.x * RK_BM, bn = blockIdx.y * RK_BN;
  // prefetch C
  float c[4][8];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int i = bm + tr + 32 * r, j = bn + 8 * tc + q;
      c[r][q] = (i < M && j < N) ? C[i + (size_t)j * ldc] : 0.f;
    }
  for (int e = tid; e < RK_BM * K; e += 256) {
    const int i = e % RK_BM, k = e / RK_BM;
    As[k][i] = bm + i < M ? A[(bm + i) + (size_t)k * lda] : 0.f;
  }
  for (int e = tid; e < RK_BN * K; e += 256) {
    int k, j;
    if (OPB == 'N') { k = e % K; j = e / K; } else { j = e % RK_BN; k = e / RK_BN; }
    float v = 0.f;
    if (bn + j < N) v = OPB == 'N' ? B[k + (size_t)(bn + j) * ldb] : B[(bn + j) + (size_t)k * ldb];
    Bs[k][j] = v;
  }
  __syncthreads();
  float acc[4][8];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 8; q++) acc[r][q] = 0.f;
  for (int k = 0; k < K; k++) {
    float a[4];
#pragma unroll
    for (int r = 0; r < 4; r++) a[r] = As[k][tr + 32 * r];
    const float4 b0 = *reinterpret_cast<const float4*>(&Bs[k][8 * tc]);
    const float4 b1 = *reinterpret_cast<const float4*>(&Bs[k][8 * tc + 4]);
    const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int q = 0; q < 8; q++) acc[r][q] = fmaf(a[r], b[q], acc[r][q]);
  }
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int i = bm + tr + 32 * r, j = bn + 8 * tc + q;
      if (i < M && j < N) C[i + (size_t)j * ldc] = fmaf(alpha, acc[r][q], c[r][q]);
    }
}

// C += alpha A op(B) for real fp32 with K <= RK_KMAX through rankk_update_kernel; 1 = not handled
template <class S>
int rankk_try(char, int, int, int, S, const S*, int, const S*, int, S*, int, cudaStream_t) {
  return 1;
}
template <>
inline int rankk_try<float>(char opb, int M, int N, int K, float alpha, const float* A, int lda, const float* B,
                            int ldb, float* C, int ldc, cudaStream_t st) {
  if (K <= 0 || K > RK_KMAX || M <= 0 || N <= 0) return 1;
  if (opb == 'C') opb = 'T';
  dim3 grid(cdiv(M, RK_BM), cdiv(N, RK_BN));
  KScope ks(KC_SIMT, 2.0 * M * N * K, st);
  if (opb == 'N') rankk_update_kernel<'N'><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, C, ldc);
  else rankk_update_kernel<'T'><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, C, ldc);
  MSY_LAUNCH_CK();
  return 0;
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
  if (opa == 'N' && beta == S(1) && K <= RK_KMAX && (size_t)M * N >= (size_t)1 << 16) {  // rank-k updates
    h = rankk_try<S>(opb, M, N, K, alpha, A, lda, B, ldb, C, ldc, st);
    if (h <= 0) return h;
  }
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
