// gemm_dmma.cuh -- fp64 GEMM on the FP64 tensor pipe (mma.sync m8n8k4 .f64 -> DMMA.8x8x4).
//
// sm_100a has no tcgen05 kind::f64, so the fp64 tensor path is the warp-level
// DMMA.  Block tile 64 x 64 x 16, 4 warps (2 x 2), warp tile
// 32 x 32 = 4 x 4 DMMA tiles, 32 fp64 accumulators per thread; double-buffered
// shared-memory tiles staged through registers; smem leading dimension 68 doubles
// makes the fragment loads bank-conflict free (a half-warp touches 16 distinct
// 8-byte bank pairs).  Used for every real fp64 contraction of the path
// (transforms, residuals, recovery, Cholesky-QR, LU updates).
#pragma once
#include "common.cuh"

namespace msy {

constexpr int DM_BM = 64, DM_BN = 64, DM_BK = 16, DM_LD = 68;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <char OPA, char OPB>
__global__ void __launch_bounds__(128) gemm_dmma_kernel(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                        int lda, const double* __restrict__ B, int ldb, double beta,
                                                        double* C, int ldc) {
  __shared__ __align__(16) double As[2][DM_BK][DM_LD];
  __shared__ __align__(16) double Bs[2][DM_BK][DM_LD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bm = blockIdx.x * DM_BM, bn = blockIdx.y * DM_BN;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[8], rb[8];
  // element e of the 64x16 A tile / 16x64 B tile handled by this thread
  auto loadA = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      int idx = tid + e * 128;
      int i, k;
      if (OPA == 'N') { i = idx & 63; k = idx >> 6; } else { k = idx & 15; i = idx >> 4; }
      int gi = bm + i, gk = k0 + k;
      ra[e] = (gi < M && gk < K) ? (OPA == 'N' ? A[gi + (size_t)gk * lda] : A[gk + (size_t)gi * lda]) : 0.0;
    }
  };
  auto loadB = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      int idx = tid + e * 128;
      int j, k;
      if (OPB == 'N') { k = idx & 15; j = idx >> 4; } else { j = idx & 63; k = idx >> 6; }
      int gj = bn + j, gk = k0 + k;
      rb[e] = (gj < N && gk < K) ? (OPB == 'N' ? B[gk + (size_t)gj * ldb] : B[gj + (size_t)gk * ldb]) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      int idx = tid + e * 128;
      int i, k;
      if (OPA == 'N') { i = idx & 63; k = idx >> 6; } else { k = idx & 15; i = idx >> 4; }
      As[buf][k][i] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < 8; e++) {
      int idx = tid + e * 128;
      int j, k;
      if (OPB == 'N') { k = idx & 15; j = idx >> 4; } else { j = idx & 63; k = idx >> 6; }
      Bs[buf][k][j] = rb[e];
    }
  };
  const int nk = (K + DM_BK - 1) / DM_BK;
  loadA(0);
  loadB(0);
  store(0);
  __syncthreads();
  const int fr = lane >> 2, fc = lane & 3;
  for (int t = 0; t < nk; t++) {
    const int cur = t & 1;
    if (t + 1 < nk) {
      loadA((t + 1) * DM_BK);
      loadB((t + 1) * DM_BK);
    }
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
  const bool b0 = beta == 0.0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int gi = bm + wm + i * 8 + fr;
    if (gi >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        int gj = bn + wn + j * 8 + fc * 2 + h;
        if (gj >= N) continue;
        double* c = &C[gi + (size_t)gj * ldc];
        double v = alpha * acc[i][j][h];
        if (!b0) v = fma(beta, *c, v);
        *c = v;
      }
    }
  }
}

// complex128: C = alpha op(A) op(B) + beta C on DMMA as two real accumulations per output
// (Re += Ar Br + (-Ai) Bi, Im += Ar Bi + Ai Br -- the 4M product, same rounding class as a
// complex fma loop).  64 x 64 x 8 block tile, re/im planes split in shared memory at staging
// time; op 'C' conjugates while staging.  Replaces the 32x32 SIMT tiles complex128 used before
// (C3's high-precision phase).
constexpr int ZM_BK = 8;

template <char OPA, char OPB>
__global__ void __launch_bounds__(128) gemm_zdmma_kernel(int M, int N, int K, cdouble alpha,
                                                         const cdouble* __restrict__ A, int lda,
                                                         const cdouble* __restrict__ B, int ldb, cdouble beta,
                                                         cdouble* C, int ldc) {
  __shared__ __align__(16) double Ar[2][ZM_BK][DM_LD], Ai[2][ZM_BK][DM_LD];
  __shared__ __align__(16) double Br[2][ZM_BK][DM_LD], Bi[2][ZM_BK][DM_LD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bm = blockIdx.x * DM_BM, bn = blockIdx.y * DM_BN;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double accR[4][4][2], accI[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) accR[i][j][0] = accR[i][j][1] = accI[i][j][0] = accI[i][j][1] = 0.0;
  double2 ra[4], rb[4];
  // element e of the 64x8 A tile / 8x64 B tile handled by this thread
  auto idxA = [&](int e, int& i, int& k) {
    int idx = tid + e * 128;
    if (OPA == 'N') { i = idx & 63; k = idx >> 6; } else { k = idx & 7; i = idx >> 3; }
  };
  auto idxB = [&](int e, int& j, int& k) {
    int idx = tid + e * 128;
    if (OPB == 'N') { k = idx & 7; j = idx >> 3; } else { j = idx & 63; k = idx >> 6; }
  };
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 4; e++) {
      int i, k;
      idxA(e, i, k);
      int gi = bm + i, gk = k0 + k;
      double2 v = make_double2(0.0, 0.0);
      if (gi < M && gk < K) {
        const cdouble* p = OPA == 'N' ? &A[gi + (size_t)gk * lda] : &A[gk + (size_t)gi * lda];
        v = *reinterpret_cast<const double2*>(p);
        if (OPA == 'C') v.y = -v.y;
      }
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
      int j, k;
      idxB(e, j, k);
      int gj = bn + j, gk = k0 + k;
      double2 v = make_double2(0.0, 0.0);
      if (gj < N && gk < K) {
        const cdouble* p = OPB == 'N' ? &B[gk + (size_t)gj * ldb] : &B[gj + (size_t)gk * ldb];
        v = *reinterpret_cast<const double2*>(p);
        if (OPB == 'C') v.y = -v.y;
      }
      rb[e] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 4; e++) {
      int i, k;
      idxA(e, i, k);
      Ar[buf][k][i] = ra[e].x;
      Ai[buf][k][i] = ra[e].y;
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
      int j, k;
      idxB(e, j, k);
      Br[buf][k][j] = rb[e].x;
      Bi[buf][k][j] = rb[e].y;
    }
  };
  const int nk = (K + ZM_BK - 1) / ZM_BK;
  load(0);
  store(0);
  __syncthreads();
  const int fr = lane >> 2, fc = lane & 3;
  for (int t = 0; t < nk; t++) {
    const int cur = t & 1;
    if (t + 1 < nk) load((t + 1) * ZM_BK);
#pragma unroll
    for (int kk = 0; kk < ZM_BK; kk += 4) {
      double ar[4], ai[4], an[4], br[4], bi[4];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        ar[i] = Ar[cur][kk + fc][wm + i * 8 + fr];
        ai[i] = Ai[cur][kk + fc][wm + i * 8 + fr];
        an[i] = -ai[i];
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        br[j] = Br[cur][kk + fc][wn + j * 8 + fr];
        bi[j] = Bi[cur][kk + fc][wn + j * 8 + fr];
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          dmma884(accR[i][j][0], accR[i][j][1], ar[i], br[j]);
          dmma884(accI[i][j][0], accI[i][j][1], ar[i], bi[j]);
          dmma884(accR[i][j][0], accR[i][j][1], an[i], bi[j]);
          dmma884(accI[i][j][0], accI[i][j][1], ai[i], br[j]);
        }
    }
    if (t + 1 < nk) store(cur ^ 1);
    __syncthreads();
  }
  const bool b0 = beta.x == 0.0 && beta.y == 0.0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int gi = bm + wm + i * 8 + fr;
    if (gi >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        int gj = bn + wn + j * 8 + fc * 2 + h;
        if (gj >= N) continue;
        double2* c = reinterpret_cast<double2*>(&C[gi + (size_t)gj * ldc]);
        const double xr = accR[i][j][h], xi = accI[i][j][h];
        double2 v = make_double2(fma(alpha.x, xr, -alpha.y * xi), fma(alpha.x, xi, alpha.y * xr));
        if (!b0) {
          const double2 o = *c;
          v.x = fma(beta.x, o.x, fma(-beta.y, o.y, v.x));
          v.y = fma(beta.x, o.y, fma(beta.y, o.x, v.y));
        }
        *c = v;
      }
    }
  }
}

template <class S>
int gemm_dmma_try(char, char, int, int, int, S, const S*, int, const S*, int, S, S*, int, cudaStream_t) {
  return 1;  // not handled: SIMT path
}

template <>
inline int gemm_dmma_try<double>(char opa, char opb, int M, int N, int K, double alpha, const double* A, int lda,
                                 const double* B, int ldb, double beta, double* C, int ldc, cudaStream_t st) {
  if (opa == 'C') opa = 'T';
  if (opb == 'C') opb = 'T';
  dim3 grid(cdiv(M, DM_BM), cdiv(N, DM_BN));
#define MSY_D(a, b)                                                                                      \
  if (opa == a && opb == b) {                                                                            \
    KScope ks__(KC_DMMA, 2.0 * M * N * K, st);                                                           \
    gemm_dmma_kernel<a, b><<<grid, 128, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);          \
    MSY_LAUNCH_CK();                                                                                     \
    return 0;                                                                                            \
  }
  MSY_D('N', 'N') MSY_D('N', 'T') MSY_D('T', 'N') MSY_D('T', 'T')
#undef MSY_D
  return 1;
}

template <>
inline int gemm_dmma_try<cdouble>(char opa, char opb, int M, int N, int K, cdouble alpha, const cdouble* A, int lda,
                                  const cdouble* B, int ldb, cdouble beta, cdouble* C, int ldc, cudaStream_t st) {
  if ((((uintptr_t)A | (uintptr_t)B | (uintptr_t)C) & 15) != 0) return 1;  // 16-byte loads need aligned bases
  dim3 grid(cdiv(M, DM_BM), cdiv(N, DM_BN));
#define MSY_Z(a, b)                                                                                      \
  if (opa == a && opb == b) {                                                                            \
    KScope ks__(KC_DMMA, 8.0 * M * N * K, st);                                                           \
    gemm_zdmma_kernel<a, b><<<grid, 128, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);         \
    MSY_LAUNCH_CK();                                                                                     \
    return 0;                                                                                            \
  }
  MSY_Z('N', 'N') MSY_Z('N', 'T') MSY_Z('T', 'N') MSY_Z('T', 'T') MSY_Z('C', 'N') MSY_Z('N', 'C')
  MSY_Z('C', 'C') MSY_Z('C', 'T') MSY_Z('T', 'C')
#undef MSY_Z
  return 1;
}

}  // namespace msy
