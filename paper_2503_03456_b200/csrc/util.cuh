// util.cuh -- elementwise kernels and deterministic norms for the refinement loop.
//
// refine_update_kernel fuses the reference's iterate update and stopping-rule
// norms (pkg/src/mpsylv/refinement.py:128-138: Y <- Y + D, ||D||_F, ||Y||_F,
// non-finite check) into one pass; all reductions use a fixed two-level order so
// results are run-to-run deterministic.
#pragma once
#include "common.cuh"

namespace msy {

constexpr int RED_BLOCKS = 592;  // 4 x 148 SMs
constexpr int RED_TPB = 256;

// dst = (D) src with overflow detection (finite -> inf is FormatOverflowError, linalg.py:113-119)
template <class D, class Sx>
__global__ void convert_kernel(int rows, int cols, const Sx* __restrict__ src, int lds, D* dst, int ldd, int* ovf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  for (; j < cols; j += gridDim.y) {
    if (i >= rows) continue;
    Sx v = src[i + (size_t)j * lds];
    D w = conv<D>(v);
    dst[i + (size_t)j * ldd] = w;
    if (ovf && !isfin(w) && isfin(v)) *ovf = 1;
  }
}
template <class D, class Sx>
static int convert(int rows, int cols, const Sx* src, int lds, D* dst, int ldd, int* ovf, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  convert_kernel<D, Sx><<<dim3(cdiv(rows, 256), std::min(cols, 65535)), 256, 0, st>>>(rows, cols, src, lds, dst, ldd,
                                                                                      ovf);
  MSY_LAUNCH_CK();
  return 0;
}

// dst = src^H (n x n tiles through smem)
template <class S>
__global__ void conj_transpose_kernel(int rows, int cols, const S* __restrict__ src, int lds, S* dst, int ldd) {
  __shared__ S t[32][33];
  int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    int i = bx + threadIdx.x, j = by + k;
    if (i < rows && j < cols) t[k][threadIdx.x] = src[i + (size_t)j * lds];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    int i = by + threadIdx.x, j = bx + k;  // dst is cols x rows
    if (i < cols && j < rows) dst[i + (size_t)j * ldd] = conj(t[threadIdx.x][k]);
  }
}
template <class S>
static int conj_transpose(int rows, int cols, const S* src, int lds, S* dst, int ldd, cudaStream_t st) {
  conj_transpose_kernel<S><<<dim3(cdiv(rows, 32), cdiv(cols, 32)), dim3(32, 8), 0, st>>>(rows, cols, src, lds, dst, ldd);
  MSY_LAUNCH_CK();
  return 0;
}

template <class S>
__global__ void copy2d_kernel(int rows, int cols, const S* __restrict__ src, int lds, S* dst, int ldd) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  for (; j < cols; j += gridDim.y)
    if (i < rows) dst[i + (size_t)j * ldd] = src[i + (size_t)j * lds];
}
template <class S>
static int copy2d(int rows, int cols, const S* src, int lds, S* dst, int ldd, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  copy2d_kernel<S><<<dim3(cdiv(rows, 256), std::min(cols, 65535)), 256, 0, st>>>(rows, cols, src, lds, dst, ldd);
  MSY_LAUNCH_CK();
  return 0;
}

template <class S>
__global__ void fill_kernel(int rows, int cols, S v, S* dst, int ldd) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  for (; j < cols; j += gridDim.y)
    if (i < rows) dst[i + (size_t)j * ldd] = v;
}
template <class S>
static int fill(int rows, int cols, S v, S* dst, int ldd, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  fill_kernel<S><<<dim3(cdiv(rows, 256), std::min(cols, 65535)), 256, 0, st>>>(rows, cols, v, dst, ldd);
  MSY_LAUNCH_CK();
  return 0;
}

// A = A + B (elementwise, same shape)
template <class S>
__global__ void add_kernel(int rows, int cols, S* A, int lda, const S* __restrict__ B, int ldb) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  for (; j < cols; j += gridDim.y)
    if (i < rows) A[i + (size_t)j * lda] = A[i + (size_t)j * lda] + B[i + (size_t)j * ldb];
}

// partial sums over a grid-stride loop: out[b*3 + {0,1,2}]
//   mode 0: sumsq(X);   mode 1: sumsq(X - Yv);   mode 2 (refine): Y += D, sumsq(D), sumsq(Y), nonfinite
// guard (mode 2, optional): skip the update (all-zero partials) unless guard[0] -- the
// previous pass's sumsq(D) -- is finite and the trsyl status word says OK, so a failed
// correction leaves Y untouched as in refinement.py:123-127 (no host round trip needed).
template <class S>
__global__ void __launch_bounds__(RED_TPB) reduce_kernel(int mode, int rows, int cols, S* X, int ldx, const S* Yv,
                                                         int ldy, double* part, const double* guard = nullptr,
                                                         const int* tstat = nullptr) {
  __shared__ double buf[RED_TPB / 32];
  double a = 0, b = 0, c = 0;
  size_t tot = (size_t)rows * cols;
  if (guard && (!isfinite(guard[0]) || (tstat && tstat[0] != 0x7fffffff))) tot = 0;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    int i = (int)(e % rows), j = (int)(e / rows);
    if (mode == 0) {
      a += (double)abs2(X[i + (size_t)j * ldx]);
    } else if (mode == 1) {
      a += (double)abs2(X[i + (size_t)j * ldx] - Yv[i + (size_t)j * ldy]);
    } else {
      S d = Yv[i + (size_t)j * ldy];
      S y = X[i + (size_t)j * ldx] + d;
      X[i + (size_t)j * ldx] = y;
      a += (double)abs2(d);
      b += (double)abs2(y);
      if (!isfin(d) || !isfin(y)) c += 1;
    }
  }
  a = block_sum(a, buf);
  b = block_sum(b, buf);
  c = block_sum(c, buf);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = a;
    part[blockIdx.x * 3 + 1] = b;
    part[blockIdx.x * 3 + 2] = c;
  }
}
__global__ void reduce_final_kernel(int nparts, const double* part, double* out) {
  __shared__ double buf[RED_TPB / 32];
  for (int q = 0; q < 3; q++) {
    double s = 0;
    for (int k = threadIdx.x; k < nparts; k += blockDim.x) s += part[k * 3 + q];
    s = block_sum(s, buf);
    if (threadIdx.x == 0) out[q] = s;
  }
}
// out[0..2] = sums (sumsq, sumsq2, nonfinite count)
template <class S>
static int reduce(int mode, int rows, int cols, S* X, int ldx, const S* Yv, int ldy, double* part, double* out,
                  cudaStream_t st, const double* guard = nullptr, const int* tstat = nullptr) {
  long tot = (long)rows * cols;
  int nb = (int)std::min<long>(RED_BLOCKS, std::max<long>(1, cdiv(tot, RED_TPB)));
  reduce_kernel<S><<<nb, RED_TPB, 0, st>>>(mode, rows, cols, X, ldx, Yv, ldy, part, guard, tstat);
  MSY_LAUNCH_CK();
  reduce_final_kernel<<<1, RED_TPB, 0, st>>>(nb, part, out);
  MSY_LAUNCH_CK();
  return 0;
}

// The refinement loop's per-iteration status record, gathered on the device so the host
// reads it with ONE copy: {trsyl status word, sumsq(D), sumsq(D) (guarded pass),
// sumsq(Y + D), nonfinite count}.
__global__ void pack_status_kernel(const int* tstat, const double* red_d, const double* red_u, double* out) {
  out[0] = (double)tstat[0];
  out[1] = red_d[0];
  out[2] = red_u[0];
  out[3] = red_u[1];
  out[4] = red_u[2];
}

// First column (in the recurrence's solve order: ascending for an upper T_B, descending for
// a lower one) holding a non-finite entry -- the column sylvester.py:147-149 names in its
// NumericBreakdownError.  out[0] must start at INT_MAX (first_nonfinite_init_kernel).
__global__ void first_nonfinite_init_kernel(int* out) { out[0] = 0x7fffffff; }
template <class S>
__global__ void first_nonfinite_kernel(int rows, int cols, const S* X, int ldx, int lowerB, int* out) {
  const size_t tot = (size_t)rows * cols;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    int i = (int)(e % rows), j = (int)(e / rows);
    if (!isfin(X[i + (size_t)j * ldx])) atomicMin(out, lowerB ? cols - 1 - j : j);
  }
}

}  // namespace msy
