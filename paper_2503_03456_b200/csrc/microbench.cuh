// microbench.cuh -- measured arithmetic peaks for the roofline denominators.
//
// MEASURED_PEAKS.json carries only HBM and bf16; the path is bound by FP32 SIMT
// (Schur, Y0) and FP64 (DMMA / DFMA) throughput, so the library measures those
// peaks on the box: long chains of independent FFMA / DFMA / DMMA.8x8x4 per warp,
// every SM busy, timed with CUDA events.
#pragma once
#include "common.cuh"
#include "gemm_dmma.cuh"

namespace msy {

template <class T>
__global__ void __launch_bounds__(256) fma_peak_kernel(int iters, T* out) {
  T a[8], b = T(1.0000001), c = T(0.9999999);
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = T(threadIdx.x + i);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fma(a[i], b, c);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += a[i];
  if (s == T(-1.2345)) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dmma_peak_kernel(int iters, double* out) {
  double d[8][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 8; i++) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) dmma884(d[i][0], d[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += d[i][0] + d[i][1];
  if (s == -1.2345) out[threadIdx.x] = s;
}

// kind 0: FFMA, 1: DFMA, 2: DMMA.  Returns TFLOP/s.
static int microbench(int kind, double* tflops, cudaStream_t st) {
  int dev, nsm;
  MSY_CK(cudaGetDevice(&dev));
  MSY_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double* out;
  MSY_CK(cudaMallocAsync(&out, 256 * sizeof(double), st));
  cudaEvent_t e0, e1;
  MSY_CK(cudaEventCreate(&e0));
  MSY_CK(cudaEventCreate(&e1));
  const int blocks = nsm * 8, threads = 256;
  int iters = kind == 2 ? 4096 : 16384;
  double flops = 0;
  for (int rep = 0; rep < 2; rep++) {  // first pass warms clocks
    MSY_CK(cudaEventRecord(e0, st));
    if (kind == 0) fma_peak_kernel<float><<<blocks, threads, 0, st>>>(iters, (float*)out);
    else if (kind == 1) fma_peak_kernel<double><<<blocks, threads, 0, st>>>(iters, out);
    else dmma_peak_kernel<<<blocks, threads, 0, st>>>(iters, out);
    MSY_LAUNCH_CK();
    MSY_CK(cudaEventRecord(e1, st));
  }
  MSY_CK(cudaEventSynchronize(e1));
  float ms = 0;
  MSY_CK(cudaEventElapsedTime(&ms, e0, e1));
  if (kind == 2) flops = (double)blocks * (threads / 32) * iters * 8 * 512.0;  // 8x8x4 MACs x2 per warp-mma
  else flops = (double)blocks * threads * iters * 8 * 2.0;
  *tflops = flops / (ms * 1e-3) / 1e12;
  MSY_CK(cudaEventDestroy(e0));
  MSY_CK(cudaEventDestroy(e1));
  MSY_CK(cudaFreeAsync(out, st));
  return 0;
}

}  // namespace msy
