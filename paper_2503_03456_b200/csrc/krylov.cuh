// krylov.cuh -- the Arnoldi step of GMRES-IR's inner solver on the device.
//
// Replaces the vector work of the reference's restarted GMRES (pkg/src/mpsylv/gmresir.py:112-205):
// modified Gram-Schmidt of w = M v_j against v_0..v_j (h_i = <v_i, w>, w -= h_i v_i in order,
// like the reference), the norm h_{j+1,j} = ||w||_2 and the new basis vector v_{j+1} = w / h_{j+1,j}
// -- one cooperative launch with grid barriers between the dependent reductions, instead of
// 2(j+1)+1 separate launches and host round trips.  Reductions are two-level in a fixed order
// (per-block partials, then every block sums the partials in block order), so the result is
// run-to-run deterministic.  The host reads h (j+2 values) once per Arnoldi step.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace msy {

namespace cgk = cooperative_groups;
constexpr int KR_TPB = 256;

template <class S>
__device__ __forceinline__ S kr_block_sum(S v, S* buf) {
  typedef typename tr<S>::R R;
  if constexpr (tr<S>::cx) {
    __shared__ R bx[KR_TPB / 32], by[KR_TPB / 32];
    R x = block_sum(v.x, bx), y = block_sum(v.y, by);
    return S(x, y);
  } else {
    return block_sum(v, buf);
  }
}

// V: N x (j+2), column-major (ld ldv); w (N) is overwritten by the orthogonalised vector; h:
// (j+2) entries, h[0..j] = the MGS coefficients, h[j+1] = ||w|| (real); v_{j+1} = w / ||w||
// written into V[:, j+1] unless ||w|| is 0 or non-finite.  part: 2 * gridDim.x scalars.
template <class S>
__global__ void __launch_bounds__(KR_TPB) krylov_mgs_kernel(int N, S* V, int ldv, int j, S* w, S* h, S* part) {
  typedef typename tr<S>::R R;
  cgk::grid_group grid = cgk::this_grid();
  __shared__ S sbuf[KR_TPB / 32];
  __shared__ S s_h;
  const int G = gridDim.x, tid = threadIdx.x;
  const size_t stride = (size_t)G * KR_TPB, first = (size_t)blockIdx.x * KR_TPB + tid;
  for (int i = 0; i <= j; i++) {
    const S* vi = V + (size_t)i * ldv;
    S acc = S(0);
    for (size_t e = first; e < (size_t)N; e += stride) acc = acc + conj(vi[e]) * w[e];
    acc = kr_block_sum(acc, sbuf);
    if (tid == 0) part[blockIdx.x + (i & 1) * G] = acc;
    grid.sync();
    if (tid == 0) {  // every block sums the partials in block order (identical h in all blocks)
      S hs = S(0);
      for (int b = 0; b < G; b++) hs = hs + part[b + (i & 1) * G];
      s_h = hs;
      if (blockIdx.x == 0) h[i] = hs;
    }
    __syncthreads();
    const S hi = s_h;
    for (size_t e = first; e < (size_t)N; e += stride) w[e] = w[e] - hi * vi[e];
    // partials of step i+1 go to the other half of `part`: no barrier needed here
  }
  R ss = 0;
  for (size_t e = first; e < (size_t)N; e += stride) ss += abs2(w[e]);
  __shared__ R rbuf[KR_TPB / 32];
  ss = block_sum(ss, rbuf);
  if (tid == 0) part[blockIdx.x + ((j + 1) & 1) * G] = S(ss);
  grid.sync();
  __shared__ R s_nrm;
  if (tid == 0) {
    R t = 0;
    for (int b = 0; b < G; b++) t += re(part[b + ((j + 1) & 1) * G]);
    s_nrm = sqrt(t);
    if (blockIdx.x == 0) h[j + 1] = S(s_nrm);
  }
  __syncthreads();
  const R nrm = s_nrm;
  if (nrm != R(0) && isfinite(nrm)) {
    S* vn = V + (size_t)(j + 1) * ldv;
    const R inv = R(1) / nrm;
    for (size_t e = first; e < (size_t)N; e += stride) vn[e] = w[e] * S(inv);
  }
}

template <class S>
int krylov_mgs(int N, S* V, int ldv, int j, S* w, S* h, S* part, int G, cudaStream_t st) {
  void* args[] = {&N, &V, &ldv, &j, &w, &h, &part};
  MSY_CK(cudaLaunchCooperativeKernel((const void*)krylov_mgs_kernel<S>, dim3(G), dim3(KR_TPB), args, 0, st));
  MSY_LAUNCH_CK();
  return 0;
}

// co-resident grid size for the cooperative launch (blocks; 0 if none)
template <class S>
int krylov_grid(int N) {
  int dev = 0, nsm = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, krylov_mgs_kernel<S>, KR_TPB, 0) != cudaSuccess) return 0;
  const int want = std::max(1, cdiv(N, KR_TPB * 4));
  return std::max(1, std::min(std::min(per, 2) * nsm, want));
}

}  // namespace msy
