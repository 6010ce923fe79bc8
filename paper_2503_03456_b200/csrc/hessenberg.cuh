// hessenberg.cuh -- blocked Householder Hessenberg reduction H = Q0^H A Q0 (large m).
//
// Replaces the reference's unblocked `_hessenberg` (pkg/src/mpsylv/linalg.py:446-464,
// reflectors from `_make_reflector` linalg.py:276-292) for matrices above the
// one-CTA size.  Panel algorithm (compact-WY, Q_panel = I - V T V^H):
//   per panel column c = k+i:
//     hess_col_kernel (1 CTA): finish Y[:, i-1] = tau (A v - Y (V^H v)) and
//        T[:, i-1], apply the panel's earlier reflectors to column c (right:
//        -Y V[c,:]^H, left: -V T^H V^H a_c), generate reflector i;
//     hess_gemv_kernel (grid): A[:, c+1:m] v_i  (the BLAS-2 half, HBM/L2 bound)
//   per panel: trailing updates as GEMMs (right: -Y V^H; left: -V T^H V^H A).
// Q0 is formed afterwards by backward blocked accumulation (form_q).
#pragma once
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "gemm.cuh"

namespace cg = cooperative_groups;

namespace msy {

#ifndef MSY_HESS_NB
#define MSY_HESS_NB 32  // the panel kernels assume 32 (one lane per panel column): other widths are not supported
#endif
constexpr int HESS_NB = MSY_HESS_NB;  // panel width
constexpr int HESS_CHUNK = 64;  // gemv column chunk
constexpr int HESS_ROWS = 128;  // gemv rows per CTA
constexpr int HESS_TPB = 512;

// out[q] = sum_r conj(V[r, q]) x[r] over rows r0..m-1 for q < nq (nq <= HESS_NB):
// every thread accumulates all nq partial sums over its rows (independent loads),
// then one warp-shuffle tree per q and a cross-warp pass through shared memory.
template <class S>
__device__ __forceinline__ void batched_vhx(int m, int r0, const S* V, int ldv, int nq, const S* x, S* out,
                                            S (*redS)[HESS_TPB / 32]) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  S acc[HESS_NB];
#pragma unroll
  for (int q = 0; q < HESS_NB; q++) acc[q] = S(0);
  for (int r = r0 + tid; r < m; r += nt) {
    const S xv = x[r];
#pragma unroll
    for (int q = 0; q < HESS_NB; q++)
      if (q < nq) acc[q] = fmacc(V[r + (size_t)q * ldv], xv, acc[q]);
  }
#pragma unroll
  for (int q = 0; q < HESS_NB; q++) {
    if (q < nq) {
      S s = warp_sum(acc[q]);
      if (lane == 0) redS[q][wid] = s;
    }
  }
  __syncthreads();
  if (tid < nq) {
    S s = S(0);
    for (int w = 0; w < nw; w++) s += redS[tid][w];
    out[tid] = s;
  }
  __syncthreads();
}

// V: m x m buffer (column c = reflector of column c, zero above row c+1)
// Y: m x NB, T: NB x NB (this panel), part: nch x m partial gemv sums,
// tau: per-column taus (length m).
template <class S>
__global__ void __launch_bounds__(HESS_TPB) hess_col_kernel(int m, S* A, int lda, int k, int i, int nbp, S* V,
                                                            int ldv, S* Y, int ldy, S* T, int ldt, const S* part,
                                                            int nch, S* tau) {
  typedef typename tr<S>::R R;
  __shared__ S u[HESS_NB];
  __shared__ S w[HESS_NB];
  __shared__ S vrow[HESS_NB];
  __shared__ S redS[HESS_NB][HESS_TPB / 32];
  __shared__ R redR[HESS_TPB / 32];
  __shared__ S sh_beta, sh_tau, sh_scal;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int c = k + i;
  const S* Vp = V + (size_t)k * ldv;  // this panel's reflectors

  // ---- finish Y[:, i-1] and T[:, i-1] ----
  if (i > 0) {
    const int j = i - 1, cj = k + j;
    const S* vj = V + (size_t)cj * ldv;
    batched_vhx<S>(m, cj + 1, Vp, ldv, j, vj, u, redS);  // u = V[:, 0:j]^H v_j
    const S tj = tau[cj];
    for (int r = tid; r < m; r += nt) {
      S y = S(0);
      for (int ch = 0; ch < nch; ch++) y += part[(size_t)ch * m + r];
      for (int q = 0; q < j; q++) y = y - Y[r + (size_t)q * ldy] * u[q];
      Y[r + (size_t)j * ldy] = tj * y;
    }
    if (tid < j) {  // T[0:j, j] = -tau_j T[0:j,0:j] u
      S s = S(0);
      for (int q = tid; q < j; q++) s = fmac(T[tid + q * ldt], u[q], s);
      T[tid + j * ldt] = -(tj * s);
    }
    if (tid == 0) T[j + j * ldt] = tj;
    __syncthreads();
  }
  if (i >= nbp) return;

  S* ac = A + (size_t)c * lda;
  if (i > 0) {
    // ---- right ops of reflectors 0..i-1 on column c (all rows): a -= Y V[c, 0:i]^H ----
    if (tid < i) vrow[tid] = conj(Vp[c + (size_t)tid * ldv]);
    __syncthreads();
    for (int r = tid; r < m; r += nt) {
      S a = ac[r];
      for (int q = 0; q < i; q++) a = a - Y[r + (size_t)q * ldy] * vrow[q];
      ac[r] = a;
    }
    __syncthreads();
    // ---- left ops: a[k+1:m] -= V T^H (V^H a) ----
    batched_vhx<S>(m, k + 1, Vp, ldv, i, ac, u, redS);
    if (tid < i) {  // w = T^H u  (T upper => T^H lower)
      S s = S(0);
      for (int q = 0; q <= tid; q++) s = fmacc(T[q + tid * ldt], u[q], s);
      w[tid] = s;
    }
    __syncthreads();
    for (int r = k + 1 + tid; r < m; r += nt) {
      S a = ac[r];
      for (int q = 0; q < i; q++) a = a - Vp[r + (size_t)q * ldv] * w[q];
      ac[r] = a;
    }
    __syncthreads();
  }
  // ---- reflector for x = a[c+1:m] ----
  {
    R s = 0;
    for (int r = c + 2 + tid; r < m; r += nt) s += abs2(ac[r]);
    s = warp_sum(s);
    if (lane == 0) redR[wid] = s;
    __syncthreads();
    if (tid == 0) {
      R t = 0;
      for (int q = 0; q < nw; q++) t += redR[q];
      S x0 = ac[c + 1];
      if (t == R(0) && im(x0) == R(0)) {
        sh_tau = S(0); sh_beta = x0; sh_scal = S(0);
      } else {
        R nrm = sqrt(abs2(x0) + t);
        R b = re(x0) >= R(0) ? -nrm : nrm;
        sh_beta = mk<S>(b);
        sh_tau = (mk<S>(b) - x0) / mk<S>(b);
        sh_scal = S(1) / (x0 - mk<S>(b));
      }
    }
    __syncthreads();
    S* vc = V + (size_t)c * ldv;
    S scal = sh_scal;
    for (int r = c + 1 + tid; r < m; r += nt) {
      vc[r] = (r == c + 1) ? S(1) : ac[r] * scal;
      ac[r] = (r == c + 1) ? sh_beta : S(0);
    }
    if (tid == 0) tau[c] = sh_tau;
  }
}

// part[ch][r] = sum over columns q in chunk ch (q >= c0) of A[r, q] v[q]
template <class S>
__global__ void __launch_bounds__(HESS_ROWS) hess_gemv_kernel(int m, const S* __restrict__ A, int lda, int c0,
                                                              const S* __restrict__ v, S* part) {
  const int r = blockIdx.x * HESS_ROWS + threadIdx.x;
  const int ch = blockIdx.y;
  const int q0 = c0 + ch * HESS_CHUNK, q1 = min(m, q0 + HESS_CHUNK);
  __shared__ S vs[HESS_CHUNK];
  for (int q = q0 + threadIdx.x; q < q1; q += HESS_ROWS) vs[q - q0] = v[q];
  __syncthreads();
  if (r >= m) return;
  S s[8];
#pragma unroll
  for (int u = 0; u < 8; u++) s[u] = S(0);
  int q = q0;
  for (; q + 7 < q1; q += 8) {
#pragma unroll
    for (int u = 0; u < 8; u++) s[u] = fmac(A[r + (size_t)(q + u) * lda], vs[q + u - q0], s[u]);
  }
  for (; q < q1; q++) s[0] = fmac(A[r + (size_t)q * lda], vs[q - q0], s[0]);
  part[(size_t)ch * m + r] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

template <class S>
__global__ void set_identity_kernel(int m, int n, S* M, int ld) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < m) M[i + (size_t)j * ld] = (i == j) ? S(1) : S(0);
}
template <class S>
__global__ void zero_kernel(size_t n, S* p) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = S(0);
}
template <class S>
__global__ void clear_below_sub_kernel(int m, S* A, int lda) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < m && i > j + 1) A[i + (size_t)j * lda] = S(0);
}

// ---------------------------------------------------------------------------
// Persistent panel kernel: one cooperative launch per panel of HESS_NB columns.
// Rows are split into 32-row slabs owned by the CTAs; every per-column step is
// row-parallel, the few cross-row reductions (V^H a, ||x||, V^H v) go through a
// deterministic two-level sum (per-CTA partials in global memory, read back by
// every CTA in the same order), separated by grid-wide barriers.  Per column:
//   (1) right ops of earlier panel reflectors on column c, partials of V^H a
//   (2) left ops (a -= V T^H V^H a), partial ||a[c+2:]||^2, x0 = a[c+1]
//   (3) reflector (computed redundantly by every CTA), v and the new column c
//   (4) y = A[:, c+1:] v over each CTA's rows (coalesced, 8 warps split the
//       columns), partials of V^H v
//   (5) Y[:, i] = tau (y - Y V^H v), T[:, i]
constexpr int HP_TPB = 512;
constexpr int HESS_SPLITK = 16;  // K splits of the skinny V^H A products

// out[q] = sum_g red[g*HESS_NB + q] for q < nq, g < G, read by the whole CTA in a fixed
// order (8 groups of g, then the groups): deterministic, latency overlapped
template <class S>
__device__ __forceinline__ void cta_sum_partials(const S* red, int G, int nq, S* out, S (*scratch)[32]) {
  constexpr int NG = HP_TPB / 32;
  const int q = threadIdx.x & 31, grp = threadIdx.x >> 5;
  S s0 = S(0), s1 = S(0), s2 = S(0), s3 = S(0);
  if (q < nq) {
    int gg = grp;
    for (; gg + 3 * NG < G; gg += 4 * NG) {
      s0 += red[gg * HESS_NB + q];
      s1 += red[(gg + NG) * HESS_NB + q];
      s2 += red[(gg + 2 * NG) * HESS_NB + q];
      s3 += red[(gg + 3 * NG) * HESS_NB + q];
    }
    for (; gg < G; gg += NG) s0 += red[gg * HESS_NB + q];
  }
  scratch[grp][q] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (threadIdx.x < nq) {
    S t = S(0);
#pragma unroll
    for (int g8 = 0; g8 < HP_TPB / 32; g8++) t += scratch[g8][threadIdx.x];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}
constexpr int HP_ROWS = 32;

template <class S>
__global__ void __launch_bounds__(HP_TPB) hess_panel_coop_kernel(int m, S* A, int lda, int k, int nbp, S* V, int ldv,
                                                                 S* Y, int ldy, S* T, int ldt, S* tau, S* red1,
                                                                 S* red2, typename tr<S>::R* redR, S* slot) {
  typedef typename tr<S>::R R;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* sv = (S*)smem_raw;  // v (m entries)
  __shared__ S s_vrow[HESS_NB], s_u[HESS_NB], s_w[HESS_NB];
  __shared__ S s_part[HP_TPB / 32][HP_ROWS];
  __shared__ S s_beta, s_tau, s_scal;
  __shared__ R s_rsum[HP_TPB / 32];
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nslab = cdiv(m, HP_ROWS);
  const S* Vp = V + (size_t)k * ldv;
  for (int i = 0; i < nbp; i++) {
    const int c = k + i;
    S* ac = A + (size_t)c * lda;
    // ---- (1) right ops on column c, partials of V^H a over rows >= k+1 ----
    if (i > 0) {
      if (tid < i) s_vrow[tid] = conj(Vp[c + (size_t)tid * ldv]);
      __syncthreads();
      if (warp == 0) {
        S part[HESS_NB];
#pragma unroll
        for (int q = 0; q < HESS_NB; q++) part[q] = S(0);
        for (int s = g; s < nslab; s += G) {
          const int r = s * HP_ROWS + lane;
          if (r < m) {
            S a = ac[r];
#pragma unroll
            for (int q = 0; q < HESS_NB; q++)  // independent loads: full unroll, predicated
              if (q < i) a = a - Y[r + (size_t)q * ldy] * s_vrow[q];
            ac[r] = a;
            if (r >= k + 1) {
#pragma unroll
              for (int q = 0; q < HESS_NB; q++)
                if (q < i) part[q] = fmacc(Vp[r + (size_t)q * ldv], a, part[q]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < HESS_NB; q++)
          if (q < i) {
            S sum = warp_sum(part[q]);
            if (lane == 0) red1[g * HESS_NB + q] = sum;
          }
      }
      grid.sync();
      // ---- (2) left ops ----
      cta_sum_partials<S>(red1, G, i, s_u, s_part);
      if (tid < i) {  // w = T^H u
        S sum = S(0);
        for (int q = 0; q <= tid; q++) sum = fmacc(T[q + tid * ldt], s_u[q], sum);
        s_w[tid] = sum;
      }
      __syncthreads();
    }
    if (warp == 0) {
      R nrm = 0;
      for (int s = g; s < nslab; s += G) {
        const int r = s * HP_ROWS + lane;
        if (r < m) {
          S a = ac[r];
          if (i > 0 && r >= k + 1) {
#pragma unroll
            for (int q = 0; q < HESS_NB; q++)
              if (q < i) a = a - Vp[r + (size_t)q * ldv] * s_w[q];
            ac[r] = a;
          }
          if (r >= c + 2) nrm += abs2(a);
          if (r == c + 1) *slot = a;
        }
      }
      nrm = warp_sum(nrm);
      if (lane == 0) redR[g] = nrm;
    }
    grid.sync();
    // ---- (3) reflector (redundant per CTA), v, new column c ----
    {
      R t = 0;
      for (int gg = tid; gg < G; gg += HP_TPB) t += redR[gg];
      t = warp_sum(t);
      if (lane == 0) s_rsum[warp] = t;
      __syncthreads();
    }
    if (tid == 0) {
      R t = 0;
#pragma unroll
      for (int w8 = 0; w8 < HP_TPB / 32; w8++) t += s_rsum[w8];
      S x0 = *slot;
      if (t == R(0) && im(x0) == R(0)) {
        s_tau = S(0); s_beta = x0; s_scal = S(0);
      } else {
        R nrmv = sqrt(abs2(x0) + t);
        R b = re(x0) >= R(0) ? -nrmv : nrmv;
        s_beta = mk<S>(b);
        s_tau = (mk<S>(b) - x0) / mk<S>(b);
        s_scal = S(1) / (x0 - mk<S>(b));
      }
    }
    __syncthreads();
    {
      S* vc = V + (size_t)c * ldv;
      const S scal = s_scal, beta = s_beta;
      for (int s = g; s < nslab; s += G) {
        const int r = s * HP_ROWS + tid;
        if (tid < HP_ROWS && r < m && r >= c + 1) {
          S a = ac[r];
          vc[r] = (r == c + 1) ? S(1) : a * scal;
          ac[r] = (r == c + 1) ? beta : S(0);
        }
      }
      if (g == 0 && tid == 0) { tau[c] = s_tau; T[i + i * ldt] = s_tau; }
    }
    grid.sync();
    // ---- (4) y = A[:, c+1:m] v over own rows; partials of V[:, 0:i]^H v ----
    {
      const S* vc = V + (size_t)c * ldv;
      for (int q = c + 1 + tid; q < m; q += HP_TPB) sv[q] = vc[q];
      __syncthreads();
      S part[HESS_NB];
#pragma unroll
      for (int q = 0; q < HESS_NB; q++) part[q] = S(0);
      for (int s = g; s < nslab; s += G) {
        const int r = s * HP_ROWS + lane;
        const int rr = r < m ? r : m - 1;
        // each warp takes every NW-th column; UB coalesced 128-byte loads are issued
        // back to back per iteration so enough bytes are in flight to cover L2/HBM latency
        constexpr int NW = HP_TPB / 32, UB = sizeof(S) > 8 ? 8 : 32;
        S acc[8];
#pragma unroll
        for (int u = 0; u < 8; u++) acc[u] = S(0);
        int q = c + 1 + warp;
        for (; q + NW * (UB - 1) < m; q += NW * UB) {
          S a[UB];
#pragma unroll
          for (int u = 0; u < UB; u++) a[u] = A[rr + (size_t)(q + NW * u) * lda];
#pragma unroll
          for (int u = 0; u < UB; u++) acc[u & 7] = fmac(a[u], sv[q + NW * u], acc[u & 7]);
        }
        for (; q < m; q += NW) acc[0] = fmac(A[rr + (size_t)q * lda], sv[q], acc[0]);
        s_part[warp][lane] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        __syncthreads();
        if (tid < HP_ROWS && r < m) {
          S y = S(0);
#pragma unroll
          for (int w = 0; w < HP_TPB / 32; w++) y += s_part[w][tid];
          Y[r + (size_t)i * ldy] = y;  // unscaled, finished in (5)
          if (i > 0 && r >= c + 1) {
            const S vr = sv[r];
#pragma unroll
            for (int qq = 0; qq < HESS_NB; qq++)
              if (qq < i) part[qq] = fmacc(Vp[r + (size_t)qq * ldv], vr, part[qq]);
          }
        }
        __syncthreads();
      }
      if (warp == 0 && i > 0) {
#pragma unroll
        for (int qq = 0; qq < HESS_NB; qq++)
          if (qq < i) {
            S sum = warp_sum(part[qq]);
            if (lane == 0) red2[g * HESS_NB + qq] = sum;
          }
      }
    }
    grid.sync();
    // ---- (5) Y[:, i] = tau (y - Y[:, 0:i] u'), T[0:i, i] = -tau T u' ----
    {
      cta_sum_partials<S>(red2, G, i, s_u, s_part);
      const S ti = s_tau;
      for (int s = g; s < nslab; s += G) {
        const int r = s * HP_ROWS + tid;
        if (tid < HP_ROWS && r < m) {
          S y = Y[r + (size_t)i * ldy];
#pragma unroll
          for (int q = 0; q < HESS_NB; q++)
            if (q < i) y = y - Y[r + (size_t)q * ldy] * s_u[q];
          Y[r + (size_t)i * ldy] = ti * y;
        }
      }
      if (g == 0 && tid < i) {
        S sum = S(0);
        for (int q = tid; q < i; q++) sum = fmac(T[tid + q * ldt], s_u[q], sum);
        T[tid + i * ldt] = -(ti * sum);
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Panel kernel v2 (cooperative).  Rows are owned in 32-row slabs (slab s by CTA
// s mod G, at most HP2_OWN per CTA); each CTA caches its rows of the panel's V and
// Y, and a copy of T, in shared memory, so the per-column vector phases touch
// global memory only for column c itself.  Per panel column c = k + i:
//   A  own rows: a = A[:, c] - Y[:, :i] V[c, :i]^H; partials of V^H a          | sync
//   B  w = T^H u; own rows: a -= V w; column c back to HBM; partial norm       | sync
//   CD every CTA: reflector, v from column c (all rows), own rows of V[:, c];
//      y = A[:, c+1:] v as (slab x 256-column) units over all CTAs (float4
//      loads on the fp32 path); own rows: partials of V^H v                    | sync
//   E  own rows: Y[:, i] = tau (y - Y[:, :i] (V^H v)); column c := (beta, 0..);
//      T[:, i] (every CTA in smem, CTA 0 to HBM)
constexpr int HP2_CW = 256;
constexpr int HP2_OWN = 4;
constexpr int HP2_LD = HESS_NB + 1;
#ifdef MSY_HESS_PROF
__device__ unsigned long long g_hess_prof[8];
#define HPROF(slot)                                                                          \
  do {                                                                                       \
    if (g == 0 && tid == 0) {                                                                \
      unsigned long long t_;                                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                 \
      if (slot > 0) atomicAdd(&g_hess_prof[slot], t_ - t_prev_);                             \
      t_prev_ = t_;                                                                          \
    }                                                                                        \
  } while (0)
#else
#define HPROF(slot) do {} while (0)
#endif
template <class S>
static size_t hess2_smem(int m) {
  return ((size_t)m + 2 * (size_t)HP2_OWN * HESS_NB * HP2_LD + (size_t)HESS_NB * HP2_LD + (size_t)HP2_OWN * HP_ROWS) *
         sizeof(S);
}
template <class S>
__global__ void __launch_bounds__(HP_TPB) hess_panel2_kernel(int m, S* A, int lda, int k, int nbp, S* V, int ldv,
                                                             S* Y, int ldy, S* T, int ldt, S* tau, S* red1, S* red2,
                                                             typename tr<S>::R* redR, S* slot, S* ypart) {
  typedef typename tr<S>::R R;
  constexpr int NWP = HP_TPB / 32;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* sv = (S*)smem_raw;                              // v (m entries, zero above row c+1)
  S* Vc = sv + m;                                    // [own][q][row]: own rows of V[:, k:k+nb]
  S* Yc = Vc + HP2_OWN * HESS_NB * HP2_LD;           // [own][q][row]: own rows of Y
  S* Tc = Yc + HP2_OWN * HESS_NB * HP2_LD;           // T, [q][p] = T(q, p)
  S* scol = Tc + HESS_NB * HP2_LD;                   // [own][row]: own rows of column c
  __shared__ S s_u[HESS_NB], s_w[HESS_NB], s_acc[HESS_NB];
  __shared__ S s_part[NWP][32];
  __shared__ float s_p4[NWP][128];  // float4 gemv partials (fp32 path)
  __shared__ S s_beta, s_tau, s_scal;
  __shared__ R s_rsum[NWP];
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nslab = cdiv(m, HP_ROWS);
  const int nown = g < nslab ? (nslab - 1 - g) / G + 1 : 0;
  const S* Vp = V + (size_t)k * ldv;
#define VC(o, q) Vc[((o) * HESS_NB + (q)) * HP2_LD + lane]
#define YC(o, q) Yc[((o) * HESS_NB + (q)) * HP2_LD + lane]
#ifdef MSY_HESS_PROF
  unsigned long long t_prev_ = 0;
#endif
  HPROF(0);
  for (int e = tid; e < HESS_NB * HP2_LD; e += HP_TPB) Tc[e] = S(0);
  __syncthreads();
  for (int i = 0; i < nbp; i++) {
    const int c = k + i;
    S* ac = A + (size_t)c * lda;
    // ---- A ----
    if (warp == 0)
      for (int o = 0; o < nown; o++) {
        const int r = (g + o * G) * HP_ROWS + lane;
        scol[o * HP_ROWS + lane] = r < m ? ac[r] : S(0);
      }
    if (i > 0) {
      if (tid < HESS_NB) s_acc[tid] = S(0);
      if (tid < i) s_w[tid] = conj(Vp[c + (size_t)tid * ldv]);  // row c of V (conjugated)
      __syncthreads();
      if (warp == 0)
        for (int o = 0; o < nown; o++) {
          S a = scol[o * HP_ROWS + lane];
          for (int q = 0; q < i; q++) a = a - YC(o, q) * s_w[q];
          scol[o * HP_ROWS + lane] = a;
        }
      __syncthreads();
      for (int o = 0; o < nown; o++) {
        const int r = (g + o * G) * HP_ROWS + lane;
        const S a = (r < m && r >= k + 1) ? scol[o * HP_ROWS + lane] : S(0);
        for (int q = warp; q < i; q += NWP) {
          S val = warp_sum(conj(VC(o, q)) * a);
          if (lane == 0) s_acc[q] += val;
        }
      }
      __syncthreads();
      if (tid < HESS_NB) red1[g * HESS_NB + tid] = s_acc[tid];
      HPROF(1);
      grid.sync();
      HPROF(2);
      // ---- B ----
      cta_sum_partials<S>(red1, G, i, s_u, s_part);
      if (tid < i) {  // w = T^H u
        S sum = S(0);
        for (int q = 0; q <= tid; q++) sum = fmacc(Tc[q * HP2_LD + tid], s_u[q], sum);
        s_w[tid] = sum;
      }
    }
    __syncthreads();
    if (warp == 0) {
      R nrm = 0;
      for (int o = 0; o < nown; o++) {
        const int r = (g + o * G) * HP_ROWS + lane;
        S a = scol[o * HP_ROWS + lane];
        if (i > 0 && r >= k + 1)
          for (int q = 0; q < i; q++) a = a - VC(o, q) * s_w[q];
        if (r < m) {
          scol[o * HP_ROWS + lane] = a;
          ac[r] = a;
          if (r >= c + 2) nrm += abs2(a);
          if (r == c + 1) *slot = a;
        }
      }
      nrm = warp_sum(nrm);
      if (lane == 0) redR[g] = nrm;
    }
    HPROF(3);
    grid.sync();
    HPROF(4);
    // ---- CD ----
    {
      R t = 0;
      for (int gg = tid; gg < G; gg += HP_TPB) t += redR[gg];
      t = warp_sum(t);
      if (lane == 0) s_rsum[warp] = t;
      __syncthreads();
      if (tid == 0) {
        R tt = 0;
#pragma unroll
        for (int w8 = 0; w8 < NWP; w8++) tt += s_rsum[w8];
        S x0 = *slot;
        if (tt == R(0) && im(x0) == R(0)) {
          s_tau = S(0); s_beta = x0; s_scal = S(0);
        } else {
          R nrmv = sqrt(abs2(x0) + tt);
          R b = re(x0) >= R(0) ? -nrmv : nrmv;
          s_beta = mk<S>(b);
          s_tau = (mk<S>(b) - x0) / mk<S>(b);
          s_scal = S(1) / (x0 - mk<S>(b));
        }
        Tc[i * HP2_LD + i] = s_tau;
      }
      __syncthreads();
      const S scal = s_scal;
      for (int q = tid; q < m; q += HP_TPB) sv[q] = q > c + 1 ? ac[q] * scal : (q == c + 1 ? S(1) : S(0));
      if (g == 0 && tid == 0) { tau[c] = s_tau; T[i + i * ldt] = s_tau; }
      __syncthreads();
      if (warp == 0)
        for (int o = 0; o < nown; o++) {
          const int r = (g + o * G) * HP_ROWS + lane;
          const S vr = r < m ? sv[r] : S(0);
          VC(o, i) = vr;
          if (r < m && r >= c + 1) V[r + (size_t)c * ldv] = vr;
        }
      const int q0 = c + 1, nq = m - q0;
      const int nch = cdiv(nq, HP2_CW);
      bool vec = false;
      if constexpr (std::is_same<S, float>::value)
        vec = (lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
      if (vec) {
        if constexpr (std::is_same<S, float>::value) {
          // 128-row units: lane loads rows 4 lane .. 4 lane + 3 of each column as one float4
          const int nsl4 = cdiv(m, 128), units = nsl4 * nch;
          for (int u = g; u < units; u += G) {
            const int sl = u % nsl4, cc = u / nsl4;
            const int r4 = sl * 128 + 4 * lane;
            const int qa = q0 + cc * HP2_CW, qb = min(qa + HP2_CW, m);
            constexpr int UB = HP2_CW / NWP;
            float4 av[UB];
#pragma unroll
            for (int j = 0; j < UB; j++) {
              const int q = qa + warp + NWP * j;
              if (q < qb && r4 + 3 < m) {
                av[j] = *reinterpret_cast<const float4*>(A + r4 + (size_t)q * lda);
              } else if (q < qb) {
                const float* col = A + (size_t)q * lda;
                av[j] = make_float4(r4 < m ? col[r4] : 0.f, r4 + 1 < m ? col[r4 + 1] : 0.f,
                                    r4 + 2 < m ? col[r4 + 2] : 0.f, 0.f);
              } else {
                av[j] = make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < UB; j++) {
              const int q = qa + warp + NWP * j;
              const float vq = q < qb ? sv[q] : 0.f;
              acc.x = fmaf(av[j].x, vq, acc.x); acc.y = fmaf(av[j].y, vq, acc.y);
              acc.z = fmaf(av[j].z, vq, acc.z); acc.w = fmaf(av[j].w, vq, acc.w);
            }
            s_p4[warp][4 * lane] = acc.x; s_p4[warp][4 * lane + 1] = acc.y;
            s_p4[warp][4 * lane + 2] = acc.z; s_p4[warp][4 * lane + 3] = acc.w;
            __syncthreads();
            if (tid < 128) {
              const int row = sl * 128 + tid;
              if (row < m) {
                float y = 0.f;
#pragma unroll
                for (int w = 0; w < NWP; w++) y += s_p4[w][tid];
                ypart[(size_t)cc * m + row] = y;
              }
            }
            __syncthreads();
          }
        }
      } else {
        const int units = nslab * nch;
        for (int u = g; u < units; u += G) {
          const int sl = u % nslab, cc = u / nslab;
          const int r = sl * HP_ROWS + lane, rr = r < m ? r : m - 1;
          const int qa = q0 + cc * HP2_CW, qb = min(qa + HP2_CW, m);
          constexpr int UB = HP2_CW / NWP;  // columns per warp (16)
          S a[UB];
#pragma unroll
          for (int j = 0; j < UB; j++) {
            const int q = qa + warp + NWP * j;
            a[j] = q < qb ? A[rr + (size_t)q * lda] : S(0);
          }
          S acc0 = S(0), acc1 = S(0);
#pragma unroll
          for (int j = 0; j < UB; j += 2) {
            const int q = qa + warp + NWP * j;
            acc0 = fmac(a[j], q < qb ? sv[q] : S(0), acc0);
            acc1 = fmac(a[j + 1], q + NWP < qb ? sv[q + NWP] : S(0), acc1);
          }
          s_part[warp][lane] = acc0 + acc1;
          __syncthreads();
          if (warp == 0 && r < m) {
            S y = S(0);
#pragma unroll
            for (int w = 0; w < NWP; w++) y += s_part[w][lane];
            ypart[(size_t)cc * m + r] = y;
          }
          __syncthreads();
        }
      }
      if (i > 0) {  // partials of V[:, :i]^H v over own rows
        if (tid < HESS_NB) s_acc[tid] = S(0);
        __syncthreads();
        for (int o = 0; o < nown; o++) {
          const int r = (g + o * G) * HP_ROWS + lane;
          const S vr = r < m ? sv[r] : S(0);
          for (int q = warp; q < i; q += NWP) {
            S val = warp_sum(conj(VC(o, q)) * vr);
            if (lane == 0) s_acc[q] += val;
          }
        }
        __syncthreads();
        if (tid < HESS_NB) red2[g * HESS_NB + tid] = s_acc[tid];
      }
    }
    HPROF(6);
    grid.sync();
    HPROF(4);
    // ---- E ----
    {
      if (i > 0) cta_sum_partials<S>(red2, G, i, s_u, s_part);
      else __syncthreads();
      const int nch = cdiv(m - (c + 1), HP2_CW);
      const S ti = s_tau, beta = s_beta;
      for (int o = 0; o < nown; o++) {
        const int r = (g + o * G) * HP_ROWS + lane;
        S pa = S(0);
        if (r < m)
          for (int cc = warp; cc < nch; cc += NWP) pa += ypart[(size_t)cc * m + r];
        s_part[warp][lane] = pa;
        __syncthreads();
        if (warp == 0) {
          S y = S(0);
#pragma unroll
          for (int w = 0; w < NWP; w++) y += s_part[w][lane];
          for (int q = 0; q < i; q++) y = y - YC(o, q) * s_u[q];
          y = ti * y;
          YC(o, i) = y;
          if (r < m) {
            Y[r + (size_t)i * ldy] = y;
            if (r >= c + 1) ac[r] = (r == c + 1) ? beta : S(0);
          }
        }
        __syncthreads();
      }
      if (tid < i) {  // T[:, i] = -tau T u'  (every CTA keeps T; CTA 0 writes it out)
        S sum = S(0);
        for (int q = tid; q < i; q++) sum = fmac(Tc[tid * HP2_LD + q], s_u[q], sum);
        const S tv = -(ti * sum);
        Tc[tid * HP2_LD + i] = tv;
        if (g == 0) T[tid + i * ldt] = tv;
      }
      __syncthreads();
    }
    HPROF(7);
  }
#undef VC
#undef YC
}

template <class S>
struct HessWs {
  S *V, *Y, *T, *part, *tau, *W1, *W2, *red1, *red2, *slot, *skp;
  typename tr<S>::R* redR;
  static void carve(Arena& ar, int m, HessWs& w) {
    w.V = ar.get<S>((size_t)m * m);
    w.Y = ar.get<S>((size_t)m * HESS_NB);
    w.T = ar.get<S>((size_t)HESS_NB * (m + HESS_NB));  // one NB x NB T per panel
    w.part = ar.get<S>((size_t)cdiv(m, HESS_CHUNK) * m);
    w.tau = ar.get<S>((size_t)m);
    w.W1 = ar.get<S>((size_t)HESS_NB * m);
    w.W2 = ar.get<S>((size_t)HESS_NB * m);
    w.red1 = ar.get<S>((size_t)1024 * HESS_NB);
    w.red2 = ar.get<S>((size_t)1024 * HESS_NB);
    w.redR = ar.get<typename tr<S>::R>(1024);
    w.slot = ar.get<S>(8);
    w.skp = ar.get<S>((size_t)HESS_SPLITK * HESS_NB * m);
  }
};

// Cap on the panel grid of the calling host thread: the concurrent Schur(A) / Schur(B) pair
// sets half the SMs each, so both cooperative panel grids stay co-resident instead of
// serialising (measured: CH solve 1075 -> 1051 ms).  0 = no cap.
inline int& hess_grid_cap() {
  thread_local int cap = 0;
  return cap;
}

// grid size of the v2 panel kernel: enough CTAs for the gemv units, all co-resident
template <class S>
int hess2_grid(int m) {
  int dev, nsm, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = hess2_smem<S>(m);
  if (smem > 200 * 1024) return 0;
  // The attribute is a per-function ceiling shared by every thread: set it once to the largest
  // size any m may need (setting it per call to this m's size races with the concurrent
  // Schur(B) thread, whose launch would then exceed the ceiling).
  {
    static std::atomic<int> done{0};
    if (!done.load(std::memory_order_acquire)) {
      if (cudaFuncSetAttribute(hess_panel2_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
          cudaSuccess)
        return 0;
      done.store(1, std::memory_order_release);
    }
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, hess_panel2_kernel<S>, HP_TPB, smem) != cudaSuccess)
    return 0;
  const int nslab = cdiv(m, HP_ROWS), units = nslab * cdiv(m, HP2_CW);
  int G = std::min(per * nsm, std::max(nslab, std::min(units, nsm)));
  // optional cap (the concurrent Schur(A) / Schur(B) pair: two co-resident cooperative grids)
  constexpr int gmax_env = MSY_HESS_GMAX;
  const int gmax = gmax_env >= 0 ? gmax_env : hess_grid_cap();
  if (gmax > 0) G = std::min(G, std::max(gmax, cdiv(nslab, HP2_OWN)));
  return (G > 0 && cdiv(nslab, G) <= HP2_OWN) ? G : 0;  // each CTA caches at most HP2_OWN slabs
}

// grid size of the cooperative panel kernel (0 if it cannot be co-resident)
template <class S>
int hess_coop_grid(int m) {
  int dev, nsm, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = (size_t)m * sizeof(S);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(hess_panel_coop_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, hess_panel_coop_kernel<S>, HP_TPB, smem) != cudaSuccess)
    return 0;
  // two Schur factorisations (A and B) run concurrently: leave room for both
  int cap = std::min(per * nsm / 2, 128);
  return std::min(cap, cdiv(m, HP_ROWS));
}

// In place: A -> H (upper Hessenberg), Q (m x m) = Q0.
template <class S>
int hessenberg_blocked_launch(int m, S* A, int lda, S* Q, int ldq, HessWs<S>& w, cudaStream_t st) {
  const int ldv = m, ldy = m, ldt = HESS_NB;
  zero_kernel<S><<<cdiv((size_t)m * m, 256), 256, 0, st>>>((size_t)m * m, w.V);
  MSY_LAUNCH_CK();
  const int last = m - 3;  // last column that gets a reflector
  constexpr int hmode = MSY_HESS_MODE;  // 0 per-column kernels, 1 v1 cooperative, 2 v2 cooperative
  const int G = hmode == 0 ? 0 : (hmode == 1 ? hess_coop_grid<S>(m) : hess2_grid<S>(m));
  int np = 0;
  for (int k = 0; k <= last; k += HESS_NB, np++) {
    const int nbp = min(HESS_NB, last - k + 1);
    S* T = w.T + (size_t)np * HESS_NB * ldt;
    zero_kernel<S><<<cdiv(HESS_NB * HESS_NB, 256), 256, 0, st>>>((size_t)HESS_NB * HESS_NB, T);
    if (G > 0) {  // one persistent cooperative launch for the whole panel
      S* Ap = A;
      int mm = m, ldaa = lda, kk = k, nb_ = nbp, ldvv = ldv, ldyy = ldy, ldtt = ldt;
      S *Vv = w.V, *Yy = w.Y, *Tt = T, *ta = w.tau, *r1 = w.red1, *r2 = w.red2, *sl = w.slot;
      typename tr<S>::R* rR = w.redR;
      S* yp = w.part;
      void* args[] = {&mm, &Ap, &ldaa, &kk, &nb_, &Vv, &ldvv, &Yy, &ldyy, &Tt, &ldtt, &ta, &r1, &r2, &rR, &sl, &yp};
      const void* fn = hmode == 1 ? (const void*)hess_panel_coop_kernel<S> : (const void*)hess_panel2_kernel<S>;
      KScope ks(KC_HESS, 0, st);
      MSY_CK(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(HP_TPB), args,
                                         hmode == 1 ? (size_t)m * sizeof(S) : hess2_smem<S>(m), st));
      MSY_LAUNCH_CK();
    }
    for (int i = 0; i < nbp && G == 0; i++) {
      const int c = k + i;
      int nch = i > 0 ? cdiv(m - c, HESS_CHUNK) : 0;  // gemv for reflector i-1 covered columns c..m-1
      hess_col_kernel<S><<<1, HESS_TPB, 0, st>>>(m, A, lda, k, i, nbp, w.V, ldv, w.Y, ldy, T, ldt, w.part, nch, w.tau);
      MSY_LAUNCH_CK();
      // gemv with v_i over columns c+1..m-1
      int nchn = cdiv(m - (c + 1), HESS_CHUNK);
      hess_gemv_kernel<S><<<dim3(cdiv(m, HESS_ROWS), nchn), HESS_ROWS, 0, st>>>(m, A, lda, c + 1, w.V + (size_t)c * ldv, w.part);
      MSY_LAUNCH_CK();
    }
    if (G == 0) {  // finish Y[:, nbp-1]
      int c = k + nbp;
      int nch = cdiv(m - c, HESS_CHUNK);
      hess_col_kernel<S><<<1, HESS_TPB, 0, st>>>(m, A, lda, k, nbp, nbp, w.V, ldv, w.Y, ldy, T, ldt, w.part, nch,
                                                 w.tau);
      MSY_LAUNCH_CK();
    }
    const int c1 = k + nbp;  // first trailing column
    const int nc = m - c1;
    if (nc > 0) {
      const S* Vp = w.V + (size_t)k * ldv;  // columns k..k+nbp-1
      // right: A[:, c1:m] -= Y V[c1:m, :]^H
      int rc = gemm<S>('N', 'C', m, nc, nbp, S(-1), w.Y, ldy, Vp + c1, ldv, S(1), A + (size_t)c1 * lda, lda, st);
      if (rc) return rc;
      // left: W1 = V[k+1:m,:]^H A[k+1:m, c1:m]; W2 = T^H W1; A -= V W2
      rc = gemm_splitk<S>('C', 'N', nbp, nc, m - k - 1, S(1), Vp + (k + 1), ldv, A + (k + 1) + (size_t)c1 * lda, lda,
                          S(0), w.W1, HESS_NB, w.skp, HESS_SPLITK, st);
      if (rc) return rc;
      rc = gemm<S>('C', 'N', nbp, nc, nbp, S(1), T, ldt, w.W1, HESS_NB, S(0), w.W2, HESS_NB, st);
      if (rc) return rc;
      rc = gemm<S>('N', 'N', m - k - 1, nc, nbp, S(-1), Vp + (k + 1), ldv, w.W2, HESS_NB, S(1),
                   A + (k + 1) + (size_t)c1 * lda, lda, st);
      if (rc) return rc;
    }
  }
#ifdef MSY_HESS_PROF
  {
    unsigned long long h[8];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_hess_prof, sizeof(h));
    fprintf(stderr, "hess panel phases (ms, CTA 0): A %.2f syncA %.2f B %.2f syncs %.2f C %.2f D %.2f E %.2f\n",
            h[1] * 1e-6, h[2] * 1e-6, h[3] * 1e-6, h[4] * 1e-6, h[5] * 1e-6, h[6] * 1e-6, h[7] * 1e-6);
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_hess_prof, z, sizeof(z));
  }
#endif
  clear_below_sub_kernel<S><<<dim3(cdiv(m, 256), m), 256, 0, st>>>(m, A, lda);
  MSY_LAUNCH_CK();
  // ---- form Q0 = P_0 ... P_{m-3} by backward panel accumulation ----
  set_identity_kernel<S><<<dim3(cdiv(m, 256), m), 256, 0, st>>>(m, m, Q, ldq);
  MSY_LAUNCH_CK();
  for (int p = np - 1; p >= 0; p--) {
    int k = p * HESS_NB;
    int nbp = min(HESS_NB, last - k + 1);
    const S* Vp = w.V + (size_t)k * ldv;
    const S* T = w.T + (size_t)p * HESS_NB * ldt;
    int r0 = k + 1, nr = m - r0;
    // Q[r0:m, r0:m] -= V T (V^H Q[r0:m, r0:m])
    int rc = gemm_splitk<S>('C', 'N', nbp, nr, nr, S(1), Vp + r0, ldv, Q + r0 + (size_t)r0 * ldq, ldq, S(0), w.W1,
                            HESS_NB, w.skp, HESS_SPLITK, st);
    if (rc) return rc;
    rc = gemm<S>('N', 'N', nbp, nr, nbp, S(1), T, ldt, w.W1, HESS_NB, S(0), w.W2, HESS_NB, st);
    if (rc) return rc;
    rc = gemm<S>('N', 'N', nr, nr, nbp, S(-1), Vp + r0, ldv, w.W2, HESS_NB, S(1), Q + r0 + (size_t)r0 * ldq, ldq, st);
    if (rc) return rc;
  }
  return 0;
}


// Batched lanes (many m ~ 512 equations, bound by the launch rate of their host threads) replay
// the reduction as a CUDA graph: for given pointers and m it is a fixed sequence of ~170 launches
// (cooperative panels included) with no host decision in between.  A lane's first reduction with
// a key runs directly (one-time kernel attributes), the second is captured, later ones replay.
#ifndef MSY_HESS_GRAPH
#define MSY_HESS_GRAPH 1
#endif
inline bool& hess_graph_lane() {
  thread_local bool b = false;
  return b;
}
struct HessGraphEntry {
  const void *A, *Q, *V;
  int m, lda, ldq, cap, state;  // state 0: seen once, 1: graph ready, -1: capture failed (launch directly)
  cudaGraphExec_t exec;
  unsigned long long nodes;     // kernel launches inside the graph (for the launch counter)
};
inline std::vector<HessGraphEntry>& hess_graph_cache() {
  thread_local std::vector<HessGraphEntry> c;
  return c;
}
template <class S>
int hessenberg_blocked(int m, S* A, int lda, S* Q, int ldq, HessWs<S>& w, cudaStream_t st) {
  if (!MSY_HESS_GRAPH || !hess_graph_lane() || ktimer().on.load(std::memory_order_relaxed))
    return hessenberg_blocked_launch<S>(m, A, lda, Q, ldq, w, st);
  auto& cache = hess_graph_cache();
  HessGraphEntry* e = nullptr;
  for (auto& c : cache)
    if (c.A == A && c.Q == Q && c.V == w.V && c.m == m && c.lda == lda && c.ldq == ldq && c.cap == hess_grid_cap()) e = &c;
  if (!e) {
    if (cache.size() >= 8) {  // a lane sees two keys (A and B) per workspace: keep the cache small
      if (cache.front().state == 1) cudaGraphExecDestroy(cache.front().exec);
      cache.erase(cache.begin());
    }
    cache.push_back({A, Q, w.V, m, lda, ldq, hess_grid_cap(), 0, nullptr, 0});
    return hessenberg_blocked_launch<S>(m, A, lda, Q, ldq, w, st);
  }
  if (e->state == 1) {
    MSY_CK(cudaGraphLaunch(e->exec, st));
    __atomic_add_fetch(&launch_counter(), e->nodes, __ATOMIC_RELAXED);
    return 0;
  }
  if (e->state < 0) return hessenberg_blocked_launch<S>(m, A, lda, Q, ldq, w, st);
  // capture
  if (cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    e->state = -1;
    return hessenberg_blocked_launch<S>(m, A, lda, Q, ldq, w, st);
  }
  const int rc = hessenberg_blocked_launch<S>(m, A, lda, Q, ldq, w, st);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(st, &g);
  if (rc != 0 || ce != cudaSuccess || g == nullptr ||
      cudaGraphInstantiate(&e->exec, g, nullptr, nullptr, 0) != cudaSuccess) {
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    e->state = -1;
    return hessenberg_blocked_launch<S>(m, A, lda, Q, ldq, w, st);  // nothing ran during the capture
  }
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);  // every node is one of the reduction's kernels
  cudaGraphDestroy(g);
  e->nodes = nn;
  e->state = 1;
  MSY_CK(cudaGraphLaunch(e->exec, st));
  return 0;
}

}  // namespace msy
