// multishift.cuh -- small-bulge multishift QR for Hessenberg matrices above the one-CTA size.
//
// Replaces the reference's single-shift sweep loop `schur` (pkg/src/mpsylv/linalg.py:518-577,
// rotations `_givens`/`_rot_rows`/`_rot_cols` :467-499) for large m.  B200 design:
//   * a chain of nb double-shift bulges (3-element reflectors, bulges 4 rows apart,
//     one warp per bulge, all bulges of a step in parallel) is chased through a
//     W x W diagonal window held in shared memory by ONE CTA (chase_kernel);
//     the window's accumulated orthogonal factor Z stays in smem too;
//   * the off-window parts of H (rows to the right, columns above) and the Schur
//     vectors U are updated with Z as in-place GEMMs over many CTAs (apply_z_kernel);
//   * deflation uses the reference's criterion (linalg.py:541-544); converged
//     trailing 1x1 (and, real, 2x2) blocks are skipped, complex 2x2 blocks are
//     split in scan_kernel; blocks of order <= NMIN finish in schur_small_kernel.
//   * shifts: eigenvalues of the trailing ns x ns block (schur_small_kernel in
//     eigenvalue mode), exceptional shifts after 6 stagnant sweeps.
#pragma once
#include <type_traits>
#include <cooperative_groups.h>

#include "common.cuh"
#include "schur_small.cuh"

namespace msy {

template <class S> struct MsCfg;
#ifndef MSY_FW
#define MSY_FW 128  // fp32 chase window (compile-time smem layout); MSY_FNB bulges per chain.
                    // Measured at m=4096: (160,24) 760-825 ms, (128,16) 670, (128,12) 703, (144,20) 750;
                    // W must be >= the one-CTA block order (128): endgame blocks go through apply_z
#endif
#ifndef MSY_FNB
#define MSY_FNB 16
#endif
template <> struct MsCfg<float> { static constexpr int W = MSY_FW, NB = MSY_FNB; };
template <> struct MsCfg<double> { static constexpr int W = 112, NB = 16; };
template <> struct MsCfg<cfloat> { static constexpr int W = 112, NB = 16; };
template <> struct MsCfg<cdouble> { static constexpr int W = 80, NB = 10; };
constexpr int ZMAX = 160;  // largest window / block order handled by apply_z
constexpr int ZMASK_OFF = ZMAX * ZMAX - 1;  // chase2_kernel: nonzero-block map of a window factor, in its buffer's last word

// ---------------------------------------------------------------------------
// window chase: one CTA, one warp per bulge, the W x W window of H and its
// accumulated Z in shared memory.  Per step: every active bulge computes its
// reflector (all lanes, broadcast reads), applies it from the left to the
// window's rows (phase A), then from the right to the window's columns and
// to Z (phase B).  Bulges sit 4 rows apart, so one step's bulges touch disjoint
// rows/columns; the two phases order the only overlapping entries.  The warp
// ops are branch-free (warp_left3 / warp_right3 redirect idle lanes to a dummy
// row/column of the smem window).
#ifndef MSY_KMAX
#define MSY_KMAX 8
#endif
constexpr int KMAX = MSY_KMAX;  // bulge chains in flight per sweep (one CTA each)
constexpr size_t ZT_DELTA = (size_t)2 * KMAX * ZMAX * ZMAX;  // chase2_kernel: row-major copy of a window factor, this far behind it
// fixed-trip, loads-first warp ops (wl3u / wr3u2) for real fp32 windows; the wider types keep
// the loop forms (the unrolled register arrays would spill)
template <class S> constexpr bool kFixedTrip = std::is_same<S, float>::value;
template <class S>
struct ChaseJobs {
  int ws[KMAX], we[KMAX], t0[KMAX], t1[KMAX];
  const typename tr<S>::R* shifts[KMAX];
  S* Z[KMAX];
};

template <class S>
__global__ void __launch_bounds__(512) chase_kernel(S* H, int ldh, int lo, int hi, int nb, const ChaseJobs<S> jobs) {
  typedef typename tr<S>::R R;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ws = jobs.ws[blockIdx.x], we = jobs.we[blockIdx.x], t0 = jobs.t0[blockIdx.x], t1 = jobs.t1[blockIdx.x];
  const R* __restrict__ shifts = jobs.shifts[blockIdx.x];
  S* Zg = jobs.Z[blockIdx.x];
  const int nw = we - ws;
  constexpr int ld = MsCfg<S>::W + 1;   // fixed stride: immediate smem offsets in the warp ops
  S* Hw = (S*)smem_raw;                 // nw rows x nw columns (stride ld)
  S* Zw = Hw + (size_t)ld * MsCfg<S>::W;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
#define HW(i, j) Hw[(i) + (j) * ld]
#define ZW(i, j) Zw[(i) + (j) * ld]
  constexpr int WW = MsCfg<S>::W;
  if (nt % WW == 0 && nt / WW >= 4) {  // thread (row i, column class jc): <= 32 loads in flight
    const int i = tid % WW, jc = tid / WW, cs = nt / WW;
    S v[32];
#pragma unroll
    for (int k = 0; k < 32; k++) {
      const int j = jc + cs * k;
      v[k] = (i < nw && j < nw) ? H[(ws + i) + (size_t)(ws + j) * ldh] : S(0);
    }
#pragma unroll
    for (int k = 0; k < 32; k++) {
      const int j = jc + cs * k;
      if (i < nw && j < nw) { HW(i, j) = v[k]; ZW(i, j) = (i == j) ? S(1) : S(0); }
    }
  } else {
    for (int e = tid; e < nw * nw; e += nt) {
      int i = e % nw, j = e / nw;
      HW(i, j) = H[(ws + i) + (size_t)(ws + j) * ldh];
      ZW(i, j) = (i == j) ? S(1) : S(0);
    }
  }
  __syncthreads();
  const int j = warp;  // bulge handled by this warp
  for (int t = t0; t < t1; t++) {
    const int p = lo - 1 + t - 4 * j;  // global position
    const bool act = (j < nb) && (p >= lo - 1) && (p <= hi - 2);
    S tau = S(0), v1 = S(0), v2 = S(0), beta = S(0);
    const int pl = p - ws;  // window-local position
    const int nr = (hi - p) >= 3 ? 3 : 2;
    if (act) {
      S x0, x1, x2;
      if (p == lo - 1) {
        const R* w4 = shifts + 4 * j;
        const int l = lo - ws;
        shift_poly<S>(HW(l, l), HW(l + 1, l), HW(l, l + 1), HW(l + 1, l + 1), (lo + 2 <= hi) ? HW(l + 2, l + 1) : S(0),
                      w4, x0, x1, x2);
      } else {
        x0 = HW(pl + 1, pl); x1 = HW(pl + 2, pl); x2 = nr > 2 ? HW(pl + 3, pl) : S(0);
      }
      refl3_fast(nr, x0, x1, x2, beta, tau, v1, v2);
      __syncwarp();
      if (!iszero(tau)) {
        constexpr int NI = (MsCfg<S>::W + 31) / 32;
        if constexpr (kFixedTrip<S>) {
          if (nr == 3) wl3u<S, ld, NI>(Hw, pl + 1, pl + 1, nw - 1, conj(tau), v1, v2, lane);
          else wl2u<S, ld, NI>(Hw, pl + 1, pl + 1, nw - 1, conj(tau), v1, lane);
        } else {
          if (nr == 3) wl3<S, ld>(Hw, pl + 1, pl + 1, nw - 1, conj(tau), v1, v2, lane);
          else wl2<S, ld>(Hw, pl + 1, pl + 1, nw - 1, conj(tau), v1, lane);
        }
      }
      if (p >= lo && lane == 0) {
        HW(pl + 1, pl) = beta;
        HW(pl + 2, pl) = S(0);
        if (nr > 2) HW(pl + 3, pl) = S(0);
      }
    }
    __syncthreads();
    if (act && !iszero(tau)) {
      // rows of H touched: window rows 0..min(p+4,hi); rows of Z that can be nonzero:
      // 0..(position of bulge 0 + 3) -- bulge 0 leads the chain, even after it left at the
      // bottom, and every row beyond it is still an identity row of Z
      const int rmax = ((p + 4 < hi) ? p + 4 : hi) - ws;
      const int zmax = min(nw - 1, (lo - 1 + t) - ws + 3);
      constexpr int NI = (MsCfg<S>::W + 31) / 32;
      if constexpr (kFixedTrip<S>) {
        if (nr == 3) wr3u2<S, ld, NI>(Hw, rmax, Zw, zmax, pl + 1, tau, v1, v2, lane);
        else wr2u2<S, ld, NI>(Hw, rmax, Zw, zmax, pl + 1, tau, v1, lane);
      } else if (nr == 3) {
        wr3<S, ld>(Hw, pl + 1, 0, rmax, tau, v1, v2, lane);
        wr3<S, ld>(Zw, pl + 1, 0, zmax, tau, v1, v2, lane);
      } else {
        wr2<S, ld>(Hw, pl + 1, 0, rmax, tau, v1, lane);
        wr2<S, ld>(Zw, pl + 1, 0, zmax, tau, v1, lane);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < nw * nw; e += nt) {
    int i = e % nw, jj = e / nw;
    H[(ws + i) + (size_t)(ws + jj) * ldh] = HW(i, jj);
    Zg[i + (size_t)jj * nw] = ZW(i, jj);
  }
#undef HW
#undef ZW
}

// ---------------------------------------------------------------------------
// fp32 window chase on a CTA pair (thread-block cluster of 2).  The accumulated factor Z never
// feeds back into the chase, so it moves to the partner CTA: rank 0 keeps the H window and, per
// step, posts each bulge's reflector into the partner's shared memory (DSMEM) and raises a step
// counter there; rank 1 replays the reflectors onto its Z (rows contiguous, one float4 per lane
// covers the 128 rows of a column) one step behind.  The chaser sheds a third of its
// shared-memory traffic and instructions, the pair finishes when the last step is replayed.
#ifndef MSY_CHASE2
#define MSY_CHASE2 1
#endif
constexpr int CZ_LD = 132, CZ_W = 128, CZ_NB = 16, CZ_THREADS = 32 * (CZ_NB + 1);
constexpr int CZ_STEPS = CZ_W + 4 * CZ_NB;  // a window holds at most W + 4 (nb - 1) steps (the last one of a sweep)
struct __align__(16) ChaseRec { float tau, v1, v2; int nr; };
static size_t chase2_smem() {
  const size_t a = (size_t)(CZ_W + 1) * CZ_W * sizeof(float);
  const size_t b = (size_t)CZ_W * CZ_LD * sizeof(float) + (size_t)CZ_STEPS * CZ_NB * sizeof(ChaseRec) + 16;
  return a > b ? a : b;
}
// H-only right application (rows 0..rH of columns c0..c0+2), fixed trip, loads first
template <int LD, int NI>
__device__ __forceinline__ void wr3h(float* H, int rH, int c0, float tau, float v1, float v2, int lane) {
  float* ph = H + c0 * LD + lane;
  float a0[NI], a1[NI], a2[NI];
#pragma unroll
  for (int k = 0; k < NI; k++)
    if (lane + 32 * k <= rH) { a0[k] = ph[32 * k]; a1[k] = ph[32 * k + LD]; a2[k] = ph[32 * k + 2 * LD]; }
#pragma unroll
  for (int k = 0; k < NI; k++)
    if (lane + 32 * k <= rH) {
      const float w = tau * fmaf(a2[k], v2, fmaf(a1[k], v1, a0[k]));
      ph[32 * k] = a0[k] - w;
      ph[32 * k + LD] = a1[k] - w * v1;
      ph[32 * k + 2 * LD] = a2[k] - w * v2;
    }
}
template <int LD, int NI>
__device__ __forceinline__ void wr2h(float* H, int rH, int c0, float tau, float v1, int lane) {
  float* ph = H + c0 * LD + lane;
  float a0[NI], a1[NI];
#pragma unroll
  for (int k = 0; k < NI; k++)
    if (lane + 32 * k <= rH) { a0[k] = ph[32 * k]; a1[k] = ph[32 * k + LD]; }
#pragma unroll
  for (int k = 0; k < NI; k++)
    if (lane + 32 * k <= rH) {
      const float w = tau * fmaf(a1[k], v1, a0[k]);
      ph[32 * k] = a0[k] - w;
      ph[32 * k + LD] = a1[k] - w * v1;
    }
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CZ_THREADS)
    chase2_kernel(float* H, int ldh, int lo, int hi, int nb, const ChaseJobs<float> jobs) {
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  const int rank = (int)cl.block_rank(), job = blockIdx.x >> 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ws = jobs.ws[job], we = jobs.we[job], t0 = jobs.t0[job], t1 = jobs.t1[job];
  const int nw = we - ws;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // partner-side layout (rank 1's shared memory; rank 0 only forms remote addresses from it)
  float* Zw = (float*)smem_raw;                                       // CZ_W columns, stride CZ_LD
  ChaseRec* recs = (ChaseRec*)(Zw + CZ_W * CZ_LD);                    // [step][bulge]
  int* flag = (int*)(recs + CZ_STEPS * CZ_NB);                            // steps posted so far
  if (rank == 1) {
    for (int e = tid; e < CZ_W * CZ_LD; e += CZ_THREADS) {
      const int i = e % CZ_LD, jj = e / CZ_LD;
      Zw[e] = (i == jj) ? 1.f : 0.f;
    }
    if (tid == 0) *flag = 0;
    __syncthreads();
    cl.sync();
    const int j = warp;
    for (int t = t0; t < t1; t++) {
      if (tid == 0) {
        volatile int* f = flag;
        while (*f < t - t0 + 1) {}
        __threadfence();
      }
      __syncthreads();
      if (j < nb) {
        const ChaseRec r = recs[(t - t0) * CZ_NB + j];
        if (r.tau != 0.f) {
          const int pl = lo - 1 + t - 4 * j - ws;
          const int zmax = min(nw - 1, (lo - 1 + t) - ws + 3);
          if (4 * lane <= zmax) {  // rows beyond zmax hold zeros in these columns: left as they are
            float* pz = Zw + (pl + 1) * CZ_LD + 4 * lane;
            const float4 z0 = *reinterpret_cast<const float4*>(pz);
            const float4 z1 = *reinterpret_cast<const float4*>(pz + CZ_LD);
            if (r.nr == 3) {
              const float4 z2 = *reinterpret_cast<const float4*>(pz + 2 * CZ_LD);
              float4 w;
              w.x = r.tau * fmaf(z2.x, r.v2, fmaf(z1.x, r.v1, z0.x));
              w.y = r.tau * fmaf(z2.y, r.v2, fmaf(z1.y, r.v1, z0.y));
              w.z = r.tau * fmaf(z2.z, r.v2, fmaf(z1.z, r.v1, z0.z));
              w.w = r.tau * fmaf(z2.w, r.v2, fmaf(z1.w, r.v1, z0.w));
              *reinterpret_cast<float4*>(pz) = make_float4(z0.x - w.x, z0.y - w.y, z0.z - w.z, z0.w - w.w);
              *reinterpret_cast<float4*>(pz + CZ_LD) =
                  make_float4(z1.x - w.x * r.v1, z1.y - w.y * r.v1, z1.z - w.z * r.v1, z1.w - w.w * r.v1);
              *reinterpret_cast<float4*>(pz + 2 * CZ_LD) =
                  make_float4(z2.x - w.x * r.v2, z2.y - w.y * r.v2, z2.z - w.z * r.v2, z2.w - w.w * r.v2);
            } else {
              float4 w;
              w.x = r.tau * fmaf(z1.x, r.v1, z0.x);
              w.y = r.tau * fmaf(z1.y, r.v1, z0.y);
              w.z = r.tau * fmaf(z1.z, r.v1, z0.z);
              w.w = r.tau * fmaf(z1.w, r.v1, z0.w);
              *reinterpret_cast<float4*>(pz) = make_float4(z0.x - w.x, z0.y - w.y, z0.z - w.z, z0.w - w.w);
              *reinterpret_cast<float4*>(pz + CZ_LD) =
                  make_float4(z1.x - w.x * r.v1, z1.y - w.y * r.v1, z1.z - w.z * r.v1, z1.w - w.w * r.v1);
            }
          }
        }
      }
    }
    __syncthreads();
    // Z goes out with a 16-bit map of its nonzero 32 x 32 blocks (bit 4 (i / 32) + j / 32): entries
    // no reflector reached are exact zeros (about half of Z), and the far application skips them
    float* Zg = jobs.Z[job];
    __shared__ unsigned s_zmask;
    if (tid == 0) s_zmask = 0u;
    __syncthreads();
    unsigned bits = 0u;
    for (int e = tid; e < nw * nw; e += CZ_THREADS) {
      const int i = e % nw, jj = e / nw;
      const float z = Zw[i + jj * CZ_LD];
      Zg[i + (size_t)jj * nw] = z;
      if (z != 0.f) bits |= 1u << (4 * (i >> 5) + (jj >> 5));
    }
    float* ZgT = Zg + ZT_DELTA;  // row-major copy: the far application stages it with 16-byte copies
    for (int e = tid; e < nw * nw; e += CZ_THREADS) {
      const int o = e % nw, k = e / nw;
      ZgT[e] = Zw[k + o * CZ_LD];
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (lane == 0 && bits) atomicOr(&s_zmask, bits);
    __syncthreads();
    if (tid == 0) reinterpret_cast<unsigned*>(Zg)[ZMASK_OFF] = s_zmask;
    return;
  }
  // ---- rank 0: the chase proper (H window only) ----
  const float* __restrict__ shifts = jobs.shifts[job];
  constexpr int ld = CZ_W + 1;
  float* Hw = (float*)smem_raw;
#define HW(i, j) Hw[(i) + (j) * ld]
  if (tid < 4 * CZ_W) {  // thread (row i, column class jc): 32 loads in flight
    const int i = tid % CZ_W, jc = tid / CZ_W;
    float v[32];
#pragma unroll
    for (int k = 0; k < 32; k++) {
      const int jj = jc + 4 * k;
      v[k] = (i < nw && jj < nw) ? H[(ws + i) + (size_t)(ws + jj) * ldh] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 32; k++) {
      const int jj = jc + 4 * k;
      if (i < nw && jj < nw) HW(i, jj) = v[k];
    }
  }
  ChaseRec* recs_r = cl.map_shared_rank(recs, 1);
  int* flag_r = cl.map_shared_rank(flag, 1);
  __syncthreads();
  cl.sync();  // the partner runs and has cleared its step counter
  const int j = warp;  // bulge handled by this warp (warp CZ_NB: the signalling warp)
  constexpr int NI = CZ_W / 32;
  for (int t = t0; t < t1; t++) {
    const int p = lo - 1 + t - 4 * j;
    const bool act = (j < nb) && (p >= lo - 1) && (p <= hi - 2);
    float tau = 0.f, v1 = 0.f, v2 = 0.f, beta = 0.f;
    const int pl = p - ws;
    const int nr = (hi - p) >= 3 ? 3 : 2;
    if (act) {
      float x0, x1, x2;
      if (p == lo - 1) {
        const int l = lo - ws;
        shift_poly<float>(HW(l, l), HW(l + 1, l), HW(l, l + 1), HW(l + 1, l + 1), (lo + 2 <= hi) ? HW(l + 2, l + 1) : 0.f,
                          shifts + 4 * j, x0, x1, x2);
      } else {
        x0 = HW(pl + 1, pl); x1 = HW(pl + 2, pl); x2 = nr > 2 ? HW(pl + 3, pl) : 0.f;
      }
      refl3_fast(nr, x0, x1, x2, beta, tau, v1, v2);
      __syncwarp();
    }
    if (j < nb && lane == 0) {
      ChaseRec r;
      r.tau = tau; r.v1 = v1; r.v2 = v2; r.nr = nr;
      recs_r[(t - t0) * CZ_NB + j] = r;
    }
    if (act) {
      if (tau != 0.f) {
        if (nr == 3) wl3u<float, ld, NI>(Hw, pl + 1, pl + 1, nw - 1, tau, v1, v2, lane);
        else wl2u<float, ld, NI>(Hw, pl + 1, pl + 1, nw - 1, tau, v1, lane);
      }
      if (p >= lo && lane == 0) {
        HW(pl + 1, pl) = beta;
        HW(pl + 2, pl) = 0.f;
        if (nr > 2) HW(pl + 3, pl) = 0.f;
      }
    }
    named_bar(1, CZ_THREADS);  // bulge warps + the signalling warp
    if (warp == CZ_NB) {
      if (lane == 0) {  // every reflector of step t was posted before the barrier
        __threadfence();
        *(volatile int*)flag_r = t - t0 + 1;
      }
      continue;  // the fence stays off the bulge warps' second barrier
    }
    if (act && tau != 0.f) {
      const int rmax = ((p + 4 < hi) ? p + 4 : hi) - ws;
      if (nr == 3) wr3h<ld, NI>(Hw, rmax, pl + 1, tau, v1, v2, lane);
      else wr2h<ld, NI>(Hw, rmax, pl + 1, tau, v1, lane);
    }
    named_bar(2, 32 * CZ_NB);
  }
  __syncthreads();
  for (int e = tid; e < nw * nw; e += CZ_THREADS) {
    const int i = e % nw, jj = e / nw;
    H[(ws + i) + (size_t)(ws + jj) * ldh] = HW(i, jj);
  }
#undef HW
}
template <class S>
constexpr bool kChase2 = std::is_same<S, float>::value && MSY_CHASE2 != 0 && MsCfg<S>::W == CZ_W && MsCfg<S>::NB <= CZ_NB;

// ---------------------------------------------------------------------------
// in-place application of a small orthogonal Z (nz x nz, ld nz, nz <= ZMAX):
//   region L: H[r0:r0+nz, cL0:cL1] <- Z^H * (.)       (tiles of 32 columns)
//   region R: H[0:rR1, r0:r0+nz]   <- (.) * Z          (tiles of 32 rows)
//   region U: U[0:mU, r0:r0+nz]    <- (.) * Z
template <class S>
__device__ __forceinline__ void apply_z_block(int b, unsigned char* smem_raw, int nz, const S* __restrict__ Zg, S* H,
                                              int ldh, int r0, int cL0, int cL1, int rlo, int rR1, S* U, int ldu,
                                              int mU) {
  constexpr int ZA = ZMAX / 32;
  const int ldz = nz + 1;
  S* Zs = (S*)smem_raw;
  S* Ts = Zs + (size_t)ldz * nz;
  const int tid = threadIdx.x;
  const int ntL = cL1 > cL0 ? cdiv(cL1 - cL0, 32) : 0, ntR = rR1 > rlo ? cdiv(rR1 - rlo, 32) : 0,
            ntU = cdiv(mU, 32);
  for (int e = tid; e < nz * nz; e += 256) Zs[(e % nz) + (e / nz) * ldz] = Zg[e];
  if (b < ntL) {
    const int c0 = cL0 + b * 32, nc = min(32, cL1 - c0);
    const int ldt = nz + 1;  // Ts[r + c*ldt], nz rows x 32 columns
    for (int e = tid; e < nz * 32; e += 256) {
      int r = e % nz, c = e / nz;
      Ts[r + c * ldt] = c < nc ? H[(r0 + r) + (size_t)(c0 + c) * ldh] : S(0);
    }
    __syncthreads();
    // out[i, c] = sum_r conj(Z[r, i]) T[r, c]; thread: rows i = tr + 32a, cols c = 4 tc + q
    const int tr_ = tid & 31, tc = tid >> 5;
    S acc[ZA][4];
#pragma unroll
    for (int a = 0; a < ZA; a++)
#pragma unroll
      for (int q = 0; q < 4; q++) acc[a][q] = S(0);
    for (int r = 0; r < nz; r++) {
      S z[ZA], t[4];
#pragma unroll
      for (int a = 0; a < ZA; a++) { int i = tr_ + 32 * a; z[a] = i < nz ? conj(Zs[r + i * ldz]) : S(0); }
#pragma unroll
      for (int q = 0; q < 4; q++) t[q] = Ts[r + (4 * tc + q) * ldt];
#pragma unroll
      for (int a = 0; a < ZA; a++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[a][q] = fmac(z[a], t[q], acc[a][q]);
    }
#pragma unroll
    for (int a = 0; a < ZA; a++) {
      int i = tr_ + 32 * a;
      if (i >= nz) continue;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        int c = 4 * tc + q;
        if (c < nc) H[(r0 + i) + (size_t)(c0 + c) * ldh] = acc[a][q];
      }
    }
    return;
  }
  b -= ntL;
  S* M;
  int ldm, rbase, nrows;
  if (b < ntR) { M = H; ldm = ldh; rbase = rlo + b * 32; nrows = min(32, rR1 - rbase); }
  else { b -= ntR; if (b >= ntU) return; M = U; ldm = ldu; rbase = b * 32; nrows = min(32, mU - rbase); }
  for (int e = tid; e < 32 * nz; e += 256) {
    int r = e % 32, c = e / 32;
    Ts[r + c * 32] = r < nrows ? M[(rbase + r) + (size_t)(r0 + c) * ldm] : S(0);
  }
  __syncthreads();
  // out[r, j] = sum_i T[r, i] Z[i, j]; thread: rows r = 4g + q, cols j = lane + 32a
  const int lane = tid & 31, g = tid >> 5;
  S acc[ZA][4];
#pragma unroll
  for (int a = 0; a < ZA; a++)
#pragma unroll
    for (int q = 0; q < 4; q++) acc[a][q] = S(0);
  for (int i = 0; i < nz; i++) {
    S z[ZA], t[4];
#pragma unroll
    for (int a = 0; a < ZA; a++) { int jj = lane + 32 * a; z[a] = jj < nz ? Zs[i + jj * ldz] : S(0); }
#pragma unroll
    for (int q = 0; q < 4; q++) t[q] = Ts[(4 * g + q) + i * 32];
#pragma unroll
    for (int a = 0; a < ZA; a++)
#pragma unroll
      for (int q = 0; q < 4; q++) acc[a][q] = fmac(t[q], z[a], acc[a][q]);
  }
#pragma unroll
  for (int q = 0; q < 4; q++) {
    int r = 4 * g + q;
    if (r >= nrows) continue;
#pragma unroll
    for (int a = 0; a < ZA; a++) {
      int jj = lane + 32 * a;
      if (jj < nz) M[(rbase + r) + (size_t)(r0 + jj) * ldm] = acc[a][q];
    }
  }
}

template <class S>
__global__ void __launch_bounds__(256) apply_z_kernel(int nz, const S* __restrict__ Zg, S* H, int ldh, int r0,
                                                      int cL0, int cL1, int rR1, S* U, int ldu, int mU) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  apply_z_block<S>(blockIdx.x, smem_raw, nz, Zg, H, ldh, r0, cL0, cL1, 0, rR1, U, ldu, mU);
}

// several windows' applications in one launch (disjoint regions; blocks [start[j], start[j+1]) -> job j)
template <class S>
struct ApplyJobs {
  int n;
  int start[KMAX + 1], nz[KMAX], r0[KMAX], cL0[KMAX], cL1[KMAX], rlo[KMAX], rR1[KMAX], mU[KMAX];
  const S* Z[KMAX];
  int zmask[KMAX];  // 1: Z[j] carries a nonzero-block map at ZMASK_OFF (factors written by chase2_kernel)
};
// algorithmic flops of one apply_z_multi launch
template <class S>
double applyz_flops(const ApplyJobs<S>& j) {
  double f = 0;
  for (int i = 0; i < j.n; i++)
    f += (double)j.nz[i] * j.nz[i] * ((j.cL1[i] > j.cL0[i] ? j.cL1[i] - j.cL0[i] : 0) +
                                      (j.rR1[i] > j.rlo[i] ? j.rR1[i] - j.rlo[i] : 0) + j.mU[i]);
  return (tr<S>::cx ? 8.0 : 2.0) * f;
}
template <class S>
__global__ void __launch_bounds__(256) apply_z_multi_kernel(S* H, int ldh, S* U, int ldu, const ApplyJobs<S> jobs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int j = 0;
  while (j + 1 < jobs.n && (int)blockIdx.x >= jobs.start[j + 1]) j++;
  apply_z_block<S>(blockIdx.x - jobs.start[j], smem_raw, jobs.nz[j], jobs.Z[j], H, ldh, jobs.r0[j], jobs.cL0[j],
                   jobs.cL1[j], jobs.rlo[j], jobs.rR1[j], U, ldu, jobs.mU[j]);
}

// ---------------------------------------------------------------------------
// Z application split over a thread-block cluster: the 32-column (region L) or 32-row
// (regions R, U) tile of a job is shared by the AZC CTAs of one cluster, each producing
// 32 of the nz output rows (L) / columns (R, U) from its 32-wide slice of Z.  Every CTA
// stages the whole nz-deep input tile before the cluster barrier, so the in-place writes
// that follow cannot race with a sibling's reads.  Five times the CTAs of apply_z_multi
// for the same region, each with a 40 KB footprint (several CTAs per SM): the near-window
// applications on the sweep's critical path finish in a fraction of the time.
template <class S> struct Azc { static constexpr int N = (MsCfg<S>::W + 31) / 32; };  // CTAs per cluster
constexpr int AZC_THREADS = 128, AZC_TP = 33, AZC_CP = 36;
template <class S>
static size_t azc_smem() { return (size_t)MsCfg<S>::W * (AZC_TP + AZC_CP) * sizeof(S); }
template <class S>
__global__ void __cluster_dims__(Azc<S>::N, 1, 1) __launch_bounds__(AZC_THREADS)
    apply_z_cl_kernel(S* H, int ldh, S* U, int ldu, const ApplyJobs<S> jobs) {
  constexpr int TP = AZC_TP, CP = AZC_CP;  // smem strides: input tile [k][32] (TP), Z slice [k][32] (CP)
  constexpr int AZC = Azc<S>::N;
  extern __shared__ __align__(16) unsigned char azc_raw[];
  S* Ts = (S*)azc_raw;
  S* Zc = Ts + MsCfg<S>::W * TP;
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  const int part = (int)cl.block_rank();
  int b = blockIdx.x / AZC;
  int j = 0;
  while (j + 1 < jobs.n && b >= jobs.start[j + 1]) j++;
  b -= jobs.start[j];
  const int nz = jobs.nz[j], r0 = jobs.r0[j];
  const S* __restrict__ Zg = jobs.Z[j];
  const int cL0 = jobs.cL0[j], cL1 = jobs.cL1[j], rlo = jobs.rlo[j], rR1 = jobs.rR1[j], mU = jobs.mU[j];
  const int ntL = cL1 > cL0 ? cdiv(cL1 - cL0, 32) : 0, ntR = rR1 > rlo ? cdiv(rR1 - rlo, 32) : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int o0 = part * 32;                 // this CTA's output slice
  const int no = min(32, nz - o0);          // <= 0: nothing to write (still joins the barrier)
  static_assert(MsCfg<S>::W <= AZC_THREADS, "one staged row per thread");
  // slice of Z: columns o0..o0+no-1 (L uses conj(Z[k, o]), R/U use Z[k, o]).  Thread k stages
  // row k: 32 independent coalesced loads in flight, then 32 shared stores.
  if (tid < nz) {
    S v[32];
#pragma unroll
    for (int o = 0; o < 32; o++) v[o] = o < no ? Zg[tid + (size_t)(o0 + o) * nz] : S(0);
#pragma unroll
    for (int o = 0; o < 32; o++) Zc[tid * CP + o] = v[o];
  }
  if (b < ntL) {  // ---- region L: H[r0 + o, c] <- sum_k conj(Z[k, o]) H[r0 + k, c] ----
    const int c0 = cL0 + b * 32, nc = min(32, cL1 - c0);
    if (tid < nz) {
      S v[32];
#pragma unroll
      for (int c = 0; c < 32; c++) v[c] = c < nc ? H[(r0 + tid) + (size_t)(c0 + c) * ldh] : S(0);
#pragma unroll
      for (int c = 0; c < 32; c++) Ts[tid * TP + c] = v[c];
    }
    cl.sync();
    if (no > 0) {
      S acc[8];
#pragma unroll
      for (int q = 0; q < 8; q++) acc[q] = S(0);
      for (int k = 0; k < nz; k++) {
        const S t = Ts[k * TP + lane];
        const S* zr = Zc + k * CP + warp * 8;
#pragma unroll
        for (int q = 0; q < 8; q++) acc[q] = fmacc(zr[q], t, acc[q]);
      }
      if (lane < nc)
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const int o = warp * 8 + q;
          if (o < no) H[(r0 + o0 + o) + (size_t)(c0 + lane) * ldh] = acc[q];
        }
    }
    return;
  }
  b -= ntL;
  S* M;
  int ldm, rbase, nrows;
  if (b < ntR) { M = H; ldm = ldh; rbase = rlo + b * 32; nrows = min(32, rR1 - rbase); }
  else { b -= ntR; M = U; ldm = ldu; rbase = b * 32; nrows = min(32, mU - rbase); }
  // ---- regions R / U: M[r, r0 + o] <- sum_k M[r, r0 + k] Z[k, o] ----
  {  // thread (r = lane, k = warp + 4 i): coalesced along r, nz / 4 independent loads per thread
    constexpr int KI = (MsCfg<S>::W + 3) / 4;
    S v[KI];
#pragma unroll
    for (int i = 0; i < KI; i++) {
      const int k = warp + 4 * i;
      v[i] = (k < nz && lane < nrows) ? M[(rbase + lane) + (size_t)(r0 + k) * ldm] : S(0);
    }
#pragma unroll
    for (int i = 0; i < KI; i++) {
      const int k = warp + 4 * i;
      if (k < nz) Ts[k * TP + lane] = v[i];
    }
  }
  cl.sync();
  if (no <= 0) return;
  S acc[8];
#pragma unroll
  for (int q = 0; q < 8; q++) acc[q] = S(0);
  for (int k = 0; k < nz; k++) {
    const S t = Ts[k * TP + lane];
    const S* zr = Zc + k * CP + warp * 8;
#pragma unroll
    for (int q = 0; q < 8; q++) acc[q] = fmac(t, zr[q], acc[q]);
  }
  if (lane < nrows)
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int o = warp * 8 + q;
      if (o < no) M[(rbase + lane) + (size_t)(r0 + o0 + o) * ldm] = acc[q];
    }
}

// ---------------------------------------------------------------------------
// Throughput-oriented Z application for the FAR regions of real fp32 sweeps (the parts of the
// rows right of / columns above a window, and U, that the next chase does not wait for).
// One CTA owns a 64-wide tile with the full nz-deep contraction (in place: the input tile is
// staged in smem before any output is written), 256 threads with an 8 x 4 register tile each:
// per contraction step two LDS.128 of the row-major Z copy and four scalar / one LDS.128 of
// the input tile feed 32 FFMAs (the cluster kernel above: 3 loads per 8 FFMAs and a 4x
// redundant input read -- it stays the low-latency path for the near regions).  Outputs go
// through smem so that global stores are warp-contiguous.
constexpr int AZF_THREADS = 256, AZF_TILE = 64, AZF_W = 128, AZF_LDZ = 132, AZF_LDT = 65, AZF_LDC = 68;
constexpr int AZF_TS = 128 * 68;  // floats of the tile / output staging buffer (>= 64 * 132, 128 * 65, 128 * 68)
#ifndef MSY_FAR_BULK
#define MSY_FAR_BULK 1   // far application: cp.async.bulk + mbarrier for full tiles
#endif
#ifndef MSY_FAR_ZT
#define MSY_FAR_ZT 1     // far application: 16-byte copies (row-major Z copy of chase2, aligned row groups of R / U tiles)
#endif
#ifndef MSY_FAR_ZMASK
#define MSY_FAR_ZMASK 1  // far application skips the zero 32 x 32 blocks of the chase2 window factors
#endif
#ifndef MSY_FAR_PAD
#define MSY_FAR_PAD 0  // extra dynamic smem (bytes): > 11 KB leaves one far CTA per SM
#endif
static size_t azf_smem() { return (size_t)(AZF_W * AZF_LDZ + AZF_TS) * sizeof(float) + MSY_FAR_PAD; }
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)), "l"(gsrc) : "memory");
}
// ---- bulk asynchronous copies (the TMA engine's linear form, cp.async.bulk) with an mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mbar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(mbar)), "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, unsigned bytes, unsigned long long* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__global__ void __launch_bounds__(AZF_THREADS, 2)
    apply_z_far_kernel(float* H, int ldh, float* U, int ldu, const ApplyJobs<float> jobs) {
  extern __shared__ __align__(16) unsigned char azf_raw[];
  float* Zs = (float*)azf_raw;         // Zs[k * LDZ + o] = Z[k, o], zero beyond nz
  float* Ts = Zs + AZF_W * AZF_LDZ;
  int b = blockIdx.x;
  int j = 0;
  while (j + 1 < jobs.n && b >= jobs.start[j + 1]) j++;
  b -= jobs.start[j];
  const int nz = jobs.nz[j], r0 = jobs.r0[j];
  const float* __restrict__ Zg = jobs.Z[j];
  const int cL0 = jobs.cL0[j], cL1 = jobs.cL1[j], rlo = jobs.rlo[j], rR1 = jobs.rR1[j], mU = jobs.mU[j];
  const int ntL = cL1 > cL0 ? cdiv(cL1 - cL0, AZF_TILE) : 0, ntR = rR1 > rlo ? cdiv(rR1 - rlo, AZF_TILE) : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Z, transposed on the way in, and the input tile below: 4-byte cp.async (LDGSTS) per element,
  // every copy of the CTA in flight at once (a register-staged loop was latency-bound: 25 of the
  // 31 us a tile took)
  // Full tiles of chase2 factors move with bulk asynchronous copies (cp.async.bulk, the TMA engine):
  // one 512-byte row of the row-major Z copy and one 256-byte column of an R / U tile per thread,
  // completion on an mbarrier; ragged tiles and region L keep the cp.async paths below.
  __shared__ __align__(8) unsigned long long mbar;
  const bool bulkz = MSY_FAR_BULK && MSY_FAR_ZT && jobs.zmask[j] && nz == AZF_W;
  bool bulkt = false;
  {
    int bb = b - ntL;
    if (bulkz && bb >= 0) {
      const float* Mb; int ldb, rb, nr;
      if (bb < ntR) { Mb = H; ldb = ldh; rb = rlo + bb * AZF_TILE; nr = min(AZF_TILE, rR1 - rb); }
      else { bb -= ntR; Mb = U; ldb = ldu; rb = bb * AZF_TILE; nr = min(AZF_TILE, mU - rb); }
      bulkt = nr == AZF_TILE && (ldb & 3) == 0 && (rb & 3) == 0 && (reinterpret_cast<uintptr_t>(Mb) & 15) == 0;
    }
  }
  if (bulkz) {
    if (tid == 0) {
      mbar_init(&mbar, 1);
      mbar_expect_tx(&mbar, (unsigned)(AZF_W * AZF_W * sizeof(float)) + (bulkt ? (unsigned)(AZF_W * AZF_TILE * sizeof(float)) : 0u));
    }
    __syncthreads();
    if (tid < AZF_W) bulk_g2s(&Zs[tid * AZF_LDZ], Zg + ZT_DELTA + (size_t)tid * AZF_W, AZF_W * sizeof(float), &mbar);
  } else if (MSY_FAR_ZT && jobs.zmask[j] && (nz & 3) == 0) {  // chase2 factor: its row-major copy, 16 bytes per copy
    const float* __restrict__ ZT = Zg + ZT_DELTA;
    for (int e = tid; e < AZF_W * (AZF_W / 4); e += AZF_THREADS) {
      const int k = e >> 5, o4 = (e & 31) * 4;
      if (k < nz && o4 < nz) cp_async16(&Zs[k * AZF_LDZ + o4], &ZT[(size_t)k * nz + o4]);
      else *reinterpret_cast<float4*>(&Zs[k * AZF_LDZ + o4]) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    for (int e = tid; e < AZF_W * AZF_W; e += AZF_THREADS) {
      const int k = e & 127, o = e >> 7;
      if (k < nz && o < nz) cp_async4(&Zs[k * AZF_LDZ + o], &Zg[k + (size_t)o * nz]);
      else Zs[k * AZF_LDZ + o] = 0.f;
    }
  }
  // warp -> (output half h, group of 16 tile columns / rows cq); lane -> (ig, cg)
  const int h = warp & 1, cq = warp >> 1, ig = lane & 7, cg = lane >> 3;
  const int oa = h * 64 + ig * 4, ob = oa + 32, tb = cq * 16 + cg * 4;
  const unsigned zbits = (MSY_FAR_ZMASK && jobs.zmask[j]) ? reinterpret_cast<const unsigned*>(Zg)[ZMASK_OFF] : 0xffffu;
  float acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; a++)
#pragma unroll
    for (int q = 0; q < 4; q++) acc[a][q] = 0.f;
  if (b < ntL) {  // ---- region L: H[r0 + o, c] <- sum_k Z[k, o] H[r0 + k, c] ----
    const int c0 = cL0 + b * AZF_TILE, nc = min(AZF_TILE, cL1 - c0);
    for (int e = tid; e < AZF_W * AZF_TILE; e += AZF_THREADS) {  // lanes along k: coalesced, conflict-free
      const int k = e & 127, c = e >> 7;
      if (k < nz && c < nc) cp_async4(&Ts[k * AZF_LDT + c], &H[(r0 + k) + (size_t)(c0 + c) * ldh]);
      else Ts[k * AZF_LDT + c] = 0.f;
    }
    cp_async_wait_all();
    if (bulkz) mbar_wait(&mbar, 0);
    __syncthreads();
    for (int kb = 0; kb < 4; kb++) {  // 32-deep slices of the contraction; zero blocks of Z skipped
      const int fa = (zbits >> (4 * kb + 2 * h)) & 1, fb = (zbits >> (4 * kb + 2 * h + 1)) & 1;
      const int k1 = min(nz, 32 * kb + 32);
      if (fa && fb) {
#pragma unroll 4
        for (int k = 32 * kb; k < k1; k++) {
          const float4 za = *reinterpret_cast<const float4*>(&Zs[k * AZF_LDZ + oa]);
          const float4 zb = *reinterpret_cast<const float4*>(&Zs[k * AZF_LDZ + ob]);
          const float z[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
          float t[4];
#pragma unroll
          for (int q = 0; q < 4; q++) t[q] = Ts[k * AZF_LDT + tb + q];
#pragma unroll
          for (int a = 0; a < 8; a++)
#pragma unroll
            for (int q = 0; q < 4; q++) acc[a][q] = fmaf(z[a], t[q], acc[a][q]);
        }
      } else if (fa || fb) {
        const int oo = fa ? oa : ob, a0 = fa ? 0 : 4;
#pragma unroll 4
        for (int k = 32 * kb; k < k1; k++) {
          const float4 zv = *reinterpret_cast<const float4*>(&Zs[k * AZF_LDZ + oo]);
          const float z[4] = {zv.x, zv.y, zv.z, zv.w};
          float t[4];
#pragma unroll
          for (int q = 0; q < 4; q++) t[q] = Ts[k * AZF_LDT + tb + q];
          if (a0 == 0) {
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
              for (int q = 0; q < 4; q++) acc[a][q] = fmaf(z[a], t[q], acc[a][q]);
          } else {
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
              for (int q = 0; q < 4; q++) acc[4 + a][q] = fmaf(z[a], t[q], acc[4 + a][q]);
          }
        }
      }
    }
    __syncthreads();
    // outputs staged as Os[c * LDZ + o] (o contiguous, like global memory)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      *reinterpret_cast<float4*>(&Ts[(tb + q) * AZF_LDZ + oa]) = make_float4(acc[0][q], acc[1][q], acc[2][q], acc[3][q]);
      *reinterpret_cast<float4*>(&Ts[(tb + q) * AZF_LDZ + ob]) = make_float4(acc[4][q], acc[5][q], acc[6][q], acc[7][q]);
    }
    __syncthreads();
    for (int e = tid; e < AZF_W * AZF_TILE; e += AZF_THREADS) {
      const int o = e & 127, c = e >> 7;
      if (o < nz && c < nc) H[(r0 + o) + (size_t)(c0 + c) * ldh] = Ts[c * AZF_LDZ + o];
    }
    return;
  }
  b -= ntL;
  float* M;
  int ldm, rbase, nrows;
  if (b < ntR) { M = H; ldm = ldh; rbase = rlo + b * AZF_TILE; nrows = min(AZF_TILE, rR1 - rbase); }
  else { b -= ntR; M = U; ldm = ldu; rbase = b * AZF_TILE; nrows = min(AZF_TILE, mU - rbase); }
  if (nrows <= 0) {  // (cannot happen for a tile index inside the job; never leave copies in flight)
    cp_async_wait_all();
    if (bulkz) mbar_wait(&mbar, 0);
    return;
  }
  // ---- regions R / U: M[r, r0 + o] <- sum_k M[r, r0 + k] Z[k, o] ----
  const bool al16 = MSY_FAR_ZT && (ldm & 3) == 0 && (rbase & 3) == 0 && (reinterpret_cast<uintptr_t>(M) & 15) == 0;
  if (bulkt) {  // column k of the tile: 64 contiguous rows, one bulk copy
    if (tid < AZF_W) bulk_g2s(&Ts[tid * AZF_LDC], &M[rbase + (size_t)(r0 + tid) * ldm], AZF_TILE * sizeof(float), &mbar);
  } else if (al16) {  // rows in aligned groups of four: 16-byte copies (4-byte ones for a ragged last group)
    for (int e = tid; e < AZF_W * (AZF_TILE / 4); e += AZF_THREADS) {
      const int r4 = (e & 15) * 4, k = e >> 4;
      float* dst = &Ts[k * AZF_LDC + r4];
      if (k < nz && r4 + 3 < nrows) {
        cp_async16(dst, &M[(rbase + r4) + (size_t)(r0 + k) * ldm]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (k < nz && r4 + q < nrows) cp_async4(dst + q, &M[(rbase + r4 + q) + (size_t)(r0 + k) * ldm]);
          else dst[q] = 0.f;
        }
      }
    }
  } else {
    for (int e = tid; e < AZF_W * AZF_TILE; e += AZF_THREADS) {  // lanes along r: coalesced, contiguous smem
      const int r = e & 63, k = e >> 6;
      if (k < nz && r < nrows) cp_async4(&Ts[k * AZF_LDC + r], &M[(rbase + r) + (size_t)(r0 + k) * ldm]);
      else Ts[k * AZF_LDC + r] = 0.f;
    }
  }
  cp_async_wait_all();
  if (bulkz) mbar_wait(&mbar, 0);
  __syncthreads();
  for (int kb = 0; kb < 4; kb++) {
    const int fa = (zbits >> (4 * kb + 2 * h)) & 1, fb = (zbits >> (4 * kb + 2 * h + 1)) & 1;
    const int k1 = min(nz, 32 * kb + 32);
    if (fa && fb) {
#pragma unroll 4
      for (int k = 32 * kb; k < k1; k++) {
        const float4 za = *reinterpret_cast<const float4*>(&Zs[k * AZF_LDZ + oa]);
        const float4 zb = *reinterpret_cast<const float4*>(&Zs[k * AZF_LDZ + ob]);
        const float z[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
        const float4 tv = *reinterpret_cast<const float4*>(&Ts[k * AZF_LDC + tb]);
        const float t[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
        for (int a = 0; a < 8; a++)
#pragma unroll
          for (int q = 0; q < 4; q++) acc[a][q] = fmaf(t[q], z[a], acc[a][q]);
      }
    } else if (fa || fb) {
      const int oo = fa ? oa : ob, a0 = fa ? 0 : 4;
#pragma unroll 4
      for (int k = 32 * kb; k < k1; k++) {
        const float4 zv = *reinterpret_cast<const float4*>(&Zs[k * AZF_LDZ + oo]);
        const float z[4] = {zv.x, zv.y, zv.z, zv.w};
        const float4 tv = *reinterpret_cast<const float4*>(&Ts[k * AZF_LDC + tb]);
        const float t[4] = {tv.x, tv.y, tv.z, tv.w};
        if (a0 == 0) {
#pragma unroll
          for (int a = 0; a < 4; a++)
#pragma unroll
            for (int q = 0; q < 4; q++) acc[a][q] = fmaf(t[q], z[a], acc[a][q]);
        } else {
#pragma unroll
          for (int a = 0; a < 4; a++)
#pragma unroll
            for (int q = 0; q < 4; q++) acc[4 + a][q] = fmaf(t[q], z[a], acc[4 + a][q]);
        }
      }
    }
  }
  __syncthreads();
  // outputs staged as Os[o * LDC + r] (r contiguous, like global memory)
#pragma unroll
  for (int a = 0; a < 8; a++) {
    const int o = a < 4 ? oa + a : ob + (a - 4);
    *reinterpret_cast<float4*>(&Ts[o * AZF_LDC + tb]) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
  }
  if (bulkt) fence_proxy_async();  // the staged outputs become visible to the bulk-copy engine
  __syncthreads();
  if (bulkt) {  // column o of the output: one bulk store from the staging buffer
    if (tid < AZF_W) bulk_s2g(&M[rbase + (size_t)(r0 + tid) * ldm], &Ts[tid * AZF_LDC], AZF_TILE * sizeof(float));
    bulk_commit_wait_read();
  } else if (al16) {
    for (int e = tid; e < AZF_W * (AZF_TILE / 4); e += AZF_THREADS) {
      const int r4 = (e & 15) * 4, o = e >> 4;
      if (o >= nz) continue;
      float* dst = &M[(rbase + r4) + (size_t)(r0 + o) * ldm];
      const float4 v = *reinterpret_cast<const float4*>(&Ts[o * AZF_LDC + r4]);
      if (r4 + 3 < nrows) {
        *reinterpret_cast<float4*>(dst) = v;
      } else {
        if (r4 < nrows) dst[0] = v.x;
        if (r4 + 1 < nrows) dst[1] = v.y;
        if (r4 + 2 < nrows) dst[2] = v.z;
      }
    }
  } else {
    for (int e = tid; e < AZF_W * AZF_TILE; e += AZF_THREADS) {
      const int r = e & 63, o = e >> 6;
      if (o < nz && r < nrows) M[(rbase + r) + (size_t)(r0 + o) * ldm] = Ts[o * AZF_LDC + r];
    }
  }
}
// launch for a job list whose `start` was built for 32-wide tiles: rebuilt here for 64-wide ones
static int apply_z_far_launch(float* H, int ldh, float* U, int ldu, ApplyJobs<float> jb, cudaStream_t st) {
  MSY_SMEM_ATTR_ONCE(apply_z_far_kernel, (int)azf_smem());
  jb.start[0] = 0;
  for (int j = 0; j < jb.n; j++)
    jb.start[j + 1] = jb.start[j] + (jb.cL1[j] > jb.cL0[j] ? cdiv(jb.cL1[j] - jb.cL0[j], AZF_TILE) : 0) +
                      (jb.rR1[j] > jb.rlo[j] ? cdiv(jb.rR1[j] - jb.rlo[j], AZF_TILE) : 0) + cdiv(jb.mU[j], AZF_TILE);
  if (jb.start[jb.n] <= 0) return 0;
  apply_z_far_kernel<<<jb.start[jb.n], AZF_THREADS, azf_smem(), st>>>(H, ldh, U, ldu, jb);
  MSY_LAUNCH_CK();
  return 0;
}
template <class S>
constexpr bool kFarKernel = std::is_same<S, float>::value && MsCfg<S>::W <= AZF_W;

template <class S>
static size_t applyz_smem(int nz) {
  return ((size_t)(nz + 1) * nz + (size_t)(nz + 1) * 33 + 32 * (size_t)nz) * sizeof(S) + 64;
}

// Apply Z (block [w0, w0+nz)) to H rows w0.. over columns [cL0, cL1), to H rows [0, rR1)
// of the block's columns, and (if U) to all rows of U's block columns.
template <class S>
int apply_z_regions(int m, int nz, const S* Z, S* H, int ldh, S* U, int ldu, int w0, int cL0, int cL1, int rR1,
                    cudaStream_t st) {
  MSY_SMEM_ATTR_ONCE(apply_z_kernel<S>, (int)applyz_smem<S>(MsCfg<S>::W));
  if (nz > MsCfg<S>::W) return -4;
  int nblk = (cL1 > cL0 ? cdiv(cL1 - cL0, 32) : 0) + cdiv(rR1, 32) + (U ? cdiv(m, 32) : 0);
  if (nblk == 0) return 0;
  KScope ks(KC_APPLYZ, (tr<S>::cx ? 8.0 : 2.0) * nz * nz * ((cL1 > cL0 ? cL1 - cL0 : 0) + rR1 + (U ? m : 0)), st);
  constexpr int azc_mode = MSY_AZC;
  if (azc_mode >= 2) {  // the cluster-split kernel with a single job
    MSY_SMEM_ATTR_ONCE(apply_z_cl_kernel<S>, (int)azc_smem<S>());
    ApplyJobs<S> j = {};
    j.n = 1; j.start[0] = 0; j.start[1] = nblk;
    j.nz[0] = nz; j.Z[0] = Z; j.r0[0] = w0; j.cL0[0] = cL0; j.cL1[0] = cL1; j.rlo[0] = 0; j.rR1[0] = rR1;
    j.mU[0] = U ? m : 0;
    if constexpr (kFarKernel<S>) {
      if (MSY_FAR_MIN_TILES >= 0 && nblk >= MSY_FAR_MIN_TILES && nz >= 64) return apply_z_far_launch(H, ldh, U, ldu, j, st);
    }
    apply_z_cl_kernel<S><<<nblk * Azc<S>::N, AZC_THREADS, azc_smem<S>(), st>>>(H, ldh, U, ldu, j);
  } else {
    apply_z_kernel<S><<<nblk, 256, applyz_smem<S>(nz), st>>>(nz, Z, H, ldh, w0, cL0, cL1, rR1, U, ldu, U ? m : 0);
  }
  MSY_LAUNCH_CK();
  return 0;
}

// Apply Z (window [w0, w0+nz)) to everything outside the window's diagonal block.
template <class S>
int apply_z(int m, int nz, const S* Z, S* H, int ldh, S* U, int ldu, int w0, cudaStream_t st) {
  return apply_z_regions<S>(m, nz, Z, H, ldh, U, ldu, w0, w0 + nz, m, w0, st);
}

// ---------------------------------------------------------------------------
// deflation scan: zero negligible subdiagonals in [1, hi]; skip converged trailing
// blocks (1x1; real 2x2; complex 2x2 after a splitting rotation); report the
// new hi and the start lo of its unreduced block.  out[0] = hi', out[1] = lo.
template <class S>
__global__ void __launch_bounds__(1024) scan_kernel(int m, S* H, int ldh, S* U, int ldu, int hi, int* out) {
  typedef typename tr<S>::R R;
  const R u = tr<S>::u();
  __shared__ int s_i, s_act;
  const int tid = threadIdx.x, nt = blockDim.x;
#define HH(i, j) H[(i) + (size_t)(j) * ldh]
  for (int k = 1 + tid; k <= hi; k += nt) {
    S h = HH(k, k - 1);
    if (!iszero(h) && absv(h) <= u * (absv(HH(k - 1, k - 1)) + absv(HH(k, k)))) HH(k, k - 1) = S(0);
  }
  __syncthreads();
  if (tid == 0) s_i = hi;
  __syncthreads();
  while (true) {
    if (tid == 0) {
      int i = s_i;
      s_act = 0;
      while (i >= 0) {
        if (i == 0) { i = -1; break; }
        if (iszero(HH(i, i - 1))) { i -= 1; continue; }
        if (i == 1 || iszero(HH(i - 1, i - 2))) {
          if (tr<S>::cx) { s_act = 1; break; }
          i -= 2;
          continue;
        }
        break;
      }
      s_i = i;
    }
    __syncthreads();
    if (!s_act) break;
    // complex 2x2 split of [i-1, i] (see schur_small_kernel, mode 2)
    const int i = s_i, l = i - 1;
    R w4[4];
    S a = HH(l, l), b = HH(l, i), c = HH(i, l), d = HH(i, i);
    eig2<S>(a, b, c, d, w4);
    S lam = mk<S>(w4[0], w4[1]);
    S va = lam - d, vb = c, wa = b, wb = lam - a;
    if (abs2(wa) + abs2(wb) > abs2(va) + abs2(vb)) { va = wa; vb = wb; }
    R nv = sqrt(abs2(va) + abs2(vb));
    S g11 = va / mk<S>(nv), g21 = vb / mk<S>(nv);
    S g12 = -conj(g21), g22 = conj(g11);
    __syncthreads();
    for (int j = l + tid; j < m; j += nt) {
      S h1 = HH(l, j), h2 = HH(i, j);
      HH(l, j) = fmacc(g11, h1, conj(g21) * h2);
      HH(i, j) = fmacc(g12, h1, conj(g22) * h2);
    }
    __syncthreads();
    for (int e = tid; e < (i + 1) + m; e += nt) {
      S* M;
      int r;
      size_t ldx;
      if (e <= i) { M = H; r = e; ldx = ldh; } else { M = U; r = e - i - 1; ldx = ldu; }
      S c1 = M[r + l * ldx], c2 = M[r + i * ldx];
      M[r + l * ldx] = c1 * g11 + c2 * g21;
      M[r + i * ldx] = c1 * g12 + c2 * g22;
    }
    __syncthreads();
    if (tid == 0) { HH(i, l) = S(0); s_i = i - 2; }
    __syncthreads();
  }
  // lo = start of the unreduced block ending at i: block-wide max over zero subdiagonals
  __shared__ int s_lo;
  if (tid == 0) s_lo = 0;
  __syncthreads();
  const int ifin = s_i;
  int mylo = 0;
  for (int k = 1 + tid; k <= ifin; k += nt)
    if (iszero(HH(k, k - 1))) mylo = k;  // k increases with the stride: last hit is this thread's max
  if (mylo) atomicMax(&s_lo, mylo);
  __syncthreads();
  if (tid == 0) {
    out[0] = ifin;
    out[1] = ifin >= 0 ? s_lo : 0;
  }
#undef HH
}

// build per-bulge shift quadruples (sr1, si1, sr2, si2) from eigenvalues (wr, wi)
// of the trailing block; exceptional shifts from the trailing subdiagonals.
template <class S>
__global__ void pair_shifts_kernel(int ns, const typename tr<S>::R* wr, const typename tr<S>::R* wi, int nb,
                                   typename tr<S>::R* out, int exceptional, const S* H, int ldh, int lo, int hi,
                                   int* nb_out) {
  typedef typename tr<S>::R R;
  // stage the eigenvalues in shared memory first (one dependent global round trip per
  // element in the serial pairing loop otherwise)
  __shared__ R swr[256], swi[256];
  for (int k = threadIdx.x; k < ns && k < 256; k += blockDim.x) { swr[k] = wr[k]; swi[k] = wi[k]; }
  __syncthreads();
  if (ns <= 256) { wr = swr; wi = swi; }
  if (threadIdx.x != 0) return;
  int b = 0;
  if (exceptional) {
    for (int k = 0; k < nb; k++) {
      int i = hi - 2 * k;
      if (i - 2 < lo) i = hi;
      R ss = absv(H[i + (size_t)(i - 1) * ldh]) + absv(H[(i - 1) + (size_t)(i - 2) * ldh]);
      S aa = mk<S>(R(0.75) * ss) + H[i + (size_t)i * ldh];
      R w4[4];
      eig2<S>(aa, mk<S>(ss), mk<S>(R(-0.4375) * ss), aa, w4);
      for (int q = 0; q < 4; q++) out[4 * b + q] = w4[q];
      b++;
    }
    *nb_out = b;
    return;
  }
  if (tr<S>::cx) {
    for (int k = 0; k + 1 < ns && b < nb; k += 2) {
      out[4 * b] = wr[k]; out[4 * b + 1] = wi[k]; out[4 * b + 2] = wr[k + 1]; out[4 * b + 3] = wi[k + 1];
      b++;
    }
  } else {
    int pend = -1;
    for (int k = 0; k < ns && b < nb; k++) {
      if (wi[k] != R(0)) {  // conjugate pair occupies k, k+1
        if (k + 1 < ns) {
          out[4 * b] = wr[k]; out[4 * b + 1] = wi[k]; out[4 * b + 2] = wr[k + 1]; out[4 * b + 3] = wi[k + 1];
          b++;
        }
        k++;
        continue;
      }
      if (pend < 0) { pend = k; continue; }
      out[4 * b] = wr[pend]; out[4 * b + 1] = 0; out[4 * b + 2] = wr[k]; out[4 * b + 3] = 0;
      b++;
      pend = -1;
    }
  }
  if (b == 0) {  // nothing pairable: fall back to the trailing diagonal entry
    R h = re(H[hi + (size_t)hi * ldh]), hi_ = im(H[hi + (size_t)hi * ldh]);
    out[0] = h; out[1] = hi_; out[2] = h; out[3] = hi_;
    b = 1;
  }
  for (int k = b; k < nb; k++)
    for (int q = 0; q < 4; q++) out[4 * k + q] = out[4 * (k % b) + q];
  *nb_out = b;
}

template <class S>
__global__ void copy_block_kernel(int n, const S* A, int lda, S* B, int ldb) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < n) B[i + (size_t)j * ldb] = A[i + (size_t)j * lda];
}

}  // namespace msy
