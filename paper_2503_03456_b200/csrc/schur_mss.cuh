// schur_mss.cuh -- one-CTA small-bulge multishift QR for blocks held in shared memory.
//
// Same contract as schur_small_kernel (replaces `_hessenberg` + `schur`,
// pkg/src/mpsylv/linalg.py:446-577, for blocks of order n <= SmallCfg<S>::NMAX),
// but each QR sweep chases a chain of nb double-shift bulges (one warp per bulge,
// bulges 4 rows apart, all bulges of a step in parallel, as in chase_kernel)
// through the whole active block instead of one bulge at a time.  A sweep over
// an active block of order s therefore costs ~s + 4 nb CTA steps for 2 nb
// shifts, where the single-bulge kernel needs ~s steps per 2 shifts.
//   * shifts: eigenvalues of the trailing 2nb x 2nb block, computed by warp 0
//     with a warp-synchronous double-shift QR (warp_eig); nb = 1 uses the
//     trailing 2x2 block (Francis double shift, as the single-bulge kernel);
//   * deflation test and exceptional shifts follow the reference
//     (linalg.py:541-557): |h_k,k-1| <= u (|h_k-1,k-1| + |h_kk|), exceptional
//     shifts after stagnant sweeps, 30 n sweep limit;
//   * real arithmetic keeps 2x2 blocks; complex arithmetic splits them with
//     the eigenvector rotation so T is triangular (like the reference).
#pragma once
#include "common.cuh"
#include "schur_small.cuh"
#include "aed.cuh"

namespace msy {

#ifndef MSY_MSS_NWARP
#define MSY_MSS_NWARP 8  // warps (= bulges per sweep) of the one-CTA multishift kernel
#endif
template <class S> struct MssCfg { static constexpr int NWARP = MSY_MSS_NWARP; };
// largest order of an eigenvalues-only call (no Z: the smem holds one matrix)
#ifndef MSY_EIGMAX_F32
#define MSY_EIGMAX_F32 192
#endif
template <class S> struct EigCfg { static constexpr int NMAX = sizeof(S) == 4 ? MSY_EIGMAX_F32 : (sizeof(S) == 8 ? 144 : 104); };
constexpr int MSS_A2 = 33;  // ld of the shift-block scratch (<= 32 x 32 plus dummy row/column)

// Eigenvalues of the k x k upper Hessenberg matrix A (smem, column-major, ld
// MSS_A2, k <= 32) by one warp; A is destroyed.
// Returns ST_OK or ST_ITERLIMIT.
template <class S>
__device__ int warp_eig(int k, S* A, typename tr<S>::R* wr, typename tr<S>::R* wi, int lane) {
  typedef typename tr<S>::R R;
  constexpr int ld = MSS_A2;
  const R u = tr<S>::u();
#define AA(i, j) A[(i) + (j) * ld]
  int i = k - 1, its = 0, total = 0;
  while (i >= 0) {
    const int kk = i - lane;
    bool neg = false;
    if (kk >= 1) {
      S h = AA(kk, kk - 1);
      neg = iszero(h) || absv(h) <= u * (absv(AA(kk - 1, kk - 1)) + absv(AA(kk, kk)));
    }
    const unsigned mask = __ballot_sync(0xffffffffu, neg);
    const int l = mask ? i - (__ffs(mask) - 1) : 0;
    __syncwarp();
    if (l > 0 && lane == 0) AA(l, l - 1) = S(0);
    if (l == i) {
      if (lane == 0) { wr[i] = re(AA(i, i)); wi[i] = im(AA(i, i)); }
      i -= 1; its = 0;
      __syncwarp();
      continue;
    }
    if (l == i - 1) {
      R w4[4];
      eig2<S>(AA(i - 1, i - 1), AA(i - 1, i), AA(i, i - 1), AA(i, i), w4);
      if (lane == 0) { wr[i - 1] = w4[0]; wi[i - 1] = w4[1]; wr[i] = w4[2]; wi[i] = w4[3]; }
      i -= 2; its = 0;
      __syncwarp();
      continue;
    }
    if (total >= 30 * k) return ST_ITERLIMIT;
    its++; total++;
    R w4[4];
    if (its % 10 == 0) {
      R s = absv(AA(i, i - 1)) + absv(AA(i - 1, i - 2));
      S h11 = mk<S>(R(0.75) * s) + AA(i, i);
      eig2<S>(h11, mk<S>(R(-0.4375) * s), mk<S>(s), h11, w4);
    } else {
      eig2<S>(AA(i - 1, i - 1), AA(i - 1, i), AA(i, i - 1), AA(i, i), w4);
      if (!tr<S>::cx && w4[1] == R(0)) {
        R hii = re(AA(i, i));
        R s0 = fabs(w4[0] - hii) <= fabs(w4[2] - hii) ? w4[0] : w4[2];
        w4[0] = w4[2] = s0;
      }
    }
    for (int p = l - 1; p <= i - 2; p++) {
      const int nr = (i - p) >= 3 ? 3 : 2;
      S x0, x1, x2, beta, tau, v1, v2;
      if (p < l) shift_poly<S>(AA(l, l), AA(l + 1, l), AA(l, l + 1), AA(l + 1, l + 1), AA(l + 2, l + 1), w4, x0, x1, x2);
      else { x0 = AA(p + 1, p); x1 = AA(p + 2, p); x2 = nr > 2 ? AA(p + 3, p) : S(0); }
      refl3_fast(nr, x0, x1, x2, beta, tau, v1, v2);
      __syncwarp();
      if (!iszero(tau)) {
        const int rmax = (p + 4 < i) ? p + 4 : i;
        if (nr == 3) {
          wl3<S, ld>(A, p + 1, p + 1, i, conj(tau), v1, v2, lane);
          __syncwarp();
          wr3<S, ld>(A, p + 1, l, rmax, tau, v1, v2, lane);
        } else {
          wl2<S, ld>(A, p + 1, p + 1, i, conj(tau), v1, lane);
          __syncwarp();
          wr2<S, ld>(A, p + 1, l, rmax, tau, v1, lane);
        }
      }
      __syncwarp();
      if (p >= l && lane == 0) {
        AA(p + 1, p) = beta;
        AA(p + 2, p) = S(0);
        if (nr > 2) AA(p + 3, p) = S(0);
      }
      __syncwarp();
    }
  }
#undef AA
  return ST_OK;
}

// Schur form T = V^H A V of the k x k upper Hessenberg matrix A (smem, ld MSS_A2,
// k <= 32) by one warp, V (ld MSS_A2) accumulated from the identity.  Real arithmetic
// keeps 2x2 blocks; complex arithmetic splits them (T triangular).  Deflation by the
// reference's criterion (linalg.py:541-544).  Returns ST_OK or ST_ITERLIMIT.
template <class S>
__device__ int warp_schur_v(int k, S* A, S* V, int lane) {
  typedef typename tr<S>::R R;
  constexpr int ld = MSS_A2;
  const R u = tr<S>::u();
#define AA(i, j) A[(i) + (j) * ld]
#define VV(i, j) V[(i) + (j) * ld]
  for (int e = lane; e < k * k; e += 32) VV(e % k, e / k) = (e % k == e / k) ? S(1) : S(0);
  __syncwarp();
  int i = k - 1, its = 0, total = 0;
  while (i >= 0) {
    const int kk = i - lane;
    bool neg = false;
    if (kk >= 1) {
      S h = AA(kk, kk - 1);
      neg = iszero(h) || absv(h) <= u * (absv(AA(kk - 1, kk - 1)) + absv(AA(kk, kk)));
    }
    const unsigned mask = __ballot_sync(0xffffffffu, neg);
    const int l = mask ? i - (__ffs(mask) - 1) : 0;
    __syncwarp();
    if (l > 0 && lane == 0) AA(l, l - 1) = S(0);
    __syncwarp();
    if (l == i) { i -= 1; its = 0; continue; }
    if (l == i - 1) {
      if (tr<S>::cx) {  // split with the eigenvector rotation (as schur_mss_kernel)
        R w4[4];
        eig2<S>(AA(l, l), AA(l, i), AA(i, l), AA(i, i), w4);
        S a = AA(l, l), b = AA(l, i), c = AA(i, l), d = AA(i, i);
        S lam = mk<S>(w4[0], w4[1]);
        S va = lam - d, vb = c, wa = b, wb = lam - a;
        if (abs2(wa) + abs2(wb) > abs2(va) + abs2(vb)) { va = wa; vb = wb; }
        R nv = sqrt(abs2(va) + abs2(vb));
        S g11 = va / mk<S>(nv), g21 = vb / mk<S>(nv);
        S g12 = -conj(g21), g22 = conj(g11);
        __syncwarp();
        for (int j = l + lane; j < k; j += 32) {
          S h1 = AA(l, j), h2 = AA(i, j);
          AA(l, j) = fmacc(g11, h1, conj(g21) * h2);
          AA(i, j) = fmacc(g12, h1, conj(g22) * h2);
        }
        __syncwarp();
        for (int e = lane; e < (i + 1) + k; e += 32) {
          S* M = e <= i ? A : V;
          const int r = e <= i ? e : e - i - 1;
          S c1 = M[r + l * ld], c2 = M[r + i * ld];
          M[r + l * ld] = c1 * g11 + c2 * g21;
          M[r + i * ld] = c1 * g12 + c2 * g22;
        }
        __syncwarp();
        if (lane == 0) AA(i, l) = S(0);
        __syncwarp();
      }
      i -= 2; its = 0;
      continue;
    }
    if (total >= 30 * k) return ST_ITERLIMIT;
    its++; total++;
    R w4[4];
    if (its % 10 == 0) {
      R s = absv(AA(i, i - 1)) + absv(AA(i - 1, i - 2));
      S h11 = mk<S>(R(0.75) * s) + AA(i, i);
      eig2<S>(h11, mk<S>(R(-0.4375) * s), mk<S>(s), h11, w4);
    } else {
      eig2<S>(AA(i - 1, i - 1), AA(i - 1, i), AA(i, i - 1), AA(i, i), w4);
      if (!tr<S>::cx && w4[1] == R(0)) {
        R hii = re(AA(i, i));
        R s0 = fabs(w4[0] - hii) <= fabs(w4[2] - hii) ? w4[0] : w4[2];
        w4[0] = w4[2] = s0;
      }
    }
    for (int p = l - 1; p <= i - 2; p++) {
      const int nr = (i - p) >= 3 ? 3 : 2;
      S x0, x1, x2, beta, tau, v1, v2;
      if (p < l) shift_poly<S>(AA(l, l), AA(l + 1, l), AA(l, l + 1), AA(l + 1, l + 1), AA(l + 2, l + 1), w4, x0, x1, x2);
      else { x0 = AA(p + 1, p); x1 = AA(p + 2, p); x2 = nr > 2 ? AA(p + 3, p) : S(0); }
      refl3_fast(nr, x0, x1, x2, beta, tau, v1, v2);
      __syncwarp();
      if (!iszero(tau)) {
        const int rmax = (p + 4 < i) ? p + 4 : i;
        if (nr == 3) {
          wl3<S, ld>(A, p + 1, p + 1, k - 1, conj(tau), v1, v2, lane);
          __syncwarp();
          wr3<S, ld>(A, p + 1, 0, rmax, tau, v1, v2, lane);
          wr3<S, ld>(V, p + 1, 0, k - 1, tau, v1, v2, lane);
        } else {
          wl2<S, ld>(A, p + 1, p + 1, k - 1, conj(tau), v1, lane);
          __syncwarp();
          wr2<S, ld>(A, p + 1, 0, rmax, tau, v1, lane);
          wr2<S, ld>(V, p + 1, 0, k - 1, tau, v1, lane);
        }
      }
      __syncwarp();
      if (p >= l && lane == 0) {
        AA(p + 1, p) = beta;
        AA(p + 2, p) = S(0);
        if (nr > 2) AA(p + 3, p) = S(0);
      }
      __syncwarp();
    }
  }
#undef AA
#undef VV
  return ST_OK;
}

// One Householder step of a warp on a window (T, V in smem, stride LD, nw <= 32):
// x = vb[r0..r1] is reduced to beta e_{r0}; applied from the left to T[r0..r1, c0..nw-1]
// and from the right to T[0..r1, r0..r1] and V[0..nw-1, r0..r1].  vb is overwritten
// with the reflector.  Returns beta.
template <class S, int LD>
__device__ S warp_hh_step(S* T, S* V, int nw, int r0, int r1, int c0, S* vb, int lane) {
  typedef typename tr<S>::R R;
  R sn = 0;
  for (int r = r0 + 1 + lane; r <= r1; r += 32) sn += abs2(vb[r]);
  sn = warp_sum(sn);
  const S x0 = vb[r0];
  __syncwarp();
  if (sn == R(0) && im(x0) == R(0)) return x0;
  const R nrm = sqrt(abs2(x0) + sn);
  const R b = re(x0) >= R(0) ? -nrm : nrm;
  const S tau = (mk<S>(b) - x0) / mk<S>(b);
  const S scal = S(1) / (x0 - mk<S>(b));
  for (int r = r0 + lane; r <= r1; r += 32) vb[r] = r == r0 ? S(1) : vb[r] * scal;
  __syncwarp();
  const S ctau = conj(tau);
  for (int c = c0 + lane; c < nw; c += 32) {
    S w = S(0);
    for (int r = r0; r <= r1; r++) w = fmacc(vb[r], T[r + c * LD], w);
    w = ctau * w;
    for (int r = r0; r <= r1; r++) T[r + c * LD] = T[r + c * LD] - vb[r] * w;
  }
  __syncwarp();
  for (int e = lane; e < (r1 + 1) + nw; e += 32) {
    S* M = e <= r1 ? T : V;
    const int i = e <= r1 ? e : e - r1 - 1;
    S w = S(0);
    for (int r = r0; r <= r1; r++) w = fmac(M[i + r * LD], vb[r], w);
    w = tau * w;
    for (int r = r0; r <= r1; r++) M[i + r * LD] = M[i + r * LD] - w * conj(vb[r]);
  }
  __syncwarp();
  return mk<S>(b);
}

// After aed_deflate_warp: reflect the undeflated spike entries s conj(V(0, 0:ns)) back
// to one entry and re-reduce T[0:ns, 0:ns] to Hessenberg form (one warp, ns <= 32).
// Returns the new subdiagonal entry coupling the window to the block above it.
template <class S, int LD>
__device__ S aed_rehess_warp(S* T, S* V, int nw, int ns, S s, S* vb, int lane) {
  if (ns <= 0) return S(0);
  const S sub0 = s * conj(V[0]);
  if (ns == 1) return sub0;
  for (int r = lane; r < ns; r += 32) vb[r] = s * conj(V[r * LD]);
  __syncwarp();
  const S newsub = warp_hh_step<S, LD>(T, V, nw, 0, ns - 1, 0, vb, lane);
  for (int kc = 0; kc + 2 < ns; kc++) {
    for (int r = kc + 1 + lane; r < ns; r += 32) vb[r] = T[r + kc * LD];
    __syncwarp();
    const S beta = warp_hh_step<S, LD>(T, V, nw, kc + 1, ns - 1, kc + 1, vb, lane);
    for (int r = kc + 1 + lane; r < ns; r += 32) T[r + kc * LD] = r == kc + 1 ? beta : S(0);
    __syncwarp();
  }
  return newsub;
}

// Pair ns eigenvalues (wr, wi) into nb bulge shift quadruples (sr1, si1, sr2, si2):
// conjugate pairs stay together, real shifts are paired in order.  Returns the
// number of distinct quadruples written (the rest repeat them).
template <class S>
__device__ int pair_shifts(int ns, const typename tr<S>::R* wr, const typename tr<S>::R* wi, int nb,
                           typename tr<S>::R* out, typename tr<S>::R fallback_re, typename tr<S>::R fallback_im) {
  typedef typename tr<S>::R R;
  int b = 0;
  if (tr<S>::cx) {
    for (int k = 0; k + 1 < ns && b < nb; k += 2) {
      out[4 * b] = wr[k]; out[4 * b + 1] = wi[k]; out[4 * b + 2] = wr[k + 1]; out[4 * b + 3] = wi[k + 1];
      b++;
    }
  } else {
    int pend = -1;
    for (int k = 0; k < ns && b < nb; k++) {
      if (wi[k] != R(0)) {
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
  if (b == 0) {
    out[0] = fallback_re; out[1] = fallback_im; out[2] = fallback_re; out[3] = fallback_im;
    b = 1;
  }
  for (int k = b; k < nb; k++)
    for (int q = 0; q < 4; q++) out[4 * k + q] = out[4 * (k % b) + q];
  return b;
}

template <class S>
struct MssShared {
  int l, status;
  S bt[2];
};

template <class S, int LDC>
__global__ void __launch_bounds__(32 * MSY_MSS_NWARP) schur_mss_kernel(int n, S* Hg, int ldh, S* Zg, int ldz, int flags,
                                                       typename tr<S>::R* wr, typename tr<S>::R* wi, int* info,
                                                       typename tr<S>::R tol) {
  typedef typename tr<S>::R R;
  constexpr int NW = MssCfg<S>::NWARP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int ld = LDC;  // fixed stride: immediate smem offsets in the warp ops
  const bool wantz = flags & SS_WANTZ;
  const bool eigonly = flags & SS_EIGONLY;
  S* H = (S*)smem_raw;                        // n x n, stride ld
  S* Zs = H + (size_t)ld * n;                 // n x n when wantz
  S* A2 = Zs + (wantz ? (size_t)ld * n : 0);  // shift block scratch, MSS_A2 x MSS_A2
  S* V2 = A2 + MSS_A2 * MSS_A2;               // AED window Schur vectors, MSS_A2 x MSS_A2
  __shared__ MssShared<S> sh;
  __shared__ S vbuf[SmallCfg<S>::NMAX + 4];
  __shared__ R sw[4 * NW];                    // bulge shift quadruples
  __shared__ R ewr[40], ewi[40];
  __shared__ S aQs[16];
  __shared__ int aok, a_nd, a_ns;
  __shared__ S a_sub;
  const int aedw = (flags >> 8) & 63;         // in-kernel AED window (0: off), <= 32
  const int aedg = (flags >> 16) & 63;        // its undeflatable-group cap
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const R u = tol > R(0) ? tol : tr<S>::u();  // deflation tolerance (looser for shift-only calls)
#define HH(i, j) H[(i) + (j) * ld]
#define ZZ(i, j) Zs[(i) + (j) * ld]
  if (n <= nt && !(flags & SS_ZIN)) {  // thread i stages row i: 16 independent loads in flight
    for (int j0 = 0; j0 < n; j0 += 16) {
      S v[16];
#pragma unroll
      for (int u = 0; u < 16; u++) v[u] = (tid < n && j0 + u < n) ? Hg[tid + (size_t)(j0 + u) * ldh] : S(0);
#pragma unroll
      for (int u = 0; u < 16; u++)
        if (tid < n && j0 + u < n) {
          HH(tid, j0 + u) = v[u];
          if (wantz) ZZ(tid, j0 + u) = (tid == j0 + u) ? S(1) : S(0);
        }
    }
  } else {
    for (int e = tid; e < n * n; e += nt) {
      int i = e % n, j = e / n;
      HH(i, j) = Hg[i + (size_t)j * ldh];
      if (wantz) ZZ(i, j) = (flags & SS_ZIN) ? Zg[i + (size_t)j * ldz] : (i == j ? S(1) : S(0));
    }
  }
  __syncthreads();
  if (flags & SS_HESS) smem_hessenberg<S>(n, H, Zs, ld, wantz, vbuf, sh.bt);

  int i = n - 1, its = 0, total = 0, status = ST_OK;
  while (i >= 0) {
    // ---- deflation search (warp 0), broadcast through smem ----
    if (warp == 0) {
      int l = 0;
      for (int base = i; base >= 1; base -= 32) {
        const int k = base - lane;
        bool neg = false;
        if (k >= 1) {
          S h = HH(k, k - 1);
          neg = iszero(h) || absv(h) <= u * (absv(HH(k - 1, k - 1)) + absv(HH(k, k)));
        }
        const unsigned mask = __ballot_sync(0xffffffffu, neg);
        if (mask) { l = base - (__ffs(mask) - 1); break; }
      }
      if (lane == 0) {
        sh.l = l;
        if (l > 0) HH(l, l - 1) = S(0);
      }
    }
    __syncthreads();
    const int l = sh.l;
    if (l == i) {
      if (wr && tid == 0) { wr[i] = re(HH(i, i)); wi[i] = im(HH(i, i)); }
      i -= 1; its = 0;
      __syncthreads();  // sh.l is rewritten by the next search
      continue;
    }
    if (l == i - 1) {
      R w4[4];
      eig2<S>(HH(i - 1, i - 1), HH(i - 1, i), HH(i, i - 1), HH(i, i), w4);
      if (wr && tid == 0) { wr[i - 1] = w4[0]; wi[i - 1] = w4[1]; wr[i] = w4[2]; wi[i] = w4[3]; }
      if (tr<S>::cx) {  // split with the eigenvector rotation (first column g = v / |v|)
        S a = HH(l, l), b = HH(l, i), c = HH(i, l), d = HH(i, i);
        S lam = mk<S>(w4[0], w4[1]);
        S va = lam - d, vb = c, wa = b, wb = lam - a;
        if (abs2(wa) + abs2(wb) > abs2(va) + abs2(vb)) { va = wa; vb = wb; }
        R nv = sqrt(abs2(va) + abs2(vb));
        S g11 = va / mk<S>(nv), g21 = vb / mk<S>(nv);
        S g12 = -conj(g21), g22 = conj(g11);
        __syncthreads();
        const int jmax = eigonly ? i : n - 1;
        for (int j = l + tid; j <= jmax; j += nt) {
          S h1 = HH(l, j), h2 = HH(i, j);
          HH(l, j) = fmacc(g11, h1, conj(g21) * h2);
          HH(i, j) = fmacc(g12, h1, conj(g22) * h2);
        }
        __syncthreads();
        const int rmin = eigonly ? l : 0;
        for (int r = rmin + tid; r <= i; r += nt) {
          S c1 = HH(r, l), c2 = HH(r, i);
          HH(r, l) = c1 * g11 + c2 * g21;
          HH(r, i) = c1 * g12 + c2 * g22;
        }
        if (wantz)
          for (int r = tid; r < n; r += nt) {
            S c1 = ZZ(r, l), c2 = ZZ(r, i);
            ZZ(r, l) = c1 * g11 + c2 * g21;
            ZZ(r, i) = c1 * g12 + c2 * g22;
          }
        __syncthreads();
        if (tid == 0) HH(i, l) = S(0);
      }
      __syncthreads();
      i -= 2; its = 0;
      continue;
    }
    if (total >= 30 * n) { status = ST_ITERLIMIT; break; }
    its++; total++;
    int sz = i - l + 1;
    // ---- in-kernel aggressive early deflation on a trailing window (aed.cuh) ----
    int aed_ns = 0;
    if (aedw > 0 && sz > 12 && its % 6 != 0) {
      const int nwa = min(sz, aedw);
      const int kw = i - nwa + 1;
      if (warp == 0) {
        for (int e = lane; e < nwa * nwa; e += 32) {
          const int r = e % nwa, c = e / nwa;
          A2[r + c * MSS_A2] = r <= c + 1 ? HH(kw + r, kw + c) : S(0);
        }
        __syncwarp();
        const int st = warp_schur_v<S>(nwa, A2, V2, lane);
        int nd = -1, nsu = 0;
        if (st == ST_OK) {
          const S s = kw > l ? HH(kw, kw - 1) : S(0);
          nsu = aed_deflate_warp<S, MSS_A2>(A2, V2, nwa, s, aedg, lane, aQs, &aok);
          nd = nwa - nsu;
          if (lane == 0) {  // eigenvalues: deflated -> wr/wi (final positions), undeflated -> shifts
            int cnt = 0;
            for (int r = nwa - 1; r >= 0;) {
              R w4[4];
              const bool two = !tr<S>::cx && r > 0 && !iszero(A2[r + (r - 1) * MSS_A2]);
              if (two) eig2<S>(A2[(r - 1) * (MSS_A2 + 1)], A2[(r - 1) + r * MSS_A2], A2[r + (r - 1) * MSS_A2],
                               A2[r * (MSS_A2 + 1)], w4);
              else { w4[0] = w4[2] = re(A2[r * (MSS_A2 + 1)]); w4[1] = w4[3] = im(A2[r * (MSS_A2 + 1)]); }
              if (r >= nsu) {
                if (wr) {
                  if (two) { wr[kw + r - 1] = w4[0]; wi[kw + r - 1] = w4[1]; }
                  wr[kw + r] = w4[2]; wi[kw + r] = w4[3];
                }
              } else if (cnt + 2 <= 40) {
                if (two) { ewr[cnt] = w4[0]; ewi[cnt] = w4[1]; ewr[cnt + 1] = w4[2]; ewi[cnt + 1] = w4[3]; cnt += 2; }
                else { ewr[cnt] = w4[0]; ewi[cnt] = w4[1]; cnt += 1; }
              }
              r -= two ? 2 : 1;
            }
          }
          if (nd > 0) {
            const S sub = aed_rehess_warp<S, MSS_A2>(A2, V2, nwa, nsu, s, vbuf, lane);
            if (lane == 0) a_sub = sub;
          }
        }
        if (lane == 0) { a_nd = nd; a_ns = nsu; }
      }
      __syncthreads();
      const int nd = a_nd;
      if (nd > 0) {
        // window <- T; V applied to the rows above it, the columns right of it and Z
        const int rtop = eigonly ? l : 0;
        const int jmx = eigonly ? i : n - 1;
        const int nR = kw - rtop, nZ = wantz ? n : 0, nC = jmx - i;
        for (int e = tid; e < nwa * nwa; e += nt) {
          const int r = e % nwa, c = e / nwa;
          HH(kw + r, kw + c) = (r > c + 1 || (r == c + 1 && r == a_ns)) ? S(0) : A2[r + c * MSS_A2];
        }
        for (int e = tid; e < nR + nZ + nC; e += nt) {
          S x[32];
          if (e < nR + nZ) {  // a row: (.) V
            S* row = e < nR ? &HH(rtop + e, kw) : &ZZ(e - nR, kw);
#pragma unroll
            for (int t = 0; t < 32; t++) x[t] = t < nwa ? row[t * ld] : S(0);
            for (int j = 0; j < nwa; j++) {
              S a = S(0);
#pragma unroll
              for (int t = 0; t < 32; t++)
                if (t < nwa) a = fmac(x[t], V2[t + j * MSS_A2], a);
              row[j * ld] = a;
            }
          } else {  // a column right of the window: V^H (.)
            S* col = &HH(kw, i + 1 + (e - nR - nZ));
#pragma unroll
            for (int t = 0; t < 32; t++) x[t] = t < nwa ? col[t] : S(0);
            for (int j = 0; j < nwa; j++) {
              S a = S(0);
#pragma unroll
              for (int t = 0; t < 32; t++)
                if (t < nwa) a = fmacc(V2[t + j * MSS_A2], x[t], a);
              col[j] = a;
            }
          }
        }
        if (tid == 0 && kw > l) HH(kw, kw - 1) = a_sub;
        __syncthreads();
        i -= nd;
        its = 0;
        if (nd * 100 > 14 * nwa || i - l + 1 <= 12) continue;
        sz = i - l + 1;
      }
      if (nd >= 0) aed_ns = a_ns;
    }
    const int nb = aed_ns >= 4 ? min(NW, max(1, min(aed_ns / 2 - 1, sz / 10))) : min(NW, max(1, sz / 10));
    const int ns = 2 * nb;
    // ---- shifts (warp 0) ----
    if (warp == 0 && aed_ns >= 4) {
      if (lane == 0) pair_shifts<S>(aed_ns, ewr, ewi, nb, sw, re(HH(i, i)), im(HH(i, i)));
    } else if (warp == 0) {
      const bool exc = (its % 6 == 0);
      if (nb == 1 || exc) {
        for (int b = 0; b < nb; b++) {
          R w4[4];
          if (exc) {
            int ii = i - 2 * b;
            if (ii - 2 < l) ii = i;
            R s = absv(HH(ii, ii - 1)) + absv(HH(ii - 1, ii - 2));
            S h11 = mk<S>(R(0.75) * s) + HH(ii, ii);
            eig2<S>(h11, mk<S>(R(-0.4375) * s), mk<S>(s), h11, w4);
          } else {
            eig2<S>(HH(i - 1, i - 1), HH(i - 1, i), HH(i, i - 1), HH(i, i), w4);
            if (!tr<S>::cx && w4[1] == R(0)) {
              R hii = re(HH(i, i));
              R s0 = fabs(w4[0] - hii) <= fabs(w4[2] - hii) ? w4[0] : w4[2];
              w4[0] = w4[2] = s0;
            }
          }
          if (lane == 0)
            for (int q = 0; q < 4; q++) sw[4 * b + q] = w4[q];
        }
      } else {
        const int k0 = i - ns + 1;
        for (int e = lane; e < ns * ns; e += 32) {
          int r = e % ns, c = e / ns;
          A2[r + c * MSS_A2] = (r <= c + 1) ? HH(k0 + r, k0 + c) : S(0);
        }
        __syncwarp();
        int st = warp_eig<S>(ns, A2, ewr, ewi, lane);
        __syncwarp();
        if (lane == 0) {
          if (st != ST_OK) {  // fall back to the trailing diagonal entry
            for (int q = 0; q < ns; q++) { ewr[q] = re(HH(i, i)); ewi[q] = im(HH(i, i)); }
          }
          pair_shifts<S>(ns, ewr, ewi, nb, sw, re(HH(i, i)), im(HH(i, i)));
        }
      }
    }
    __syncthreads();
    // ---- sweep: nb bulges, one warp each, 4 rows apart ----
    const int jmax = eigonly ? i : n - 1;  // last column of left ops
    const int rmin = eigonly ? l : 0;      // first row of right ops
    const int T = (i - l) + 4 * (nb - 1);
    const int j = warp;
    for (int t = 0; t < T; t++) {
      const int p = l - 1 + t - 4 * j;
      const bool act = (j < nb) && (p >= l - 1) && (p <= i - 2);
      const int nr = (i - p) >= 3 ? 3 : 2;
      S tau = S(0), v1 = S(0), v2 = S(0);
      if (act) {
        S x0, x1, x2, beta;
        if (p == l - 1) {
          shift_poly<S>(HH(l, l), HH(l + 1, l), HH(l, l + 1), HH(l + 1, l + 1), (l + 2 <= i) ? HH(l + 2, l + 1) : S(0),
                        sw + 4 * j, x0, x1, x2);
        } else {
          x0 = HH(p + 1, p); x1 = HH(p + 2, p); x2 = nr > 2 ? HH(p + 3, p) : S(0);
        }
        refl3_fast(nr, x0, x1, x2, beta, tau, v1, v2);
        __syncwarp();
        if (!iszero(tau)) {
          if (nr == 3) wl3<S, ld>(H, p + 1, p + 1, jmax, conj(tau), v1, v2, lane);
          else wl2<S, ld>(H, p + 1, p + 1, jmax, conj(tau), v1, lane);
        }
        if (p >= l && lane == 0) {
          HH(p + 1, p) = beta;
          HH(p + 2, p) = S(0);
          if (nr > 2) HH(p + 3, p) = S(0);
        }
      }
      __syncthreads();
      if (act && !iszero(tau)) {
        const int rmax = (p + 4 < i) ? p + 4 : i;
        if (nr == 3) {
          wr3<S, ld>(H, p + 1, rmin, rmax, tau, v1, v2, lane);
          if (wantz) wr3<S, ld>(Zs, p + 1, 0, n - 1, tau, v1, v2, lane);
        } else {
          wr2<S, ld>(H, p + 1, rmin, rmax, tau, v1, lane);
          if (wantz) wr2<S, ld>(Zs, p + 1, 0, n - 1, tau, v1, lane);
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) { sh.status = status; }
  __syncthreads();
  if (!eigonly)  // eigenvalue-only calls (the sweeps' shifts) read the matrix in place and leave it alone
    for (int e = tid; e < n * n; e += nt) {
      int r = e % n, c = e / n;
      Hg[r + (size_t)c * ldh] = HH(r, c);
      if (wantz) Zg[r + (size_t)c * ldz] = ZZ(r, c);
    }
  if (tid == 0 && info) {
    info[0] = sh.status;
    info[1] = total;
  }
#undef HH
#undef ZZ
}

template <class S>
static size_t mss_smem_bytes(int n, bool wantz) {
  const size_t ld = (n <= SmallCfg<S>::NMAX ? SmallCfg<S>::NMAX : EigCfg<S>::NMAX) + 1;
  return (ld * n * (wantz ? 2 : 1) + (size_t)2 * MSS_A2 * MSS_A2) * sizeof(S) + 64;
}

}  // namespace msy
