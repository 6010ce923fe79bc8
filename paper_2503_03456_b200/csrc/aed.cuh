// aed.cuh -- aggressive early deflation (AED) for the large-matrix Schur loop.
//
// The reference deflates one subdiagonal at a time inside its single-shift sweep
// (pkg/src/mpsylv/linalg.py:541-544).  For m above the one-CTA size the B200 path
// instead examines a trailing window of the active block (the published
// Braman-Byers-Mathias AED scheme, as in LAPACK's xLAQR3):
//   1. the nw x nw window is copied out and brought to Schur form T = V^H W V
//      with its Schur vectors V (schur_small_launch, one CTA);
//   2. aed_kernel (one CTA, T and V in shared memory): the "spike" s V(0, :)
//      (s = the subdiagonal entry coupling the window to the rest of the block)
//      decides, block by block from the bottom, which eigenvalues are converged
//      (|s V(0, j)| <= u |T_jj|).  Undeflatable blocks are collected in a group
//      kept at the bottom of the undeflated part; the next candidate is swapped
//      below that group (direct block swaps, below) before it is tested.  The
//      group size is capped (gmax): past it the check stops;
//   3. the spike of the undeflated part is reflected back to one entry and that
//      part re-reduced to Hessenberg form; the window is written back to H and V
//      returned, so the caller applies V to the rest of H and to U (apply_z).
// The undeflated eigenvalues (bottom-most first) become the next sweep's shifts.
//
// Deflation bound: a deflated eigenvalue drops a spike entry of size <= u |T_jj|,
// a backward perturbation of the same order as the reference's subdiagonal
// criterion.
#pragma once
#include "common.cuh"
#include "schur_small.cuh"

namespace msy {

template <class S> struct wide;
template <> struct wide<float> { typedef double T; };
template <> struct wide<double> { typedef double T; };
template <> struct wide<cfloat> { typedef cdouble T; };
template <> struct wide<cdouble> { typedef cdouble T; };

template <class D> __host__ __device__ __forceinline__ D dconj(D a) { return conj(a); }

// Swap of adjacent diagonal blocks of a (quasi-)triangular k x k matrix M (k = p+q <= 4,
// column-major M[i + 4 j]): the p x p block A11 above the q x q block A22.  Solves
// A11 X - X A22 = A12 (Kronecker system, complete pivoting), takes the QR
// factorisation of [-X; I_q] (its columns span the invariant subspace of A22's
// eigenvalues) and returns the k x k unitary Q (Q[i + 4 j]) with Q^H M Q =
// [[A22', *], [0, A11']].  Returns false when the swapped lower-left block is not
// negligible (relative to `tol`), in which case the swap must not be applied.
template <class D>
__host__ __device__ bool block_swap_q(const D* M, int p, int q, D* Q, double tol) {
  typedef typename tr<D>::R R;
  const int k = p + q, nu = p * q;
  D K[16], rhs[4];
  for (int i = 0; i < 16; i++) K[i] = D(0);
  // unknown index of X[r][c] = r + c p ; equation (r, c)
  for (int c = 0; c < q; c++)
    for (int r = 0; r < p; r++) {
      const int e = r + c * p;
      rhs[e] = M[r + 4 * (p + c)];
      for (int t = 0; t < p; t++) K[e + 4 * (t + c * p)] += M[r + 4 * t];              // (A11 X)[r][c]
      for (int t = 0; t < q; t++) K[e + 4 * (r + t * p)] -= M[(p + t) + 4 * (p + c)];  // (X A22)[r][c]
    }
  R kmax = 0;
  for (int i = 0; i < nu; i++)
    for (int j = 0; j < nu; j++) kmax = fmax(kmax, abs1(K[i + 4 * j]));
  const R smin = fmax(R(4.0e-16) * kmax, R(1e-300));
  int perm[4];
  for (int i = 0; i < 4; i++) perm[i] = i;
  // Gaussian elimination with complete pivoting
  for (int s = 0; s < nu; s++) {
    int pi = s, pj = s;
    R best = -1;
    for (int i = s; i < nu; i++)
      for (int j = s; j < nu; j++)
        if (abs1(K[i + 4 * j]) > best) { best = abs1(K[i + 4 * j]); pi = i; pj = j; }
    if (pi != s) {
      for (int j = 0; j < nu; j++) { D t = K[s + 4 * j]; K[s + 4 * j] = K[pi + 4 * j]; K[pi + 4 * j] = t; }
      D t = rhs[s]; rhs[s] = rhs[pi]; rhs[pi] = t;
    }
    if (pj != s) {
      for (int i = 0; i < nu; i++) { D t = K[i + 4 * s]; K[i + 4 * s] = K[i + 4 * pj]; K[i + 4 * pj] = t; }
      int t = perm[s]; perm[s] = perm[pj]; perm[pj] = t;
    }
    if (abs1(K[s + 4 * s]) < smin) K[s + 4 * s] = D(smin);
    for (int i = s + 1; i < nu; i++) {
      D f = K[i + 4 * s] / K[s + 4 * s];
      for (int j = s + 1; j < nu; j++) K[i + 4 * j] -= f * K[s + 4 * j];
      rhs[i] -= f * rhs[s];
    }
  }
  D y[4], x[4];
  for (int s = nu - 1; s >= 0; s--) {
    D a = rhs[s];
    for (int j = s + 1; j < nu; j++) a -= K[s + 4 * j] * y[j];
    y[s] = a / K[s + 4 * s];
  }
  for (int s = 0; s < nu; s++) x[perm[s]] = y[s];
  // W = [-X; I_q] (k x q), Householder QR, Q = H_0 ... H_{q-1}
  D W[16];
  for (int c = 0; c < q; c++)
    for (int r = 0; r < k; r++) W[r + 4 * c] = r < p ? -x[r + c * p] : (r - p == c ? D(1) : D(0));
  for (int i = 0; i < 16; i++) Q[i] = (i % 4 == i / 4) ? D(1) : D(0);
  for (int c = 0; c < q; c++) {
    R sn = 0;
    for (int r = c + 1; r < k; r++) sn += abs2(W[r + 4 * c]);
    D x0 = W[c + 4 * c];
    if (sn == R(0) && im(x0) == R(0)) continue;
    R nrm = sqrt(abs2(x0) + sn);
    R b = re(x0) >= R(0) ? -nrm : nrm;
    D tau = (mk<D>(b) - x0) / mk<D>(b);
    D scal = D(1) / (x0 - mk<D>(b));
    D v[4];
    for (int r = 0; r < k; r++) v[r] = r < c ? D(0) : (r == c ? D(1) : W[r + 4 * c] * scal);
    // W <- H^H W (columns c+1..q-1), Q <- Q H
    for (int j = c + 1; j < q; j++) {
      D s = D(0);
      for (int r = c; r < k; r++) s += dconj(v[r]) * W[r + 4 * j];
      s = dconj(tau) * s;
      for (int r = c; r < k; r++) W[r + 4 * j] -= v[r] * s;
    }
    for (int i = 0; i < k; i++) {
      D s = D(0);
      for (int r = c; r < k; r++) s += Q[i + 4 * r] * v[r];
      s = tau * s;
      for (int r = c; r < k; r++) Q[i + 4 * r] -= s * dconj(v[r]);
    }
  }
  // stability check: the lower-left (p x q) block of Q^H M Q must be negligible
  R mn = 0, ll = 0;
  for (int i = 0; i < k; i++)
    for (int j = 0; j < k; j++) mn = fmax(mn, abs1(M[i + 4 * j]));
  for (int i = q; i < k; i++)
    for (int j = 0; j < q; j++) {
      D s = D(0);
      for (int a = 0; a < k; a++) {
        D mq = D(0);
        for (int b = 0; b < k; b++) mq += M[a + 4 * b] * Q[b + 4 * j];
        s += dconj(Q[a + 4 * i]) * mq;
      }
      ll = fmax(ll, abs1(s));
    }
  return ll <= tol * fmax(mn, R(1e-300));
}

// Deflation check of a window in Schur form (one warp; T, V in smem with stride LD;
// Qs: 16 smem scratch entries, okf: smem flag).  Candidates are tested from the
// bottom; an undeflatable block joins a group kept at the bottom of the undeflated
// part, and each later candidate is swapped below that group before its test.
// Returns ns, the number of undeflated leading rows (the deflated blocks occupy
// [ns, nw)).  s == 0 deflates everything.
template <class S, int LD>
__device__ int aed_deflate_warp(S* T, S* V, int nw, S s, int gmax, int lane, S* Qs, int* okf) {
  typedef typename tr<S>::R R;
  typedef typename wide<S>::T D;
  const R u = tr<S>::u();
#define TT(i, j) T[(i) + (j) * LD]
#define VV(i, j) V[(i) + (j) * LD]
  int ns = nw, g = 0;
  bool stop = iszero(s);  // s == 0: everything deflates
  if (stop) ns = 0;
  while (!stop && ns - g > 0) {
    const int e = ns - g - 1;
    const int b = (!tr<S>::cx && e > 0 && !iszero(TT(e, e - 1))) ? 2 : 1;
    int pos = e - b + 1;
    // swap the candidate below the undeflatable group
    bool ok = true;
    while (pos + b < ns) {
      const int nxt = pos + b;
      const int q = (!tr<S>::cx && nxt + 1 < ns && !iszero(TT(nxt + 1, nxt))) ? 2 : 1;
      const int k = b + q;
      if (lane == 0) {
        D M[16], Q[16];
        for (int i = 0; i < 16; i++) M[i] = D(0);
        for (int j = 0; j < k; j++)
          for (int i = 0; i < k; i++) M[i + 4 * j] = conv<D>(TT(pos + i, pos + j));
        const bool good = block_swap_q<D>(M, b, q, Q, 64.0 * (double)u);
        (*okf) = good;
        for (int j = 0; j < 4; j++)
          for (int i = 0; i < 4; i++) Qs[i + 4 * j] = conv<S>(Q[i + 4 * j]);
      }
      __syncwarp();
      if (!(*okf)) { ok = false; break; }
      S qv[16];
#pragma unroll
      for (int i = 0; i < 16; i++) qv[i] = Qs[i];
      // rows pos..pos+k-1 of T, columns pos..nw-1: Q^H (.)
      for (int c = pos + lane; c < nw; c += 32) {
        S t[4], o[4];
#pragma unroll
        for (int i = 0; i < 4; i++) t[i] = i < k ? TT(pos + i, c) : S(0);
#pragma unroll
        for (int i = 0; i < 4; i++) {
          S a = S(0);
#pragma unroll
          for (int l = 0; l < 4; l++) a = fmacc(qv[l + 4 * i], t[l], a);
          o[i] = a;
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
          if (i < k) TT(pos + i, c) = o[i];
      }
      __syncwarp();
      // columns pos..pos+k-1 of T (rows 0..pos+k-1) and of V (all rows): (.) Q
      for (int e2 = lane; e2 < (pos + k) + nw; e2 += 32) {
        S* Mx = e2 < pos + k ? T : V;
        const int r = e2 < pos + k ? e2 : e2 - pos - k;
        S t[4], o[4];
#pragma unroll
        for (int i = 0; i < 4; i++) t[i] = i < k ? Mx[r + (pos + i) * LD] : S(0);
#pragma unroll
        for (int i = 0; i < 4; i++) {
          S a = S(0);
#pragma unroll
          for (int l = 0; l < 4; l++) a = fmac(t[l], qv[l + 4 * i], a);
          o[i] = a;
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
          if (i < k) Mx[r + (pos + i) * LD] = o[i];
      }
      __syncwarp();
      if (lane == 0)
        for (int r = pos + q; r < pos + k; r++)
          for (int c = pos; c < pos + q; c++) TT(r, c) = S(0);
      __syncwarp();
      pos += q;
    }
    if (!ok) break;
    // candidate now occupies [ns - b, ns)
    const int bt = ns - 1;
    R foo = absv(TT(bt, bt));
    R sp = absv(s * conj(VV(0, bt)));
    if (b == 2) {
      foo += sqrt(absv(TT(bt, bt - 1))) * sqrt(absv(TT(bt - 1, bt)));
      sp = fmax(sp, absv(s * conj(VV(0, bt - 1))));
    }
    if (foo == R(0)) foo = absv(s);
    if (sp <= fmax(R(1e-30), u * foo)) {
      ns -= b;
    } else {
      g += b;
      if (g >= gmax) stop = true;
    }
  }
  return ns;
#undef TT
#undef VV
}

template <class S> struct AedCfg { static constexpr int NW = SmallCfg<S>::NMAX; };
constexpr int AED_THREADS = 256;

template <class S>
static size_t aed_smem_bytes() {
  constexpr int LD = AedCfg<S>::NW + 1;
  return (size_t)2 * LD * AedCfg<S>::NW * sizeof(S) + 64;
}

// one Householder step of the CTA: reflector (I - tau v v^H) with v = vb[r0..r1] (vb[r0] = 1)
//   left:  T[r0..r1, c0..nw-1] <- H^H (.)
//   right: T[0..r1, r0..r1] <- (.) H ;  V[0..nw-1, r0..r1] <- (.) H
template <class S, int LD>
__device__ void aed_reflect(S* T, S* V, int nw, int r0, int r1, int c0, const S* vb, S tau) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const S ctau = conj(tau);
  for (int c = c0 + tid; c < nw; c += nt) {
    S w = S(0);
    for (int r = r0; r <= r1; r++) w = fmacc(vb[r], T[r + c * LD], w);
    w = ctau * w;
    for (int r = r0; r <= r1; r++) T[r + c * LD] = T[r + c * LD] - vb[r] * w;
  }
  __syncthreads();
  for (int e = tid; e < (r1 + 1) + nw; e += nt) {
    S* M = e <= r1 ? T : V;
    const int i = e <= r1 ? e : e - r1 - 1;
    S w = S(0);
    for (int r = r0; r <= r1; r++) w = fmac(M[i + r * LD], vb[r], w);
    w = tau * w;
    for (int r = r0; r <= r1; r++) M[i + r * LD] = M[i + r * LD] - w * conj(vb[r]);
  }
  __syncthreads();
}

// T, V: Schur form and Schur vectors of the window (global, ld nw), produced by
// schur_small_launch; H: the full matrix; window = rows/cols [kwtop, kwtop + nw).
// Outputs: info[0] = nd (deflated), info[1] = ls (undeflated), info[2] = 1 if the
// window was written back (then Vout holds V, ld nw, for apply_z); wr/wi = the ls
// undeflated eigenvalues, bottom-most first (2x2 pairs adjacent).
template <class S>
__global__ void __launch_bounds__(AED_THREADS) aed_kernel(int nw, const S* Tg, S* Vg, S* H, int ldh, int kwtop,
                                                          int lo, typename tr<S>::R* wr, typename tr<S>::R* wi,
                                                          int* info, int gmax, const int* sinfo) {
  typedef typename tr<S>::R R;
  typedef typename wide<S>::T D;
  constexpr int LD = AedCfg<S>::NW + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* T = (S*)smem_raw;
  S* V = T + (size_t)LD * AedCfg<S>::NW;
  __shared__ S Qs[16];
  __shared__ S vb[AedCfg<S>::NW + 4];
  __shared__ S sh_tau, sh_beta;
  __shared__ int sh_ns, sh_ok;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const R u = tr<S>::u();
  if (sinfo[0] != 0) {  // the window's Schur form did not converge: no deflation, no shifts
    if (tid == 0) { info[0] = 0; info[1] = 0; info[2] = 0; }
    return;
  }
  for (int e = tid; e < nw * nw; e += nt) {
    const int i = e % nw, j = e / nw;
    T[i + j * LD] = Tg[e];
    V[i + j * LD] = Vg[e];
  }
  const S s = kwtop > lo ? H[kwtop + (size_t)(kwtop - 1) * ldh] : S(0);
  __syncthreads();
#define TT(i, j) T[(i) + (j) * LD]
#define VV(i, j) V[(i) + (j) * LD]
  // ---------------- deflation check (warp 0) --------------------------------
  if (warp == 0) {
    const int ns = aed_deflate_warp<S, LD>(T, V, nw, s, gmax, lane, Qs, &sh_ok);
    if (lane == 0) sh_ns = ns;
  }
  __syncthreads();
  const int ns = sh_ns, nd = nw - ns;
  // eigenvalues of the undeflated part, bottom-most first
  if (tid == 0) {
    int cnt = 0;
    for (int i = ns - 1; i >= 0;) {
      if (!tr<S>::cx && i > 0 && !iszero(TT(i, i - 1))) {
        R w4[4];
        eig2<S>(TT(i - 1, i - 1), TT(i - 1, i), TT(i, i - 1), TT(i, i), w4);
        wr[cnt] = w4[0]; wi[cnt] = w4[1]; wr[cnt + 1] = w4[2]; wi[cnt + 1] = w4[3];
        cnt += 2; i -= 2;
      } else {
        wr[cnt] = re(TT(i, i)); wi[cnt] = im(TT(i, i));
        cnt += 1; i -= 1;
      }
    }
    info[0] = nd;
    info[1] = ns;
    info[2] = nd > 0 ? 1 : 0;
  }
  if (nd == 0) return;  // nothing deflated: H stays as it was (like xLAQR3)
  // ---------------- spike reflection + Hessenberg re-reduction ----------------
  // the deflated spike entries are dropped; the undeflated ones w_j = s conj(V(0, j))
  if (ns > 1) {
    if (tid < 32) {
      R sn = 0;
      for (int r = 1 + lane; r < ns; r += 32) sn += abs2(s * conj(VV(0, r)));
      sn = warp_sum(sn);
      if (lane == 0) {
        const S x0 = s * conj(VV(0, 0));
        if (sn == R(0) && im(x0) == R(0)) {
          sh_tau = S(0); sh_beta = x0;
        } else {
          const R nrm = sqrt(abs2(x0) + sn);
          const R b = re(x0) >= R(0) ? -nrm : nrm;
          sh_beta = mk<S>(b);
          sh_tau = (mk<S>(b) - x0) / mk<S>(b);
          vb[AedCfg<S>::NW + 1] = S(1) / (x0 - mk<S>(b));
        }
      }
    }
    __syncthreads();
    if (!iszero(sh_tau)) {
      const S scal = vb[AedCfg<S>::NW + 1];
      for (int r = tid; r < ns; r += nt) vb[r] = r == 0 ? S(1) : (s * conj(VV(0, r))) * scal;
      __syncthreads();
      aed_reflect<S, LD>(T, V, nw, 0, ns - 1, 0, vb, sh_tau);
    }
    // Hessenberg reduction of T[0:ns, 0:ns] (columns 0..ns-3)
    for (int kc = 0; kc + 2 < ns; kc++) {
      if (tid < 32) {
        R sn = 0;
        for (int r = kc + 2 + lane; r < ns; r += 32) sn += abs2(TT(r, kc));
        sn = warp_sum(sn);
        if (lane == 0) {
          const S x0 = TT(kc + 1, kc);
          if (sn == R(0) && im(x0) == R(0)) {
            sh_ok = 0;
          } else {
            const R nrm = sqrt(abs2(x0) + sn);
            const R b = re(x0) >= R(0) ? -nrm : nrm;
            Qs[0] = mk<S>(b);
            Qs[1] = (mk<S>(b) - x0) / mk<S>(b);
            Qs[2] = S(1) / (x0 - mk<S>(b));
            sh_ok = 1;
          }
        }
      }
      __syncthreads();
      if (!sh_ok) { __syncthreads(); continue; }
      const S tau = Qs[1], scal = Qs[2], beta = Qs[0];
      for (int r = kc + 1 + tid; r < ns; r += nt) vb[r] = r == kc + 1 ? S(1) : TT(r, kc) * scal;
      __syncthreads();
      aed_reflect<S, LD>(T, V, nw, kc + 1, ns - 1, kc + 1, vb, tau);
      if (tid == 0) TT(kc + 1, kc) = beta;
      for (int r = kc + 2 + tid; r < ns; r += nt) TT(r, kc) = S(0);
      __syncthreads();
    }
  }
  // ---------------- write back ------------------------------------------------
  const S newsub = ns > 1 ? sh_beta : (ns == 1 ? s * conj(VV(0, 0)) : S(0));
  for (int e = tid; e < nw * nw; e += nt) {
    const int i = e % nw, j = e / nw;
    S v = TT(i, j);
    if (i > j + 1 || (i == j + 1 && i == ns)) v = S(0);
    H[(kwtop + i) + (size_t)(kwtop + j) * ldh] = v;
    Vg[e] = VV(i, j);
  }
  if (tid == 0 && kwtop > lo) H[kwtop + (size_t)(kwtop - 1) * ldh] = newsub;
#undef TT
#undef VV
}

}  // namespace msy
