// schur.cuh -- A = U T U^H on the device (replaces `schur`, pkg/src/mpsylv/linalg.py:518-577).
//
//   m <= NMIN : schur_small_kernel (Hessenberg + double-shift QR in one CTA's smem)
//   m >  NMIN : hessenberg_blocked, then a host-driven loop of
//               scan (deflation) -> shifts (trailing block eigenvalues) -> multishift sweep
//               (window chase + Z application), finishing blocks <= NMIN in one CTA.
// Status: 0 ok, 3 = iteration limit (IterationLimitError, linalg.py:552-554).
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "hessenberg.cuh"
#include "multishift.cuh"
#include "schur_small.cuh"
#include "schur_mss.cuh"

#include <chrono>
#include <cstdlib>

namespace msy {

template <class S>
struct SchurWs {
  typedef typename tr<S>::R R;
  HessWs<S> hw;
  S* Z;       // 2 x ZMAX^2: window factors, double-buffered across overlapping windows
  S* sblk;    // trailing block copy
  R* wr;
  R* wi;
  R* shifts;  // 4 per bulge
  int* dinfo; // small device ints
  static void carve(Arena& ar, int m, SchurWs& w) {
    if (m > SmallCfg<S>::NMAX) HessWs<S>::carve(ar, m, w.hw);
    w.Z = ar.get<S>(2 * ZMAX * ZMAX);
    w.sblk = ar.get<S>(128 * 128);
    w.wr = ar.get<R>(256);
    w.wi = ar.get<R>(256);
    w.shifts = ar.get<R>(4 * 64);
    w.dinfo = ar.get<int>(64);
  }
};

struct SchurStats {
  int status, sweeps, small_calls, windows;
  double ms_hess, ms_scan, ms_small, ms_shift, ms_sweep;  // filled when MSY_SCHUR_TIMING=1
};

// diagnostic phase timer: synchronises the stream at each mark (only when enabled)
struct PhaseTimer {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(cudaStream_t s) : on(getenv("MSY_SCHUR_TIMING") != nullptr), st(s) { t = now(); }
  static std::chrono::steady_clock::time_point now() { return std::chrono::steady_clock::now(); }
  void lap(double* acc) {
    if (!on) return;
    host_sync(st);
    auto t2 = now();
    *acc += std::chrono::duration<double, std::milli>(t2 - t).count();
    t = t2;
  }
};

// auxiliary stream + events used to overlap the window chases (one CTA) with the
// off-window Z applications (many CTAs).  Owned by a solve lane (solver.cu) or,
// for direct sylv_schur calls, by the calling host thread.
struct SweepCtx {
  cudaStream_t aux = nullptr;  // nullptr: serial mode (everything on the caller's stream)
  cudaEvent_t evC = nullptr, evN = nullptr, evD = nullptr;
  int dev = -1;
  void ensure() {
    int d = 0;
    cudaGetDevice(&d);
    if (aux != nullptr && dev == d) return;
    cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&evC, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evN, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evD, cudaEventDisableTiming);
    dev = d;
  }
};
inline SweepCtx* sweep_ctx() {
  thread_local SweepCtx c;
  c.ensure();
  return &c;
}

// One multishift sweep over the active block [lo, hi] with nb bulges.
// Windows are planned on the host (bulge positions are a function of the step).
// Pipeline: chase(k+1) on `st` runs concurrently with the far part of apply(k)
// on `aux`; the near part (columns the next window will load) runs first.
template <class S>
int ms_sweep(int m, S* H, int ldh, S* U, int ldu, int lo, int hi, int nb, const typename tr<S>::R* shifts, S* Zbuf,
             cudaStream_t st, int* nwin, SweepCtx* sc) {
  constexpr int W = MsCfg<S>::W;
  const size_t smem_max = (size_t)(W + 1) * (2 * W + 1) * sizeof(S);  // H window + dummy column, Z
  MSY_SMEM_ATTR_ONCE(chase_kernel<S>, smem_max);
  const int span = hi - lo;
  const long Tn = 4L * (nb - 1) + span;
  auto Lf = [&](long t) {
    long jt = std::min<long>(nb - 1, t / 4);
    long P = lo - 1 + t - 4 * jt;
    return (int)std::max<long>(P, lo);
  };
  auto Uf = [&](long t) {
    long x = t - (span - 1);
    long jh = x > 0 ? (x + 3) / 4 : 0;
    long P = lo - 1 + t - 4 * jh;
    return (int)std::min<long>(P + 4, hi);
  };
  struct Win { int ws, we, t0, t1; };
  Win wins[4096];
  int nwins = 0;
  for (long t = 0; t < Tn;) {
    int ws = Lf(t);
    int we = std::min(ws + W, hi + 1);
    long t1 = t;
    while (t1 < Tn && Uf(t1) <= we - 1) t1++;
    if (t1 == t || nwins >= 4096) return -5;
    wins[nwins++] = {ws, we, (int)t, (int)t1};
    t = t1;
  }
  const int nthr = 32 * std::max(nb, 4);
  auto chase = [&](int k) -> int {
    const Win& w = wins[k];
    int nw = w.we - w.ws;
    chase_kernel<S><<<1, nthr, (size_t)(nw + 1) * (2 * nw + 1) * sizeof(S), st>>>(H, ldh, lo, hi, nb, shifts, w.ws, w.we,
                                                                            w.t0, w.t1, Zbuf + (k & 1) * ZMAX * ZMAX);
    MSY_LAUNCH_CK();
    if (sc->aux) MSY_CK(cudaEventRecord(sc->evC, st));
    return 0;
  };
  int rc = chase(0);
  if (rc) return rc;
  if (sc->aux == nullptr) {  // serial lane (batched executor): one stream, one Z application per window
    for (int k = 0; k < nwins; k++) {
      const Win& w = wins[k];
      rc = apply_z<S>(m, w.we - w.ws, Zbuf + (k & 1) * ZMAX * ZMAX, H, ldh, U, ldu, w.ws, st);
      if (rc) return rc;
      if (k + 1 < nwins && (rc = chase(k + 1))) return rc;
      if (nwin) (*nwin)++;
    }
    return 0;
  }
  for (int k = 0; k < nwins; k++) {
    const Win& w = wins[k];
    const int nw = w.we - w.ws;
    const S* Zk = Zbuf + (k & 1) * ZMAX * ZMAX;
    const int cn = std::min(w.we + W, m);
    MSY_CK(cudaStreamWaitEvent(sc->aux, sc->evC, 0));
    rc = apply_z_regions<S>(m, nw, Zk, H, ldh, nullptr, ldu, w.ws, w.we, cn, 0, sc->aux);  // near
    if (rc) return rc;
    MSY_CK(cudaEventRecord(sc->evN, sc->aux));
    rc = apply_z_regions<S>(m, nw, Zk, H, ldh, U, ldu, w.ws, cn, m, w.ws, sc->aux);        // far
    if (rc) return rc;
    if (k + 1 < nwins) {
      MSY_CK(cudaStreamWaitEvent(st, sc->evN, 0));
      rc = chase(k + 1);
      if (rc) return rc;
    }
    if (nwin) (*nwin)++;
  }
  MSY_CK(cudaEventRecord(sc->evD, sc->aux));
  MSY_CK(cudaStreamWaitEvent(st, sc->evD, 0));
  return 0;
}

// In place: A (m x m, lda) -> T; U (m x m, ldu) = Schur vectors.
template <class S>
int schur_device(int m, S* A, int lda, S* U, int ldu, SchurWs<S>& w, cudaStream_t st, SchurStats* stats,
                 SweepCtx* sc = nullptr) {
  if (!sc) sc = sweep_ctx();
  typedef typename tr<S>::R R;
  constexpr int NMIN = SmallCfg<S>::NMAX;
  SchurStats loc = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (m <= NMIN) {
    int rc = schur_small_launch<S>(m, A, lda, U, ldu, SS_HESS | SS_WANTZ, nullptr, nullptr, w.dinfo, st);
    if (rc) return rc;
    int hinfo[2];
    MSY_CK(d2h(hinfo, w.dinfo, sizeof(hinfo), st));
    MSY_CK(host_sync(st));
    loc.status = hinfo[0];
    loc.sweeps = hinfo[1];
    loc.small_calls = 1;
    if (stats) *stats = loc;
    return 0;
  }
  PhaseTimer pt(st);
  int rc = hessenberg_blocked<S>(m, A, lda, U, ldu, w.hw, st);
  if (rc) return rc;
  pt.lap(&loc.ms_hess);
  int hi = m - 1, stag = 0, last_hi = m;
  const int limit = 30 * m;
  while (true) {
    scan_kernel<S><<<1, 1024, 0, st>>>(m, A, lda, U, ldu, hi, w.dinfo);
    MSY_LAUNCH_CK();
    int hinfo[4];
    MSY_CK(d2h(hinfo, w.dinfo, 2 * sizeof(int), st));
    MSY_CK(host_sync(st));
    hi = hinfo[0];
    int lo = hinfo[1];
    pt.lap(&loc.ms_scan);
    if (hi < 0) break;
    if (hi < last_hi) { stag = 0; last_hi = hi; } else stag++;
    int sz = hi - lo + 1;
    if (sz <= NMIN) {
      S* blk = A + lo + (size_t)lo * lda;
      rc = schur_small_launch<S>(sz, blk, lda, w.Z, sz, SS_WANTZ, nullptr, nullptr, w.dinfo + 8, st);
      if (rc) return rc;
      rc = apply_z<S>(m, sz, w.Z, A, lda, U, ldu, lo, st);
      if (rc) return rc;
      int sinfo[2];
      MSY_CK(d2h(sinfo, w.dinfo + 8, 2 * sizeof(int), st));
      MSY_CK(host_sync(st));
      pt.lap(&loc.ms_small);
      loc.small_calls++;
      loc.sweeps += sinfo[1];
      if (sinfo[0]) { loc.status = sinfo[0]; break; }
      hi = lo - 1;
      last_hi = hi + 1;
      stag = 0;
      if (hi < 0) break;
      continue;
    }
    if (loc.sweeps >= limit) { loc.status = ST_ITERLIMIT; break; }
    int nb = std::min(MsCfg<S>::NB, std::max(1, (sz - 8) / 8));
    int ns = 2 * nb;
    bool exc = (stag > 0 && stag % 6 == 0);
    if (!exc) {
      const S* src = A + (hi - ns + 1) + (size_t)(hi - ns + 1) * lda;
      copy_block_kernel<S><<<dim3(cdiv(ns, 128), ns), 128, 0, st>>>(ns, src, lda, w.sblk, ns);
      MSY_LAUNCH_CK();
      rc = schur_small_launch<S>(ns, w.sblk, ns, nullptr, 0, SS_EIGONLY, w.wr, w.wi, w.dinfo + 16, st);
      if (rc) return rc;
    }
    pair_shifts_kernel<S><<<1, 32, 0, st>>>(ns, w.wr, w.wi, nb, w.shifts, exc ? 1 : 0, A, lda, lo, hi, w.dinfo + 24);
    MSY_LAUNCH_CK();
    pt.lap(&loc.ms_shift);
    rc = ms_sweep<S>(m, A, lda, U, ldu, lo, hi, nb, w.shifts, w.Z, st, &loc.windows, sc);
    if (rc) return rc;
    pt.lap(&loc.ms_sweep);
    loc.sweeps++;
  }
  if (stats) *stats = loc;
  return 0;
}

}  // namespace msy
