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
#include "util.cuh"

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace msy {

#ifndef MSY_SUBMAX
#define MSY_SUBMAX 640  // detached blocks up to this order are factored beside the sweeps (0: off)
#endif
#ifndef MSY_SUB_PRIO
#define MSY_SUB_PRIO 1  // helper streams: 0 least, 1 middle, 2 greatest priority
#endif
#ifndef MSY_SUB_HELPERS
#define MSY_SUB_HELPERS 3
#endif
constexpr int SUB_NH = MSY_SUB_HELPERS;  // helper host threads (and block workspaces) per Schur factorisation

// workspace of one QR loop (deflation scan, shifts, sweeps, endgame blocks)
template <class S>
struct SchurLoopWs {
  typedef typename tr<S>::R R;
  S* Z;       // 2 x ZMAX^2: window factors, double-buffered across overlapping windows
  S* sblk;    // trailing block copy
  R* wr;
  R* wi;
  R* shifts;  // 4 per bulge
  int* dinfo; // small device ints
  S* Zend;    // Schur vectors of the endgame blocks (sum of block orders^2 <= NMAX * m)
  int* dend;  // their [status, sweeps] words
  static void carve(Arena& ar, int m, SchurLoopWs& w) {
    w.Z = ar.get<S>((size_t)4 * KMAX * ZMAX * ZMAX);  // second half: row-major copies (ZT_DELTA)
    w.sblk = ar.get<S>((size_t)EigCfg<S>::NMAX * EigCfg<S>::NMAX);
    w.wr = ar.get<R>(256);
    w.wi = ar.get<R>(256);
    w.shifts = ar.get<R>(4 * 128);
    w.dinfo = ar.get<int>(64);
    w.Zend = m > SmallCfg<S>::NMAX ? ar.get<S>((size_t)SmallCfg<S>::NMAX * (m + SmallCfg<S>::NMAX)) : nullptr;
    w.dend = m > SmallCfg<S>::NMAX ? ar.get<int>(2 * (size_t)(m + 1)) : nullptr;
  }
};

// Detached mid-size blocks (NMAX < order <= MSY_SUBMAX) are factored in place by a helper host
// thread beside the sweeps of the remaining matrix (schur_device): `sub` is that QR loop's own
// workspace, Zsub holds the blocks' Schur vectors (sum of orders^2 <= SUBMAX * m) and subtmp
// the out-of-place product of one block's Z with its H rows / U columns.
template <class S>
struct SchurWs : SchurLoopWs<S> {
  HessWs<S> hw;
  SchurLoopWs<S> sub[SUB_NH];
  S* Zsub = nullptr;
  S* subtmp[SUB_NH] = {};
  static void carve(Arena& ar, int m, SchurWs& w) {
    if (m > SmallCfg<S>::NMAX) HessWs<S>::carve(ar, m, w.hw);
    SchurLoopWs<S>::carve(ar, m, w);
    w.Zsub = nullptr;
    if (MSY_SUBMAX > SmallCfg<S>::NMAX && m > MSY_SUBMAX) {
      w.Zsub = ar.get<S>((size_t)MSY_SUBMAX * m);
      for (int i = 0; i < SUB_NH; i++) {
        SchurLoopWs<S>::carve(ar, MSY_SUBMAX, w.sub[i]);
        w.subtmp[i] = ar.get<S>((size_t)MSY_SUBMAX * m);
      }
    }
  }
};

struct SchurStats {
  int status, sweeps, small_calls, windows;
  double ms_hess, ms_scan, ms_small, ms_shift, ms_sweep;  // filled when MSY_SCHUR_TIMING=1
  int aed_calls, aed_deflated, ms_sweeps;                  // AED windows, eigenvalues they deflated, QR sweeps
  double ms_aed;
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
// Persistent helper host threads of one Schur factorisation: they run the QR loops of detached
// mid-size blocks (shared FIFO), each on its own stream, while the owner keeps sweeping the rest.
struct SubHelper {
  static constexpr int NH = SUB_NH;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::function<void(int)>> q;
  int pending = 0;
  cudaStream_t st[NH] = {};
  cudaEvent_t ev1[NH] = {};
  std::vector<cudaEvent_t> evpool;  // one "block detached" event per job of the current loop
  explicit SubHelper(int dev) {
    int lo_pri = 0, hi_pri = 0;
    cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
    for (int i = 0; i < NH; i++) {
      cudaStreamCreateWithPriority(&st[i], cudaStreamNonBlocking, MSY_SUB_PRIO == 2 ? hi_pri : (MSY_SUB_PRIO == 0 ? lo_pri : (lo_pri + hi_pri) / 2));
      cudaEventCreateWithFlags(&ev1[i], cudaEventDisableTiming);
      std::thread([this, dev, i]() {
        cudaSetDevice(dev);
        for (;;) {
          std::function<void(int)> j;
          {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [this] { return !q.empty(); });
            j = std::move(q.front());
            q.pop_front();
          }
          j(i);
          {
            std::lock_guard<std::mutex> lk(mu);
            pending--;
          }
          cv.notify_all();
        }
      }).detach();  // process lifetime, like the pair's side worker
    }
  }
  cudaEvent_t job_event(size_t k) {  // owner thread only
    while (evpool.size() <= k) {
      cudaEvent_t e = nullptr;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      evpool.push_back(e);
    }
    return evpool[k];
  }
  void push(std::function<void(int)> j) {
    {
      std::lock_guard<std::mutex> lk(mu);
      q.push_back(std::move(j));
      pending++;
    }
    cv.notify_all();
  }
  void drain() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return pending == 0; });
  }
};

struct SweepCtx {
  cudaStream_t aux = nullptr;  // nullptr: serial mode (everything on the caller's stream)
  cudaStream_t eg = nullptr;   // endgame blocks (one-CTA Schur + row-side Z), beside the sweeps
  cudaEvent_t evC = nullptr, evN = nullptr, evD = nullptr, evE0 = nullptr, evE1 = nullptr;
  int dev = -1;
  SubHelper* helper = nullptr;  // created on first use (never for serial lanes)
  SubHelper* sub_helper() {
    if (!helper) helper = new SubHelper(dev);
    return helper;
  }
  void ensure() {
    int d = 0;
    cudaGetDevice(&d);
    if (aux != nullptr && dev == d) return;
    helper = nullptr;  // a helper of another device keeps its own stream
    cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&eg, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&evC, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evN, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evD, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evE0, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evE1, cudaEventDisableTiming);
    dev = d;
  }
};
inline SweepCtx* sweep_ctx() {
  thread_local SweepCtx c;
  c.ensure();
  return &c;
}

// One multishift sweep over the active block [lo, hi]: K chains of nb bulges each
// (chain c uses shifts[4 nb c ..]).  Windows are planned on the host (bulge positions
// are a function of the step); every chain walks the same window sequence, chain c
// D windows behind chain c-1, D the smallest lag that keeps concurrent windows
// disjoint.
//   K = 1: chase(k+1) on `st` overlaps the far part of apply(k) on `aux`; the near
//          part (columns the next window loads) runs first.
//   K > 1: per time step one launch chases every active chain (one CTA each), then
//          one launch applies all their Z to the rows right of the windows and one to
//          the columns above them and to U (row / column regions of different chains
//          are disjoint; a row region of one chain meets a column region of the next
//          only across the two launches).
template <class S>
int ms_sweep(int m, S* H, int ldh, S* U, int ldu, int lo, int hi, int nb, int K, const typename tr<S>::R* shifts,
             S* Zbuf, cudaStream_t st, int* nwin, SweepCtx* sc) {
  constexpr int W = MsCfg<S>::W;
  const size_t smem_max = (size_t)(W + 1) * (2 * W) * sizeof(S);  // H window + Z, stride W + 1
  MSY_SMEM_ATTR_ONCE(chase_kernel<S>, smem_max);
  if constexpr (kChase2<S>) MSY_SMEM_ATTR_ONCE(chase2_kernel, chase2_smem());
  MSY_SMEM_ATTR_ONCE(apply_z_kernel<S>, (int)applyz_smem<S>(W));
  MSY_SMEM_ATTR_ONCE(apply_z_multi_kernel<S>, (int)applyz_smem<S>(W));
  MSY_SMEM_ATTR_ONCE(apply_z_cl_kernel<S>, (int)azc_smem<S>());
  constexpr int azc_mode = MSY_AZC;
  if (K < 1 || K > KMAX) return -5;
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
  static thread_local Win wins[4096];
  int nwins = 0;
  for (long t = 0; t < Tn;) {
    int ws = Lf(t);
    int we = std::min(ws + W, hi + 1);
    long t1 = t;
    while (t1 < Tn && Uf(t1) <= we - 1) t1++;
    if (t1 == t || nwins >= 4096 || t1 - t > W + 4 * nb) return -5;  // (a window never holds more steps)
    wins[nwins++] = {ws, we, (int)t, (int)t1};
    t = t1;
  }
  const int nthr = 32 * std::max(nb, 4);
  if (K > 1) {
    int D = 1;
    for (bool ok = false; !ok; D++) {
      ok = true;
      for (int k = 0; k + D < nwins && ok; k++) ok = wins[k].we <= wins[k + D].ws;
      if (ok) break;
    }
    // per time step tau, on st: chase (all chains) -> near rows -> near columns; on aux:
    // far rows -> far columns + U, overlapping the next chase.  near(tau) waits for
    // far(tau-1) (their regions can meet); Z buffers alternate with tau.
    constexpr bool mc_serial = MSY_MC_SERIAL != 0;
    const bool ovl = sc->aux != nullptr && !mc_serial;
    cudaStream_t fst = ovl ? sc->aux : st;
    for (int tau = 0; tau < nwins + (K - 1) * D; tau++) {
      ChaseJobs<S> cj;
      ApplyJobs<S> jr[2] = {}, jc[2] = {};  // [0] near, [1] far
      int nj = 0;
      // Consistency: a block hit by one chain's row update and another's column update must
      // see the whole row update first, so near rows reach past every window of this step;
      // far parts stay clear of the next step's windows (rows >= rstar, columns < cstar).
      int we_max = 0, rstar = m, cstar = 0;
      for (int c = 0; c < K; c++) {
        const int k = tau - c * D, k1 = k + 1;
        if (k >= 0 && k < nwins) we_max = std::max(we_max, wins[k].we);
        if (k1 >= 0 && k1 < nwins) { rstar = std::min(rstar, wins[k1].ws); cstar = std::max(cstar, wins[k1].we); }
      }
      for (int c = 0; c < K; c++) {
        const int k = tau - c * D;
        if (k < 0 || k >= nwins) continue;
        const Win& w = wins[k];
        const int nz = w.we - w.ws;
        S* Zc = Zbuf + ((size_t)2 * c + (tau & 1)) * ZMAX * ZMAX;
        cj.ws[nj] = w.ws; cj.we[nj] = w.we; cj.t0[nj] = w.t0; cj.t1[nj] = w.t1;
        cj.shifts[nj] = shifts + 4 * nb * c;
        cj.Z[nj] = Zc;
        const int cn = std::min(m, std::max({w.we + W, we_max, cstar}));
        const int rn = std::max(0, std::min(w.ws - W, rstar));
        for (int f = 0; f < 2; f++) {
          ApplyJobs<S>& r = jr[f];
          r.zmask[nj] = jc[f].zmask[nj] = kChase2<S> ? 1 : 0;
          r.nz[nj] = nz; r.Z[nj] = Zc; r.r0[nj] = w.ws; r.rR1[nj] = 0; r.mU[nj] = 0;
          r.cL0[nj] = f == 0 ? w.we : cn;
          r.cL1[nj] = f == 0 ? cn : m;
        }
        // column regions: rows [rn, ws) (near) and [0, rn) + U (far)
        jc[0].nz[nj] = nz; jc[0].Z[nj] = Zc; jc[0].r0[nj] = w.ws; jc[0].cL0[nj] = jc[0].cL1[nj] = 0;
        jc[0].rR1[nj] = w.ws; jc[0].mU[nj] = 0;
        jc[1].nz[nj] = nz; jc[1].Z[nj] = Zc; jc[1].r0[nj] = w.ws; jc[1].cL0[nj] = jc[1].cL1[nj] = 0;
        jc[1].rR1[nj] = rn; jc[1].mU[nj] = m;
        jc[0].rlo[nj] = rn;
        if (!ovl) {  // one stream (batched lanes): whole row regions, then whole column regions + U
          jr[0].cL1[nj] = m; jr[1].cL0[nj] = jr[1].cL1[nj] = 0;
          jc[0].rlo[nj] = 0; jc[0].mU[nj] = m; jc[1].rR1[nj] = 0; jc[1].mU[nj] = 0;
        }
        nj++;
      }
      if (nj == 0) continue;
      for (int f = 0; f < 2; f++) {
        jr[f].n = jc[f].n = nj;
        jr[f].start[0] = jc[f].start[0] = 0;
        for (int j = 0; j < nj; j++) {
          jr[f].start[j + 1] = jr[f].start[j] + (jr[f].cL1[j] > jr[f].cL0[j] ? cdiv(jr[f].cL1[j] - jr[f].cL0[j], 32) : 0);
          jc[f].start[j + 1] = jc[f].start[j] + (jc[f].rR1[j] > jc[f].rlo[j] ? cdiv(jc[f].rR1[j] - jc[f].rlo[j], 32) : 0) +
                               cdiv(jc[f].mU[j], 32);
        }
      }
      {
        KScope ks(KC_CHASE, 0, st);
        if constexpr (kChase2<S>) chase2_kernel<<<2 * nj, CZ_THREADS, chase2_smem(), st>>>(H, ldh, lo, hi, nb, cj);
        else chase_kernel<S><<<nj, nthr, smem_max, st>>>(H, ldh, lo, hi, nb, cj);
        MSY_LAUNCH_CK();
      }
      if (ovl && tau > 0) MSY_CK(cudaStreamWaitEvent(st, sc->evD, 0));  // far(tau-1) done
      for (int f = 0; f < 2; f++) {
        cudaStream_t s2 = f == 0 ? st : fst;
        if (f == 1 && ovl) {
          MSY_CK(cudaEventRecord(sc->evN, st));
          MSY_CK(cudaStreamWaitEvent(fst, sc->evN, 0));
        }
        // cluster-split application (apply_z_cl_kernel) for the near parts on the chase's
        // critical path (MSY_AZC: 0 off, 1 near only, 2 near and far)
        const bool cl = azc_mode >= 2 || (azc_mode == 1 && f == 0);
        for (int rc_ = 0; rc_ < 2; rc_++) {
          const ApplyJobs<S>& jb = rc_ == 0 ? jr[f] : jc[f];
          if (jb.start[nj] <= 0) continue;
          KScope ks(KC_APPLYZ, applyz_flops<S>(jb), s2);
          if constexpr (kFarKernel<S>) {
            if (f == 1 && MSY_FAR_MIN_TILES >= 0) {  // far parts: the throughput kernel
              int rcf = apply_z_far_launch(H, ldh, U, ldu, jb, s2);
              if (rcf) return rcf;
              continue;
            }
          }
          if (cl)
            apply_z_cl_kernel<S><<<jb.start[nj] * Azc<S>::N, AZC_THREADS, azc_smem<S>(), s2>>>(H, ldh, U, ldu, jb);
          else
            apply_z_multi_kernel<S><<<jb.start[nj], 256, applyz_smem<S>(W), s2>>>(H, ldh, U, ldu, jb);
          MSY_LAUNCH_CK();
        }
      }
      if (ovl) MSY_CK(cudaEventRecord(sc->evD, fst));
      if (nwin) (*nwin) += nj;
    }
    if (ovl) MSY_CK(cudaStreamWaitEvent(st, sc->evD, 0));
    return 0;
  }
  auto chase = [&](int k) -> int {
    const Win& w = wins[k];
    ChaseJobs<S> cj;
    cj.ws[0] = w.ws; cj.we[0] = w.we; cj.t0[0] = w.t0; cj.t1[0] = w.t1;
    cj.shifts[0] = shifts;
    cj.Z[0] = Zbuf + (k & 1) * ZMAX * ZMAX;
    {
      KScope ks(KC_CHASE, 0, st);
      if constexpr (kChase2<S>) chase2_kernel<<<2, CZ_THREADS, chase2_smem(), st>>>(H, ldh, lo, hi, nb, cj);
      else chase_kernel<S><<<1, nthr, smem_max, st>>>(H, ldh, lo, hi, nb, cj);
      MSY_LAUNCH_CK();
    }
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

// Detached blocks handed to the helper thread: where they sit, where their Schur vectors are,
// and what their QR loop reported.
struct SubBlock { int lo, sz; size_t zoff; int rc, status, sweeps; };
template <class S>
struct SubPlan {  // set for the top-level loop of a matrix that can spawn block jobs
  SchurLoopWs<S>* ws;  // [SubHelper::NH]
  S* Zsub;
  S* const* tmp;       // [SubHelper::NH]
};

// C <- op(Z) C (left = true: rows x cols block C, Z rows x rows applied as Z^H) or C <- C Z
// (left = false: Z cols x cols) through the out-of-place buffer tmp.
template <class S>
int apply_block_z(bool left, int rows, int cols, const S* Z, int ldz, S* C, int ldc, S* tmp, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  int rc = left ? gemm<S>('C', 'N', rows, cols, rows, S(1), Z, ldz, C, ldc, S(0), tmp, rows, st)
                : gemm<S>('N', 'N', rows, cols, cols, S(1), C, ldc, Z, ldz, S(0), tmp, rows, st);
  if (rc) return rc;
  return copy2d<S>(rows, cols, tmp, rows, C, ldc, st);
}

// The QR iteration on an upper Hessenberg matrix, in place: A (m x m, lda) -> T, U (m x m, ldu)
// <- U * (accumulated transformations).  `plan` (top level only) lets detached mid-size blocks
// run on the helper thread.
template <class S>
int schur_qr_loop(int m, S* A, int lda, S* U, int ldu, SchurLoopWs<S>& w, cudaStream_t st, SchurStats& loc,
                  SweepCtx* sc, PhaseTimer& pt, const SubPlan<S>* plan) {
  typedef typename tr<S>::R R;
  constexpr int NMIN = SmallCfg<S>::NMAX;
  int rc = 0;
  int hi = m - 1, stag = 0, last_hi = m;
  std::vector<SubBlock> subs;
  subs.reserve(256);  // jobs hold pointers into it: never reallocated while they run (<= m / NMIN entries)
  size_t zsoff = 0;
  const bool sub_ok = plan != nullptr && plan->Zsub != nullptr && sc->aux != nullptr && MSY_SUBMAX > NMIN;
  SubHelper* helper = nullptr;
  int dev = 0;
  if (sub_ok) cudaGetDevice(&dev);
  const bool blocking = host_sync_blocking();
  struct DrainGuard {  // jobs reference this frame: never leave it with jobs in flight
    SubHelper*& h;
    ~DrainGuard() { if (h) h->drain(); }
  } drain_guard{helper};
  const int limit = 30 * m;
  // Endgame blocks (order <= NMAX split off below the active block) are solved beside the
  // sweeps on the endgame stream: their one-CTA Schur, the row-side Z (H rows of the block,
  // columns to its right) and U run at once; the column-side update (rows above the block)
  // is deferred to the end.  Sweeps only multiply rows above the block from the left, so the
  // deferred right multiplication commutes with them and no entry is written concurrently.
  constexpr bool sync_end = MSY_SYNC_ENDGAME != 0;
  const bool async_end = sc->aux != nullptr && sc->eg != nullptr && !sync_end && w.Zend != nullptr;
  struct Deferred { int lo, sz; size_t zoff; };
  std::vector<Deferred> defs;
  size_t zoff = 0;
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
    if (sub_ok && sz > NMIN && sz <= MSY_SUBMAX && subs.size() < 256 &&
        zsoff + (size_t)sz * sz <= (size_t)MSY_SUBMAX * m) {
      // detached block: its QR loop, the row side of its Z and U run on the helper's stream;
      // the column side (rows above the block) is deferred to the end like the endgame blocks'
      if (!helper) helper = sc->sub_helper();
      cudaEvent_t evj = helper->job_event(subs.size());
      MSY_CK(cudaEventRecord(evj, st));
      subs.push_back({lo, sz, zsoff, 0, 0, 0});
      SubBlock* sb = &subs.back();
      zsoff += (size_t)sz * sz;
      SubHelper* hp = helper;
      const SubPlan<S> pl = *plan;
      helper->push([=](int hidx) {
        host_sync_blocking() = blocking;
        cudaStream_t hs = hp->st[hidx];
        cudaStreamWaitEvent(hs, evj, 0);
        S* blk = A + sb->lo + (size_t)sb->lo * lda;
        S* Zb = pl.Zsub + sb->zoff;
        const int bs = sb->sz, b0 = sb->lo;
        set_identity_kernel<S><<<dim3(cdiv(bs, 256), bs), 256, 0, hs>>>(bs, bs, Zb, bs);
        __atomic_add_fetch(&launch_counter(), 1ULL, __ATOMIC_RELAXED);
        SchurStats ls = {};
        PhaseTimer pt2(hs);
        pt2.on = false;
        int r = schur_qr_loop<S>(bs, blk, lda, Zb, bs, pl.ws[hidx], hs, ls, sweep_ctx(), pt2, nullptr);
        if (!r) r = apply_block_z<S>(true, bs, m - b0 - bs, Zb, bs, A + b0 + (size_t)(b0 + bs) * lda, lda, pl.tmp[hidx], hs);
        if (!r) r = apply_block_z<S>(false, m, bs, Zb, bs, U + (size_t)b0 * ldu, ldu, pl.tmp[hidx], hs);
        sb->rc = r;
        sb->status = ls.status;
        sb->sweeps = ls.sweeps;
      });
      loc.small_calls++;
      hi = lo - 1;
      last_hi = hi + 1;
      stag = 0;
      if (hi < 0) break;
      continue;
    }
    if (sz <= NMIN && async_end) {
      S* blk = A + lo + (size_t)lo * lda;
      S* Zb = w.Zend + zoff;
      MSY_CK(cudaEventRecord(sc->evE0, st));
      MSY_CK(cudaStreamWaitEvent(sc->eg, sc->evE0, 0));
      rc = schur_small_launch<S>(sz, blk, lda, Zb, sz, SS_WANTZ, nullptr, nullptr, w.dend + 2 * defs.size(), sc->eg);
      if (rc) return rc;
      rc = apply_z_regions<S>(m, sz, Zb, A, lda, U, ldu, lo, lo + sz, m, 0, sc->eg);  // rows right + U
      if (rc) return rc;
      defs.push_back({lo, sz, zoff});
      zoff += (size_t)sz * sz;
      loc.small_calls++;
      hi = lo - 1;
      last_hi = hi + 1;
      stag = 0;
      if (hi < 0) break;
      continue;
    }
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
    constexpr int kmax_env = MSY_CHAINS;
    // bulges per chain (a chain of nb bulges spans 4 nb rows of the W-row chase window)
    const int NBc = std::max(2, std::min(MsCfg<S>::NB, MSY_NB_CHAIN > 0 ? MSY_NB_CHAIN : MsCfg<S>::NB));
    bool exc = (stag > 0 && stag % 6 == 0);
    int nb, K = 1, ns;
    nb = std::min(NBc, std::max(1, (sz - 8) / 8));
    // several chains per sweep when the active block is large and the trailing
    // block that supplies their shifts fits the one-CTA kernel
    if (nb == NBc && kmax_env > 1)
      K = std::max(1, std::min({std::min(kmax_env, KMAX), EigCfg<S>::NMAX / (2 * nb), sz / (12 * nb)}));
    ns = 2 * nb * K;
    if (!exc) {
      // the eigenvalue-only kernel stages the trailing block from A itself and writes nothing back
      S* src = A + (hi - ns + 1) + (size_t)(hi - ns + 1) * lda;
      // shifts need not be converged to working accuracy: a looser deflation tolerance
      // cuts the eigenvalue iteration roughly in half
      constexpr double stol = MSY_SHIFT_TOL;
      rc = schur_small_launch<S>(ns, src, lda, nullptr, 0, SS_EIGONLY, w.wr, w.wi, w.dinfo + 16, st,
                                 (R)std::max<double>(stol, tr<S>::u()));
      if (rc) return rc;
    }
    pair_shifts_kernel<S><<<1, 32, 0, st>>>(ns, w.wr, w.wi, nb * K, w.shifts, exc ? 1 : 0, A, lda, lo, hi,
                                            w.dinfo + 24);
    MSY_LAUNCH_CK();
    pt.lap(&loc.ms_shift);
    const double sw0 = loc.ms_sweep;
    const int nw0 = loc.windows;
    rc = ms_sweep<S>(m, A, lda, U, ldu, lo, hi, nb, K, w.shifts, w.Z, st, &loc.windows, sc);
    if (rc) return rc;
    pt.lap(&loc.ms_sweep);
    if (pt.on && getenv("MSY_SCHUR_TRACE"))
      fprintf(stderr, "sweep %d lo %d hi %d sz %d nb %d K %d wins %d ms %.3f\n", loc.ms_sweeps, lo, hi, sz, nb, K,
              loc.windows - nw0, loc.ms_sweep - sw0);
    loc.sweeps++;
    loc.ms_sweeps++;
  }
  if (!defs.empty()) {  // join the endgame stream, apply the deferred column sides, read statuses
    MSY_CK(cudaEventRecord(sc->evE1, sc->eg));
    MSY_CK(cudaStreamWaitEvent(st, sc->evE1, 0));
    for (const Deferred& d : defs) {
      if (d.lo == 0) continue;
      rc = apply_z_regions<S>(m, d.sz, w.Zend + d.zoff, A, lda, nullptr, ldu, d.lo, 0, 0, d.lo, st);
      if (rc) return rc;
    }
    const size_t nd = defs.size();
    for (size_t k0 = 0; k0 < nd; k0 += 500) {
      const size_t cnt = std::min<size_t>(500, nd - k0);
      int hs[1000];
      MSY_CK(d2h(hs, w.dend + 2 * k0, 2 * cnt * sizeof(int), st));
      for (size_t k = 0; k < cnt; k++) {
        loc.sweeps += hs[2 * k + 1];
        if (hs[2 * k] && !loc.status) loc.status = hs[2 * k];
      }
    }
    pt.lap(&loc.ms_small);
  }
  if (helper) {  // join the helper, then the deferred column sides of its blocks
    helper->drain();
    for (int i = 0; i < SubHelper::NH; i++) {
      MSY_CK(cudaEventRecord(helper->ev1[i], helper->st[i]));
      MSY_CK(cudaStreamWaitEvent(st, helper->ev1[i], 0));
    }
    for (const SubBlock& b : subs) {
      if (b.rc) return b.rc;
      loc.sweeps += b.sweeps;
      if (b.status && !loc.status) loc.status = b.status;
      rc = apply_block_z<S>(false, b.lo, b.sz, plan->Zsub + b.zoff, b.sz, A + (size_t)b.lo * lda, lda, plan->tmp[0], st);
      if (rc) return rc;
    }
    pt.lap(&loc.ms_small);
  }
  return 0;
}

// In place: A (m x m, lda) -> T; U (m x m, ldu) = Schur vectors.
template <class S>
int schur_device(int m, S* A, int lda, S* U, int ldu, SchurWs<S>& w, cudaStream_t st, SchurStats* stats,
                 SweepCtx* sc = nullptr) {
  if (!sc) sc = sweep_ctx();
  constexpr int NMIN = SmallCfg<S>::NMAX;
  SchurStats loc = {};
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
  SubPlan<S> plan = {w.sub, w.Zsub, w.subtmp};
  rc = schur_qr_loop<S>(m, A, lda, U, ldu, w, st, loc, sc, pt, &plan);
  if (stats) *stats = loc;
  return rc;
}

}  // namespace msy
