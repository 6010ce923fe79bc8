// solver.cu -- mp_orth / mp_inv drivers and the C ABI (include/mpsylv_b200.h).
//
// Restates pkg/src/mpsylv/refinement.py:95-297 (Alg. 1, 3, 4 of the paper) on the
// device.  Flow of sylv_solve (real: fp64 data, fp32 Schur; complex: c128 / c64):
//   1. A, B -> u_l (overflow -> FORMAT_OVERFLOW); Schur(A) || Schur(B) on two
//      streams / host threads (Lyapunov: one Schur, T_B = T_A^H, U_B = U_A)
//   2. Q = orth(U) in u_h (Cholesky-QR, positive diagonal R)        [mp_orth]
//      LU(U_A^H), LU(U_B) in u_h                                     [mp_inv]
//   3. F = Q_A^H C Q_B, S_A = Q_A^H A Q_A, S_B = Q_B^H B Q_B (S = T + L)
//   4. Y0 = trsyl(T_A, T_B, fl_l(F)) in u_l; singular / non-finite -> typed failure
//      at the initial solve (or Y0 = 0 with y0_zero)
//   5. repeat: R = F - S_A Y - Y S_B; D = trsyl(T_A, T_B, R) (u_h, or u_l in the
//      fast mode); Y += D; stop when ||D||_F <= eps ||Y||_F (first pass always runs)
//   6. X = Q_A Y Q_B^H; residual and backward error in fp64.
#include "../../include/mpsylv_b200.h"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "krylov.cuh"
#include "gemm.cuh"
#include "gemm_dmma.cuh"
#include "lu.cuh"
#include "microbench.cuh"
#include "orth.cuh"
#include "schur.cuh"
#include "trsyl.cuh"
#include "util.cuh"

using namespace msy;

namespace {

struct StreamCtx {
  SweepCtx swA, swB;  // aux streams of the two concurrent Schur factorisations
  SweepCtx serial;    // no aux stream: batched lanes run everything on their own stream
  cudaStream_t side = nullptr;
  cudaStream_t hiA = nullptr;  // Schur(A)'s critical path (high priority; side is Schur(B)'s)
  cudaEvent_t ev_a = nullptr;
  cudaEvent_t ev_in = nullptr, ev_side = nullptr;
  cudaEvent_t ev[8];
  bool init = false;
  int device = -1;
};
thread_local StreamCtx g_ctx;
// batched lanes: one stream per lane, Schur(A) then Schur(B) (concurrency comes from the lanes)
thread_local bool t_serial_lane = false;
// low-precision Schur factors supplied by the caller (sylv_solve_factored), column-major
struct GivenFactors {
  const void *TA, *UA, *TB, *UB;
  int ldta, ldua, ldtb, ldub;
};
thread_local const GivenFactors* t_given = nullptr;

int ctx_init() {
  int dev;
  MSY_CK(cudaGetDevice(&dev));
  if (g_ctx.init && g_ctx.device == dev) return 0;
  // The chase / near-Z / shift kernels of both Schur factorisations run on high-priority
  // streams; their far Z applications and endgame blocks (SweepCtx aux / eg) keep the
  // default (least) priority, so queued far work yields SMs to the critical path.
  int lo_pri = 0, hi_pri = 0;
  MSY_CK(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
  constexpr bool no_pri = MSY_NO_STREAM_PRIORITY != 0;
  MSY_CK(cudaStreamCreateWithPriority(&g_ctx.side, cudaStreamNonBlocking, no_pri ? lo_pri : hi_pri));
  MSY_CK(cudaStreamCreateWithPriority(&g_ctx.hiA, cudaStreamNonBlocking, no_pri ? lo_pri : hi_pri));
  MSY_CK(cudaEventCreateWithFlags(&g_ctx.ev_a, cudaEventDisableTiming));
  MSY_CK(cudaEventCreateWithFlags(&g_ctx.ev_in, cudaEventDisableTiming));
  MSY_CK(cudaEventCreateWithFlags(&g_ctx.ev_side, cudaEventDisableTiming));
  for (int i = 0; i < 8; i++) MSY_CK(cudaEventCreate(&g_ctx.ev[i]));
  g_ctx.swA.ensure();
  g_ctx.swB.ensure();
  g_ctx.init = true;
  g_ctx.device = dev;
  return 0;
}

template <class Hh, class Ll>
struct SolveWs {
  Ll *TA, *UA, *TB, *UB, *Fl;
  SchurWs<Ll> swA, swB;
  TrsylWs<Ll> tsl;
  Hh *QA, *QB, *SA, *SB, *TAh, *TBh, *G, *F, *Y, *R, *tmp;
  TrsylWs<Hh> tsh;
  LuWs<Hh> luA, luB;
  double* part;
  double* red;
  int* ints;
  Hh *GB, *tmpB;     // B-side scratch: orth(B) and S_B run beside the A side (mp_orth, Sylvester)
  double *partB, *redB;
  int* intsB;
  static void carve(Arena& ar, int m, int n, int kind, int variant, SolveWs& w) {
    size_t mm = (size_t)m * m, nn = (size_t)n * n, mn = (size_t)m * n;
    w.TA = ar.get<Ll>(mm);
    w.UA = ar.get<Ll>(mm);
    w.TB = ar.get<Ll>(nn);
    w.UB = ar.get<Ll>(nn);
    w.Fl = ar.get<Ll>(mn);
    SchurWs<Ll>::carve(ar, m, w.swA);
    if (kind != SYLV_KIND_LYAPUNOV) SchurWs<Ll>::carve(ar, n, w.swB);
    TrsylWs<Ll>::carve(ar, m, n, w.tsl);
    TrsylWs<Hh>::carve(ar, m, n, w.tsh);
    w.QA = ar.get<Hh>(mm);
    w.QB = ar.get<Hh>(nn);
    w.SA = ar.get<Hh>(mm);
    w.SB = ar.get<Hh>(nn);
    w.TAh = ar.get<Hh>(mm);
    w.TBh = ar.get<Hh>(nn);
    size_t big = std::max(mm, nn);
    w.G = ar.get<Hh>(big);
    w.F = ar.get<Hh>(mn);
    w.Y = ar.get<Hh>(mn);
    w.R = ar.get<Hh>(mn);
    w.tmp = ar.get<Hh>(std::max(big, mn));
    if (variant == SYLV_VARIANT_INV) {
      LuWs<Hh>::carve(ar, m, w.luA);
      if (kind != SYLV_KIND_LYAPUNOV) LuWs<Hh>::carve(ar, n, w.luB);
    }
    w.part = ar.get<double>(3 * RED_BLOCKS);
    w.red = ar.get<double>(16);
    w.ints = ar.get<int>(64);
    w.GB = w.tmpB = nullptr;
    w.partB = w.redB = nullptr;
    w.intsB = nullptr;
    if (variant == SYLV_VARIANT_ORTH && kind != SYLV_KIND_LYAPUNOV) {
      w.GB = ar.get<Hh>(nn);
      w.tmpB = ar.get<Hh>(nn);
      w.partB = ar.get<double>(3 * RED_BLOCKS);
      w.redB = ar.get<double>(16);
      w.intsB = ar.get<int>(16);
    }
  }
};

struct HostTimer {
  cudaStream_t st;
  int k = 0;
  HostTimer(cudaStream_t s) : st(s) {}
  void mark() {
    if (k < 8) cudaEventRecord(g_ctx.ev[k++], st);
  }
  double ms(int a, int b) {
    float t = 0;
    if (b < k) cudaEventElapsedTime(&t, g_ctx.ev[a], g_ctx.ev[b]);
    return t;
  }
};

template <class S>
int read_reduce(S* X, int rows, int cols, int ld, const S* Yv, int ldy, int mode, double* part, double* red,
                double out[3], cudaStream_t st) {
  int rc = reduce<S>(mode, rows, cols, X, ld, Yv, ldy, part, red, st);
  if (rc) return rc;
  MSY_CK(d2h(out, red, 3 * sizeof(double), st));
  MSY_CK(host_sync(st));
  return 0;
}

// decode the trsyl status word into (status, row, col)
int read_trsyl_status(int* dstat, int m, int n, int lowerB, int* row, int* col, cudaStream_t st) {
  int h[4];
  MSY_CK(d2h(h, dstat, sizeof(h), st));
  MSY_CK(host_sync(st));
  if (h[0] == 0x7fffffff) return SYLV_OK;
  int crank = h[0] / m, i = m - 1 - h[0] % m;
  *row = i;
  *col = lowerB ? n - 1 - crank : crank;
  return SYLV_SINGULAR_EQUATION;
}

// Column index (0-based, in the matrix) of the first column in solve order holding a
// non-finite entry; -1 if none.  Only called on the failure path.
template <class S>
int first_nonfinite_col(const S* X, int rows, int cols, int ld, int lowerB, int* dint, int* col, cudaStream_t st) {
  first_nonfinite_init_kernel<<<1, 1, 0, st>>>(dint);
  MSY_LAUNCH_CK();
  long tot = (long)rows * cols;
  int nb = (int)std::min<long>(RED_BLOCKS, std::max<long>(1, cdiv(tot, RED_TPB)));
  first_nonfinite_kernel<S><<<nb, RED_TPB, 0, st>>>(rows, cols, X, ld, lowerB, dint);
  MSY_LAUNCH_CK();
  int h = 0;
  MSY_CK(d2h(&h, dint, sizeof(int), st));
  *col = h == 0x7fffffff ? -1 : (lowerB ? cols - 1 - h : h);
  return 0;
}

// The refinement loop (Alg. 1, refinement.py:95-141) on device buffers:
// S_A = T_A + dT_A and S_B = T_B + dT_B already formed; T's in Hh.
// One host readback per iteration: the trsyl status word, ||D||_F^2 and ||Y+D||_F^2 are
// packed on the device (pack_status_kernel); the iterate update is guarded on the device
// so a failed correction leaves Y as the reference leaves it.
template <class Hh, class Ll>
int refine_loop(int m, int n, const Hh* TAh, const Hh* TBh, int lowerB, const Hh* SA, const Hh* SB, const Hh* F, Hh* Y,
                Hh* R, Ll* Rl, const Ll* TAl, const Ll* TBl, int corr_bits, double eps, int max_iter,
                TrsylWs<Hh>& tsh, TrsylWs<Ll>& tsl, double* part, double* red, int* ints, cudaStream_t st,
                sylv_report* rep) {
  rep->iterations = 0;
  rep->converged = 0;
  rep->n_norms = 0;
  double* red_d = red;      // sumsq(D)
  double* red_u = red + 3;  // guarded Y += D: sumsq(D), sumsq(Y), nonfinite
  double* packed = red + 10;
  int i = 0;
  while (i < max_iter) {
    // R = F - S_A Y - Y S_B
    int rc = copy2d<Hh>(m, n, F, m, R, m, st);
    if (rc) return rc;
    rc = gemm<Hh>('N', 'N', m, n, m, Hh(-1), SA, m, Y, m, Hh(1), R, m, st);
    if (rc) return rc;
    rc = gemm<Hh>('N', 'N', m, n, n, Hh(-1), Y, m, SB, n, Hh(1), R, m, st);
    if (rc) return rc;
    trsyl_status_init<<<1, 1, 0, st>>>(ints);
    MSY_LAUNCH_CK();
    if (corr_bits == 32 && Rl != nullptr) {
      rc = convert<Ll, Hh>(m, n, R, m, Rl, m, nullptr, st);
      if (rc) return rc;
      rc = trsyl<Ll>(m, n, TAl, m, TBl, n, lowerB, Rl, m, tsl, ints, st);
      if (rc) return rc;
      rc = convert<Hh, Ll>(m, n, Rl, m, R, m, nullptr, st);
    } else {
      rc = trsyl<Hh>(m, n, TAh, m, TBh, n, lowerB, R, m, tsh, ints, st);
    }
    if (rc) return rc;
    rc = reduce<Hh>(0, m, n, R, m, nullptr, 0, part, red_d, st);
    if (!rc) rc = reduce<Hh>(2, m, n, Y, m, R, m, part, red_u, st, red_d, ints);  // Y += D (guarded)
    if (rc) return rc;
    pack_status_kernel<<<1, 1, 0, st>>>(ints, red_d, red_u, packed);
    MSY_LAUNCH_CK();
    double o[5];
    MSY_CK(d2h(o, packed, sizeof(o), st));
    if ((int)o[0] != 0x7fffffff) {  // singular diagonal pair (refinement.py:242-245)
      int hs = (int)o[0];
      int crank = hs / m;
      rep->status = SYLV_SINGULAR_EQUATION;
      rep->fail_stage = SYLV_STAGE_REFINEMENT;
      rep->fail_row = m - 1 - hs % m;
      rep->fail_col = lowerB ? n - 1 - crank : crank;
      return 0;
    }
    if (!std::isfinite(o[1])) {  // NumericBreakdownError inside solve_sylv_tri (refinement.py:125-127)
      rep->status = SYLV_NUMERIC_BREAKDOWN;
      rep->fail_stage = SYLV_STAGE_REFINEMENT;
      rc = first_nonfinite_col<Hh>(R, m, n, m, lowerB, ints + 8, &rep->fail_col, st);
      if (rc) return rc;
      break;
    }
    i++;
    double nD = std::sqrt(o[2]), nY = std::sqrt(o[3]);
    if (rep->n_norms < SYLV_MAX_NORMS) rep->correction_norms[rep->n_norms++] = nD;
    if (!(std::isfinite(nD) && std::isfinite(nY))) {  // refinement.py:133-135
      rep->status = SYLV_NUMERIC_BREAKDOWN;
      rep->fail_stage = SYLV_STAGE_DIVERGED;
      break;
    }
    if (nD <= eps * nY) {
      rep->converged = 1;
      break;
    }
  }
  rep->iterations = i;
  if (rep->status == SYLV_OK && !rep->converged) rep->status = SYLV_NON_CONVERGENCE;
  return 0;
}

// One persistent host thread drives Schur(B) (and orth(B)/S_B) beside the calling thread's
// Schur(A).  It replaces a std::thread per solve: its thread-local pinned staging buffer and
// sync event are allocated once for the process.  Pair solves are serialised by pair_mutex()
// (the side streams of g_ctx are shared).
struct SideWorker {
  std::mutex mu;
  std::condition_variable cv;
  std::function<void()>* job = nullptr;
  bool done = true;
  SideWorker() {
    std::thread([this]() {
      for (;;) {
        std::function<void()>* j;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [this] { return job != nullptr; });
          j = job;
        }
        (*j)();
        {
          std::lock_guard<std::mutex> lk(mu);
          job = nullptr;
          done = true;
        }
        cv.notify_all();
      }
    }).detach();
  }
  void start(std::function<void()>* j) {
    std::lock_guard<std::mutex> lk(mu);
    job = j;
    done = false;
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return done; });
  }
};
inline SideWorker& side_worker() {
  static SideWorker* w = new SideWorker();  // process lifetime (never joined)
  return *w;
}
inline std::mutex& pair_mutex() {
  static std::mutex m;
  return m;
}

template <class Hh, class Ll>
int run_schur_pair(int m, int n, int kind, const Hh* A, int lda, const Hh* B, int ldb, SolveWs<Hh, Ll>& w,
                   cudaStream_t st, int* ovf, SchurStats* sa, SchurStats* sb,
                   const std::function<int(cudaStream_t)>* post_b = nullptr) {
  int rc = convert<Ll, Hh>(m, m, A, lda, w.TA, m, ovf, st);
  if (rc) return rc;
  SweepCtx* sca = t_serial_lane ? &g_ctx.serial : &g_ctx.swA;
  if (kind == SYLV_KIND_LYAPUNOV) {
    rc = schur_device<Ll>(m, w.TA, m, w.UA, m, w.swA, st, sa, sca);
    if (rc) return rc;
    rc = conj_transpose<Ll>(m, m, w.TA, m, w.TB, n, st);
    if (rc) return rc;
    rc = copy2d<Ll>(m, m, w.UA, m, w.UB, n, st);
    *sb = *sa;
    return rc;
  }
  if (t_serial_lane) {
    rc = schur_device<Ll>(m, w.TA, m, w.UA, m, w.swA, st, sa, sca);
    if (!rc) rc = convert<Ll, Hh>(n, n, B, ldb, w.TB, n, ovf + 1, st);
    if (!rc) rc = schur_device<Ll>(n, w.TB, n, w.UB, n, w.swB, st, sb, sca);
    return rc;
  }
  std::lock_guard<std::mutex> pair_lock(pair_mutex());
  MSY_CK(cudaEventRecord(g_ctx.ev_in, st));
  MSY_CK(cudaStreamWaitEvent(g_ctx.side, g_ctx.ev_in, 0));
  int dev;
  MSY_CK(cudaGetDevice(&dev));
  int rcb = 0;
  cudaStream_t side = g_ctx.side;
  int* ovf_b = ovf + 1;
  SweepCtx* scb = &g_ctx.swB;
  const bool blocking = host_sync_blocking();
  int nsm = 0;
  MSY_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // the two cooperative Hessenberg panel grids share the SMs in proportion to the matrices'
  // sizes (m = n: half each; C2's 4096 / 2048 pair: 118 / 30, so the large reduction is not
  // held to half the GPU long after the small one is done)
  const double wa = (double)m * m, wb = (double)n * n;
  const int cap_sm_a = std::max(16, std::min(nsm - 16, (int)(nsm * (wa / (wa + wb)) + 0.5)));
  const int cap_sm_b = nsm - cap_sm_a;
  struct CapGuard {
    int old;
    explicit CapGuard(int c) : old(hess_grid_cap()) { hess_grid_cap() = c; }
    ~CapGuard() { hess_grid_cap() = old; }
  } cap_a(cap_sm_a);
  std::function<void()> job_b = [&]() {
    cudaSetDevice(dev);
    host_sync_blocking() = blocking;
    hess_grid_cap() = cap_sm_b;
    rcb = convert<Ll, Hh>(n, n, B, ldb, w.TB, n, ovf_b, side);
    if (!rcb) rcb = schur_device<Ll>(n, w.TB, n, w.UB, n, w.swB, side, sb, scb);
    if (!rcb && post_b && sb->status == 0) rcb = (*post_b)(side);
  };
  side_worker().start(&job_b);
  cudaStream_t sa_st = g_ctx.hiA;  // ev_in (recorded above, after convert(A)) orders it after st
  cudaError_t we = cudaStreamWaitEvent(sa_st, g_ctx.ev_in, 0);
  rc = we == cudaSuccess ? schur_device<Ll>(m, w.TA, m, w.UA, m, w.swA, sa_st, sa, &g_ctx.swA) : SYLV_ECUDA;
  side_worker().wait();  // always joined before job_b's captures go out of scope
  if (rc) return rc;
  if (rcb) return rcb;
  if (getenv("MSY_SCHUR_TIMING"))  // diagnostic only (the phase timer synchronises at every lap)
    for (const SchurStats* s : {sa, sb})
      fprintf(stderr, "pair schur: hess %.1f ms, scan %.1f, small %.1f, shift %.1f, sweep %.1f | qr sweeps %d\n",
              s->ms_hess, s->ms_scan, s->ms_small, s->ms_shift, s->ms_sweep, s->ms_sweeps);
  MSY_CK(cudaEventRecord(g_ctx.ev_a, sa_st));
  MSY_CK(cudaStreamWaitEvent(st, g_ctx.ev_a, 0));
  MSY_CK(cudaEventRecord(g_ctx.ev_side, side));
  MSY_CK(cudaStreamWaitEvent(st, g_ctx.ev_side, 0));
  return 0;
}

template <class Hh, class Ll>
int final_report(int m, int n, const Hh* A, int lda, const Hh* B, int ldb, const Hh* C, int ldc, Hh* X, int ldx,
                 SolveWs<Hh, Ll>& w, cudaStream_t st, sylv_report* rep);

template <class Hh, class Ll>
int solve_impl(const sylv_params* p, const Hh* A, int lda, const Hh* B, int ldb, const Hh* C, int ldc, Hh* X, int ldx,
               void* wsp, size_t wsb, cudaStream_t st, sylv_report* rep) {
  const int m = p->m, n = p->n;
  Arena ar(wsp, wsb);
  SolveWs<Hh, Ll> w;
  SolveWs<Hh, Ll>::carve(ar, m, n, p->kind, p->variant, w);
  if (!ar.ok()) return SYLV_EWORKSPACE;
  int rc = ctx_init();
  if (rc) return rc;
  memset(rep, 0, sizeof(*rep));
  rep->fail_row = rep->fail_col = -1;
  auto t0 = std::chrono::steady_clock::now();
  HostTimer tm(st);
  tm.mark();  // 0
  const bool lyap = p->kind == SYLV_KIND_LYAPUNOV;
  const bool inv = p->variant == SYLV_VARIANT_INV;
  int* ovf = w.ints + 32;
  MSY_CK(cudaMemsetAsync(ovf, 0, 2 * sizeof(int), st));
  // ---- 1. low-precision Schur pair ----
  SchurStats sa{}, sb{};
  // mp_orth, Sylvester: orth(B) and S_B = Q_B^H B Q_B run in the Schur(B) thread on its stream,
  // overlapping the A side (the two chains are latency-bound small-kernel sequences)
  const bool b_beside = !inv && !lyap && !t_serial_lane && w.GB != nullptr;
  int b_rank = 0;
  std::function<int(cudaStream_t)> post_b = [&](cudaStream_t ss) -> int {
    int r2 = convert<Hh, Ll>(n, n, w.UB, n, w.TBh, n, nullptr, ss);
    if (r2) return r2;
    int* dflag = w.intsB;
    double* ddiag = w.redB + 8;
    MSY_CK(cudaMemsetAsync(dflag, 0, sizeof(int), ss));
    fill<double>(1, 1, INFINITY, ddiag, 1, ss);
    r2 = orth_cholqr<Hh>(n, w.TBh, n, w.QB, n, w.GB, n, dflag, ddiag, ss);
    if (r2) return r2;
    double o[3];
    r2 = read_reduce<Hh>(w.TBh, n, n, n, nullptr, 0, 0, w.partB, w.redB, o, ss);
    if (r2) return r2;
    int hflag;
    double hdiag;
    MSY_CK(d2h(&hflag, dflag, sizeof(int), ss));
    MSY_CK(d2h(&hdiag, ddiag, sizeof(double), ss));
    if (hflag || hdiag <= n * tr<Hh>::u() * std::sqrt(o[0])) { b_rank = 1; return 0; }
    r2 = gemm<Hh>('C', 'N', n, n, n, Hh(1), w.QB, n, B, ldb, Hh(0), w.tmpB, n, ss);
    if (!r2) r2 = gemm<Hh>('N', 'N', n, n, n, Hh(1), w.tmpB, n, w.QB, n, Hh(0), w.SB, n, ss);
    return r2;
  };
  if (t_given != nullptr) {  // sylv_solve_factored: the low-precision Schur factors come from the caller
    const GivenFactors& g = *t_given;
    rc = copy2d<Ll>(m, m, (const Ll*)g.TA, g.ldta, w.TA, m, st);
    if (!rc) rc = copy2d<Ll>(m, m, (const Ll*)g.UA, g.ldua, w.UA, m, st);
    if (!rc) rc = copy2d<Ll>(n, n, (const Ll*)g.TB, g.ldtb, w.TB, n, st);
    if (!rc) rc = copy2d<Ll>(n, n, (const Ll*)g.UB, g.ldub, w.UB, n, st);
    if (!rc && b_beside) rc = post_b(st);
  } else {
    rc = run_schur_pair<Hh, Ll>(m, n, p->kind, A, lda, B, ldb, w, st, ovf, &sa, &sb, b_beside ? &post_b : nullptr);
  }
  if (rc) return rc;
  rep->schur_sweeps_a = sa.sweeps;
  rep->schur_sweeps_b = sb.sweeps;
  int hovf[2];
  MSY_CK(d2h(hovf, ovf, sizeof(hovf), st));
  MSY_CK(host_sync(st));
  if (hovf[0] || hovf[1]) { rep->status = SYLV_FORMAT_OVERFLOW; return 0; }
  if (sa.status || sb.status) { rep->status = SYLV_ITERATION_LIMIT; return 0; }
  tm.mark();  // 1
  // ---- 2. orthonormalise (mp_orth) / LU (mp_inv) in u_h ----
  rc = convert<Hh, Ll>(m, m, w.UA, m, w.TAh, m, nullptr, st);  // TAh used as U_A (hi) scratch
  if (rc) return rc;
  if (!inv) {
    int* dflag = w.ints + 40;
    double* ddiag = w.red + 8;
    MSY_CK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
    fill<double>(1, 1, INFINITY, ddiag, 1, st);
    rc = orth_cholqr<Hh>(m, w.TAh, m, w.QA, m, w.G, m, dflag, ddiag, st);
    if (rc) return rc;
    double o[3];
    rc = read_reduce<Hh>(w.TAh, m, m, m, nullptr, 0, 0, w.part, w.red, o, st);
    if (rc) return rc;
    int hflag;
    double hdiag;
    MSY_CK(d2h(&hflag, dflag, sizeof(int), st));
    MSY_CK(d2h(&hdiag, ddiag, sizeof(double), st));
    MSY_CK(host_sync(st));
    // _check_rank (linalg.py:244-249): min R_jj <= n u ||U||_F
    if (hflag || hdiag <= m * tr<Hh>::u() * std::sqrt(o[0])) { rep->status = SYLV_RANK_DEFICIENT; return 0; }
    if (lyap) {
      rc = copy2d<Hh>(m, m, w.QA, m, w.QB, n, st);
    } else if (b_beside) {
      if (b_rank) { rep->status = SYLV_RANK_DEFICIENT; return 0; }
    } else {
      rc = convert<Hh, Ll>(n, n, w.UB, n, w.TBh, n, nullptr, st);
      if (rc) return rc;
      MSY_CK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
      fill<double>(1, 1, INFINITY, ddiag, 1, st);
      rc = orth_cholqr<Hh>(n, w.TBh, n, w.QB, n, w.G, n, dflag, ddiag, st);
      if (rc) return rc;
      rc = read_reduce<Hh>(w.TBh, n, n, n, nullptr, 0, 0, w.part, w.red, o, st);
      if (rc) return rc;
      MSY_CK(d2h(&hflag, dflag, sizeof(int), st));
      MSY_CK(d2h(&hdiag, ddiag, sizeof(double), st));
      MSY_CK(host_sync(st));
      if (hflag || hdiag <= n * tr<Hh>::u() * std::sqrt(o[0])) { rep->status = SYLV_RANK_DEFICIENT; return 0; }
    }
    if (rc) return rc;
  }
  tm.mark();  // 2
  // ---- 3. transformed data: F, S_A, S_B (and T in u_h) ----
  if (!inv) {
    rc = gemm<Hh>('C', 'N', m, n, m, Hh(1), w.QA, m, C, ldc, Hh(0), w.tmp, m, st);
    if (!rc) rc = gemm<Hh>('N', 'N', m, n, n, Hh(1), w.tmp, m, w.QB, n, Hh(0), w.F, m, st);
    if (!rc) rc = gemm<Hh>('C', 'N', m, m, m, Hh(1), w.QA, m, A, lda, Hh(0), w.tmp, m, st);
    if (!rc) rc = gemm<Hh>('N', 'N', m, m, m, Hh(1), w.tmp, m, w.QA, m, Hh(0), w.SA, m, st);
    if (rc) return rc;
    if (lyap) {
      rc = conj_transpose<Hh>(m, m, w.SA, m, w.SB, n, st);
    } else if (!b_beside) {
      rc = gemm<Hh>('C', 'N', n, n, n, Hh(1), w.QB, n, B, ldb, Hh(0), w.tmp, n, st);
      if (!rc) rc = gemm<Hh>('N', 'N', n, n, n, Hh(1), w.tmp, n, w.QB, n, Hh(0), w.SB, n, st);
    }
    if (rc) return rc;
  } else {
    // mp_inv (refinement.py:264-279): LU(U_A^H), LU(U_B);
    // F = U_A^H C U_B; S_A = (U_A^H A) U_A^{-H}; S_B = U_B^{-1} (B U_B)
    Hh* UAh = w.TAh;                       // U_A in u_h (scratch, filled above)
    rc = conj_transpose<Hh>(m, m, UAh, m, w.QA, m, st);  // QA := U_A^H, factored in place
    if (rc) return rc;
    rc = lu_factor<Hh>(m, w.QA, m, w.luA, st);
    if (rc) return rc;
    Hh* UBh = w.TBh;
    if (lyap) {
      rc = copy2d<Hh>(m, m, UAh, m, UBh, n, st);
    } else {
      rc = convert<Hh, Ll>(n, n, w.UB, n, UBh, n, nullptr, st);
      if (!rc) rc = copy2d<Hh>(n, n, UBh, n, w.QB, n, st);
      if (!rc) rc = lu_factor<Hh>(n, w.QB, n, w.luB, st);
    }
    if (rc) return rc;
    int sing = 0;
    rc = lu_read_status<Hh>(w.luA, &sing, st);
    if (rc) return rc;
    if (!lyap && !sing) {
      rc = lu_read_status<Hh>(w.luB, &sing, st);
      if (rc) return rc;
    }
    if (sing) { rep->status = SYLV_SINGULAR_MATRIX; return 0; }
    rc = gemm<Hh>('C', 'N', m, n, m, Hh(1), UAh, m, C, ldc, Hh(0), w.tmp, m, st);
    if (!rc) rc = gemm<Hh>('N', 'N', m, n, n, Hh(1), w.tmp, m, UBh, n, Hh(0), w.F, m, st);
    if (!rc) rc = gemm<Hh>('C', 'N', m, m, m, Hh(1), UAh, m, A, lda, Hh(0), w.SA, m, st);
    // S_A = W U_A^{-H}:  X (U_A^H) = W  -> right solve with LU of U_A^H
    if (!rc) rc = lu_solve<Hh>(m, w.QA, m, w.luA, /*right=*/1, /*conj=*/0, m, w.SA, m, w.tmp, st);
    if (rc) return rc;
    if (lyap) {
      rc = conj_transpose<Hh>(m, m, w.SA, m, w.SB, n, st);
    } else {
      rc = gemm<Hh>('N', 'N', n, n, n, Hh(1), B, ldb, UBh, n, Hh(0), w.SB, n, st);
      if (!rc) rc = lu_solve<Hh>(n, w.QB, n, w.luB, /*right=*/0, /*conj=*/0, n, w.SB, n, w.tmp, st);
    }
    if (rc) return rc;
  }
  rc = convert<Hh, Ll>(m, m, w.TA, m, w.TAh, m, nullptr, st);
  if (!rc) rc = convert<Hh, Ll>(n, n, w.TB, n, w.TBh, n, nullptr, st);
  if (rc) return rc;
  tm.mark();  // 3
  // ---- 4. Y0 in u_l ----
  rc = convert<Ll, Hh>(m, n, w.F, m, w.Fl, m, nullptr, st);
  if (rc) return rc;
  int* tstat = w.ints;
  trsyl_status_init<<<1, 1, 0, st>>>(tstat);
  rc = trsyl<Ll>(m, n, w.TA, m, w.TB, n, lyap ? 1 : 0, w.Fl, m, w.tsl, tstat, st);
  if (rc) return rc;
  int row = -1, col = -1;
  int ts = read_trsyl_status(tstat, m, n, lyap ? 1 : 0, &row, &col, st);
  if (ts < 0) return ts;
  double o[3];
  if (ts == SYLV_OK) {
    rc = read_reduce<Ll>(w.Fl, m, n, m, nullptr, 0, 0, w.part, w.red, o, st);
    if (rc) return rc;
    if (!std::isfinite(o[0])) {
      ts = SYLV_NUMERIC_BREAKDOWN;
      rc = first_nonfinite_col<Ll>(w.Fl, m, n, m, lyap ? 1 : 0, tstat + 8, &col, st);
      if (rc) return rc;
    }
  }
  if (ts != SYLV_OK) {
    if (!p->y0_zero) {
      rep->status = ts;
      rep->fail_stage = SYLV_STAGE_INITIAL;
      rep->fail_row = row;
      rep->fail_col = col;
      rep->iterations = 0;
      rep->residual = NAN;
      fill<Hh>(m, n, mk<Hh>(NAN, NAN), X, ldx, st);
      MSY_CK(host_sync(st));
      return 0;
    }
    fill<Hh>(m, n, Hh(0), w.Y, m, st);
  } else {
    rc = convert<Hh, Ll>(m, n, w.Fl, m, w.Y, m, nullptr, st);
    if (rc) return rc;
  }
  tm.mark();  // 4
  // ---- 5. refinement ----
  double eps = p->epsilon > 0 ? p->epsilon : 1e-12 * std::max(m, n);
  rc = refine_loop<Hh, Ll>(m, n, w.TAh, w.TBh, lyap ? 1 : 0, w.SA, w.SB, w.F, w.Y, w.R, w.Fl, w.TA, w.TB,
                           p->correction_bits, eps, p->max_iter, w.tsh, w.tsl, w.part, w.red, w.ints, st, rep);
  if (rc) return rc;
  if (rep->status == SYLV_SINGULAR_EQUATION) {  // _failed_report (refinement.py:244-245)
    rep->iterations = 0;
    rep->n_norms = 0;
    rep->converged = 0;
    rep->residual = NAN;
    fill<Hh>(m, n, mk<Hh>(NAN, NAN), X, ldx, st);
    MSY_CK(host_sync(st));
    return 0;
  }
  tm.mark();  // 5
  // ---- 6. recovery X = Q_A Y Q_B^H  (mp_inv: X = U_A^{-H} Y U_B^{-1}) ----
  if (!inv) {
    rc = gemm<Hh>('N', 'N', m, n, m, Hh(1), w.QA, m, w.Y, m, Hh(0), w.tmp, m, st);
    if (!rc) rc = gemm<Hh>('N', 'C', m, n, n, Hh(1), w.tmp, m, w.QB, n, Hh(0), X, ldx, st);
  } else {
    // Z = lu_solve(lu_A, Y) (left), X = Z U_B^{-1} (right, or (U_A^H)^{-H}... for Lyapunov)
    rc = copy2d<Hh>(m, n, w.Y, m, w.R, m, st);
    if (!rc) rc = lu_solve<Hh>(m, w.QA, m, w.luA, 0, 0, n, w.R, m, w.tmp, st);
    if (!rc) {
      if (lyap) rc = lu_solve<Hh>(m, w.QA, m, w.luA, 1, 1, m, w.R, m, w.tmp, st);
      else rc = lu_solve<Hh>(n, w.QB, n, w.luB, 1, 0, m, w.R, m, w.tmp, st);
    }
    if (!rc) rc = copy2d<Hh>(m, n, w.R, m, X, ldx, st);
  }
  if (rc) return rc;
  tm.mark();  // 6
  // ---- 7. residual (sylvester.py:199-209) and backward error ----
  rc = final_report<Hh, Ll>(m, n, A, lda, B, ldb, C, ldc, X, ldx, w, st, rep);
  if (rc) return rc;
  tm.mark();  // 7
  MSY_CK(host_sync(st));
  rep->ms_schur = tm.ms(0, 1);
  rep->ms_orth = tm.ms(1, 2);
  rep->ms_setup = tm.ms(2, 3);
  rep->ms_y0 = tm.ms(3, 4);
  rep->ms_refine = tm.ms(4, 5);
  rep->ms_recover = tm.ms(5, 7);
  rep->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return 0;
}

// residual (sylvester.py:199-209) and the north star's backward error, in fp64
template <class Hh, class Ll>
int final_report(int m, int n, const Hh* A, int lda, const Hh* B, int ldb, const Hh* C, int ldc, Hh* X, int ldx,
                 SolveWs<Hh, Ll>& w, cudaStream_t st, sylv_report* rep) {
  int rc = gemm<Hh>('N', 'N', m, n, m, Hh(1), A, lda, X, ldx, Hh(0), w.R, m, st);
  if (!rc) rc = gemm<Hh>('N', 'N', m, n, n, Hh(1), X, ldx, B, ldb, Hh(1), w.R, m, st);
  if (rc) return rc;
  double nr[3], nA[3], nB[3], nC[3], nX[3];
  rc = read_reduce<Hh>(w.R, m, n, m, C, ldc, 1, w.part, w.red, nr, st);
  if (!rc) rc = read_reduce<Hh>((Hh*)A, m, m, lda, nullptr, 0, 0, w.part, w.red, nA, st);
  if (!rc) rc = read_reduce<Hh>((Hh*)B, n, n, ldb, nullptr, 0, 0, w.part, w.red, nB, st);
  if (!rc) rc = read_reduce<Hh>((Hh*)C, m, n, ldc, nullptr, 0, 0, w.part, w.red, nC, st);
  if (!rc) rc = read_reduce<Hh>(X, m, n, ldx, nullptr, 0, 0, w.part, w.red, nX, st);
  if (rc) return rc;
  double num = std::sqrt(nr[0]), a = std::sqrt(nA[0]), b = std::sqrt(nB[0]), c = std::sqrt(nC[0]),
         x = std::sqrt(nX[0]);
  double den = c + x * (a + b);
  rep->residual = den == 0.0 ? 0.0 : num / den;
  rep->backward_error = (a + b) * x == 0.0 ? 0.0 : num / ((a + b) * x);
  rep->norm_x = x;
  return 0;
}

// Bartels-Stewart in one precision (sylvester.py:160-178, the paper's fp64 comparator):
// Schur(A) || Schur(B) in Hh, F = U_A^H C U_B, Y = trsyl(T_A, T_B, F), X = U_A Y U_B^H.
// A singular or non-finite triangular solve is reported as a typed failure at the
// initial solve with X all NaN (the wrapper raises the reference's exceptions).
template <class Hh>
int bs_impl(const sylv_params* p, const Hh* A, int lda, const Hh* B, int ldb, const Hh* C, int ldc, Hh* X, int ldx,
            void* wsp, size_t wsb, cudaStream_t st, sylv_report* rep) {
  const int m = p->m, n = p->n;
  Arena ar(wsp, wsb);
  SolveWs<Hh, Hh> w;
  SolveWs<Hh, Hh>::carve(ar, m, n, p->kind, p->variant, w);  // same carve as sylv_workspace_size
  if (!ar.ok()) return SYLV_EWORKSPACE;
  int rc = ctx_init();
  if (rc) return rc;
  memset(rep, 0, sizeof(*rep));
  rep->fail_row = rep->fail_col = -1;
  auto t0 = std::chrono::steady_clock::now();
  HostTimer tm(st);
  tm.mark();  // 0
  const bool lyap = p->kind == SYLV_KIND_LYAPUNOV;
  int* ovf = w.ints + 32;
  MSY_CK(cudaMemsetAsync(ovf, 0, 2 * sizeof(int), st));
  SchurStats sa{}, sb{};
  rc = run_schur_pair<Hh, Hh>(m, n, p->kind, A, lda, B, ldb, w, st, ovf, &sa, &sb);
  if (rc) return rc;
  rep->schur_sweeps_a = sa.sweeps;
  rep->schur_sweeps_b = sb.sweeps;
  MSY_CK(host_sync(st));
  if (sa.status || sb.status) { rep->status = SYLV_ITERATION_LIMIT; return 0; }
  tm.mark();  // 1
  rc = gemm<Hh>('C', 'N', m, n, m, Hh(1), w.UA, m, C, ldc, Hh(0), w.tmp, m, st);
  if (!rc) rc = gemm<Hh>('N', 'N', m, n, n, Hh(1), w.tmp, m, w.UB, n, Hh(0), w.F, m, st);
  if (rc) return rc;
  tm.mark();  // 2
  int* tstat = w.ints;
  trsyl_status_init<<<1, 1, 0, st>>>(tstat);
  MSY_LAUNCH_CK();
  rc = trsyl<Hh>(m, n, w.TA, m, w.TB, n, lyap ? 1 : 0, w.F, m, w.tsh, tstat, st);
  if (rc) return rc;
  int row = -1, col = -1;
  int ts = read_trsyl_status(tstat, m, n, lyap ? 1 : 0, &row, &col, st);
  if (ts < 0) return ts;
  if (ts == SYLV_OK) {
    double o[3];
    rc = read_reduce<Hh>(w.F, m, n, m, nullptr, 0, 0, w.part, w.red, o, st);
    if (rc) return rc;
    if (!std::isfinite(o[0])) {
      ts = SYLV_NUMERIC_BREAKDOWN;
      rc = first_nonfinite_col<Hh>(w.F, m, n, m, lyap ? 1 : 0, tstat + 8, &col, st);
      if (rc) return rc;
    }
  }
  if (ts != SYLV_OK) {
    rep->status = ts;
    rep->fail_stage = SYLV_STAGE_INITIAL;
    rep->fail_row = row;
    rep->fail_col = col;
    rep->residual = NAN;
    fill<Hh>(m, n, mk<Hh>(NAN, NAN), X, ldx, st);
    MSY_CK(host_sync(st));
    return 0;
  }
  tm.mark();  // 3
  rc = gemm<Hh>('N', 'N', m, n, m, Hh(1), w.UA, m, w.F, m, Hh(0), w.tmp, m, st);
  if (!rc) rc = gemm<Hh>('N', 'C', m, n, n, Hh(1), w.tmp, m, w.UB, n, Hh(0), X, ldx, st);
  if (rc) return rc;
  tm.mark();  // 4
  rc = final_report<Hh, Hh>(m, n, A, lda, B, ldb, C, ldc, X, ldx, w, st, rep);
  if (rc) return rc;
  rep->converged = 1;
  tm.mark();  // 5
  MSY_CK(host_sync(st));
  rep->ms_schur = tm.ms(0, 1);
  rep->ms_setup = tm.ms(1, 2);
  rep->ms_y0 = tm.ms(2, 3);
  rep->ms_recover = tm.ms(3, 5);
  rep->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return 0;
}

bool valid_dtype(int d) { return d >= 0 && d <= 3; }

}  // namespace

// ===========================================================================
// C ABI (linkage from include/mpsylv_b200.h)

int sylv_version(void) { return 1; }

unsigned long long sylv_launch_count(void) { return __atomic_load_n(&msy::launch_counter(), __ATOMIC_RELAXED); }

int sylv_microbench(int kind, double* tflops, void* stream) {
  if (kind < 0 || kind > 2 || !tflops) return SYLV_EINVAL;
  return msy::microbench(kind, tflops, (cudaStream_t)stream);
}

int sylv_ktimer(int op, int ncls, long long* launches, double* ms, double* flops) {
  msy::KTimer& t = msy::ktimer();
  if (op == 0 || op == 1) {
    t.on.store(0);
    std::lock_guard<std::mutex> g(t.mu);
    for (auto& r : t.recs) { t.pool.push_back(r.a); t.pool.push_back(r.b); }
    t.recs.clear();
    if (op == 1) t.on.store(1);
    return SYLV_OK;
  }
  if (op != 2 || ncls < 0) return SYLV_EINVAL;
  std::lock_guard<std::mutex> g(t.mu);
  for (int c = 0; c < ncls; c++) { launches[c] = 0; ms[c] = 0; flops[c] = 0; }
  for (auto& r : t.recs) {
    float e = 0;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&e, r.a, r.b) != cudaSuccess) e = 0;
    if (r.cls < ncls) { launches[r.cls]++; ms[r.cls] += e; flops[r.cls] += r.flops; }
    t.pool.push_back(r.a);
    t.pool.push_back(r.b);
  }
  t.recs.clear();
  return SYLV_OK;
}

const char* sylv_status_string(int s) {
  switch (s) {
    case SYLV_OK: return "ok";
    case SYLV_SINGULAR_EQUATION: return "singular_equation";
    case SYLV_NUMERIC_BREAKDOWN: return "nan_breakdown";
    case SYLV_ITERATION_LIMIT: return "iteration_limit";
    case SYLV_RANK_DEFICIENT: return "rank_deficient";
    case SYLV_SINGULAR_MATRIX: return "singular_matrix";
    case SYLV_FORMAT_OVERFLOW: return "format_overflow";
    case SYLV_NON_CONVERGENCE: return "non_convergence";
    case SYLV_EINVAL: return "invalid_argument";
    case SYLV_EUNSUPPORTED: return "unsupported";
    case SYLV_EWORKSPACE: return "workspace_too_small";
    default: return s <= SYLV_ECUDA ? "cuda_error" : "unknown";
  }
}

static int check_params(const sylv_params* p) {
  if (!p || p->m < 1 || p->n < 1 || p->max_iter < 1) return SYLV_EINVAL;
  if (p->kind != SYLV_KIND_GENERAL && p->kind != SYLV_KIND_LYAPUNOV) return SYLV_EINVAL;
  if (p->kind == SYLV_KIND_LYAPUNOV && p->m != p->n) return SYLV_EINVAL;
  if (p->variant != SYLV_VARIANT_ORTH && p->variant != SYLV_VARIANT_INV && p->variant != SYLV_VARIANT_BS)
    return SYLV_EINVAL;
  if (p->low_bits != 32 && p->low_bits != 64) return SYLV_EUNSUPPORTED;
  if (p->variant == SYLV_VARIANT_BS && p->low_bits != 64) return SYLV_EUNSUPPORTED;
  if (p->correction_bits != 32 && p->correction_bits != 64) return SYLV_EUNSUPPORTED;
  return 0;
}

int sylv_workspace_size(const sylv_params* p, size_t* bytes) {
  int rc = check_params(p);
  if (rc) return rc;
  Arena ar(nullptr, 0);
  if (!p->complex_data) {
    if (p->low_bits == 32) { SolveWs<double, float> w; SolveWs<double, float>::carve(ar, p->m, p->n, p->kind, p->variant, w); }
    else { SolveWs<double, double> w; SolveWs<double, double>::carve(ar, p->m, p->n, p->kind, p->variant, w); }
  } else {
    if (p->low_bits == 32) { SolveWs<cdouble, cfloat> w; SolveWs<cdouble, cfloat>::carve(ar, p->m, p->n, p->kind, p->variant, w); }
    else { SolveWs<cdouble, cdouble> w; SolveWs<cdouble, cdouble>::carve(ar, p->m, p->n, p->kind, p->variant, w); }
  }
  *bytes = ar.off + 256;
  return 0;
}

int sylv_solve(const sylv_params* p, const void* A, int lda, const void* B, int ldb, const void* C, int ldc, void* X,
               int ldx, void* ws, size_t ws_bytes, void* stream, sylv_report* rep) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!A || !B || !C || !X || !rep || lda < p->m || ldb < p->n || ldc < p->m || ldx < p->m) return SYLV_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->variant == SYLV_VARIANT_BS) {
    if (!p->complex_data)
      return bs_impl<double>(p, (const double*)A, lda, (const double*)B, ldb, (const double*)C, ldc, (double*)X,
                             ldx, ws, ws_bytes, st, rep);
    return bs_impl<cdouble>(p, (const cdouble*)A, lda, (const cdouble*)B, ldb, (const cdouble*)C, ldc,
                            (cdouble*)X, ldx, ws, ws_bytes, st, rep);
  }
  if (!p->complex_data) {
    if (p->low_bits == 32)
      return solve_impl<double, float>(p, (const double*)A, lda, (const double*)B, ldb, (const double*)C, ldc,
                                       (double*)X, ldx, ws, ws_bytes, st, rep);
    return solve_impl<double, double>(p, (const double*)A, lda, (const double*)B, ldb, (const double*)C, ldc,
                                      (double*)X, ldx, ws, ws_bytes, st, rep);
  }
  if (p->low_bits == 32)
    return solve_impl<cdouble, cfloat>(p, (const cdouble*)A, lda, (const cdouble*)B, ldb, (const cdouble*)C, ldc,
                                       (cdouble*)X, ldx, ws, ws_bytes, st, rep);
  return solve_impl<cdouble, cdouble>(p, (const cdouble*)A, lda, (const cdouble*)B, ldb, (const cdouble*)C, ldc,
                                      (cdouble*)X, ldx, ws, ws_bytes, st, rep);
}

// ---- batched executor (C4) ---------------------------------------------------
// A persistent pool of host worker threads ("lanes").  Each lane owns a stream,
// its thread-local solve context (side / aux streams, events) and a slice of the
// caller's workspace; lanes pull equation indices from a shared counter and run
// the ordinary single-equation driver with blocking-sync host waits.
namespace {

class LanePool {
 public:
  static LanePool& get() {
    static LanePool* p = new LanePool;  // leaked on purpose: workers outlive static destruction
    return *p;
  }
  // run fn(lane) on lanes 0..n-1 concurrently; returns when all have finished
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> call(call_mu_);
    std::unique_lock<std::mutex> g(mu_);
    while ((int)th_.size() < n) {
      int id = (int)th_.size();
      th_.emplace_back([this, id] { loop(id); });
    }
    fn_ = &fn;
    nrun_ = n;
    pending_ = n;
    gen_++;
    cv_.notify_all();
    done_cv_.wait(g, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int id) {
    int seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= nrun_) continue;
        f = fn_;
      }
      (*f)(id);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> th_;
  const std::function<void(int)>* fn_ = nullptr;
  int nrun_ = 0, pending_ = 0, gen_ = 0;
};

struct LaneStream {
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  int dev = -1;
};

constexpr int kDefaultLanes = 64;  // measured C4 optimum on one B200 (16: 103, 32: 151, 64: 178, 96: 173 solves/s)

int lanes_for(int lanes, int batch) { return std::max(1, std::min(lanes > 0 ? lanes : kDefaultLanes, batch)); }

}  // namespace

int sylv_batched_workspace_size(const sylv_params* p, int lanes, size_t* bytes) {
  if (!bytes) return SYLV_EINVAL;
  size_t one = 0;
  int rc = sylv_workspace_size(p, &one);
  if (rc) return rc;
  one = (one + 255) & ~(size_t)255;
  *bytes = one * (size_t)(lanes > 0 ? lanes : kDefaultLanes);
  return 0;
}

int sylv_solve_batched(const sylv_params* p, int batch, const void* const* A, int lda, const void* const* B, int ldb,
                       const void* const* C, int ldc, void* const* X, int ldx, int lanes, void* ws, size_t ws_bytes,
                       void* stream, sylv_report* reports) {
  int rc = check_params(p);
  if (rc) return rc;
  if (batch < 0 || (batch > 0 && (!A || !B || !C || !X || !reports))) return SYLV_EINVAL;
  if (batch == 0) return 0;
  const int nl = lanes_for(lanes, batch);
  size_t one = 0;
  rc = sylv_workspace_size(p, &one);
  if (rc) return rc;
  one = (one + 255) & ~(size_t)255;
  if (!ws || ws_bytes < one * (size_t)nl) return SYLV_EWORKSPACE;
  int dev;
  MSY_CK(cudaGetDevice(&dev));
  cudaStream_t cst = (cudaStream_t)stream;
  cudaEvent_t start;
  MSY_CK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  MSY_CK(cudaEventRecord(start, cst));
  std::atomic<int> next{0}, err{0};
  std::vector<cudaEvent_t> done(nl, nullptr);
  std::function<void(int)> fn = [&](int lane) {
    thread_local LaneStream ls;
    if (cudaSetDevice(dev) != cudaSuccess) { err.store(SYLV_ECUDA); return; }
    if (ls.st == nullptr || ls.dev != dev) {
      cudaStreamCreateWithFlags(&ls.st, cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&ls.done, cudaEventDisableTiming);
      ls.dev = dev;
    }
    host_sync_blocking() = true;
    t_serial_lane = true;
    // many lanes' cooperative Hessenberg panels must be co-resident: small grids per lane
    const int cap_saved = hess_grid_cap();
    hess_grid_cap() = MSY_LANE_HESS_CAP;
    hess_graph_lane() = true;
    cudaStreamWaitEvent(ls.st, start, 0);
    char* mine = (char*)ws + one * (size_t)lane;
    for (int i; (i = next.fetch_add(1)) < batch && err.load() == 0;) {
      int r = sylv_solve(p, A[i], lda, B[i], ldb, C[i], ldc, X[i], ldx, mine, one, ls.st, &reports[i]);
      if (r) { int z = 0; err.compare_exchange_strong(z, r); }
    }
    cudaEventRecord(ls.done, ls.st);
    done[lane] = ls.done;
    host_sync_blocking() = false;
    t_serial_lane = false;
    hess_grid_cap() = cap_saved;
    hess_graph_lane() = false;
  };
  LanePool::get().run(nl, fn);
  for (int l = 0; l < nl; l++)
    if (done[l]) MSY_CK(cudaStreamWaitEvent(cst, done[l], 0));
  cudaEventDestroy(start);
  return err.load();
}

// ---- solve_pert_sylv_tri_stat --------------------------------------------
template <class Hh>
static void refine_carve(Arena& ar, int m, int n, Hh** SA, Hh** SB, Hh** R, TrsylWs<Hh>* t, double** part,
                         double** red, int** ints) {
  *SA = ar.get<Hh>((size_t)m * m);
  *SB = ar.get<Hh>((size_t)n * n);
  *R = ar.get<Hh>((size_t)m * n);
  TrsylWs<Hh>::carve(ar, m, n, *t);
  *part = ar.get<double>(3 * RED_BLOCKS);
  *red = ar.get<double>(16);
  *ints = ar.get<int>(64);
}

int sylv_refine_workspace_size(int dtype, int m, int n, size_t* bytes) {
  if ((dtype != 1 && dtype != 3) || m < 1 || n < 1) return SYLV_EINVAL;
  Arena ar(nullptr, 0);
  double *part, *red;
  int* ints;
  if (dtype == 1) {
    double *SA, *SB, *R;
    TrsylWs<double> t;
    refine_carve<double>(ar, m, n, &SA, &SB, &R, &t, &part, &red, &ints);
  } else {
    cdouble *SA, *SB, *R;
    TrsylWs<cdouble> t;
    refine_carve<cdouble>(ar, m, n, &SA, &SB, &R, &t, &part, &red, &ints);
  }
  *bytes = ar.off + 256;
  return 0;
}

template <class Hh>
static int refine_entry(int m, int n, const Hh* TA, int ldta, const Hh* dTA, int lddta, const Hh* TB, int ldtb,
                        const Hh* dTB, int lddtb, int b_lower, const Hh* C, int ldc, const Hh* Y0, int ldy0, double eps,
                        int max_iter, Hh* Y, int ldy, void* ws, size_t wsb, cudaStream_t st, sylv_report* rep) {
  Arena ar(ws, wsb);
  Hh *SA, *SB, *R;
  TrsylWs<Hh> t;
  double *part, *red;
  int* ints;
  refine_carve<Hh>(ar, m, n, &SA, &SB, &R, &t, &part, &red, &ints);
  if (!ar.ok()) return SYLV_EWORKSPACE;
  memset(rep, 0, sizeof(*rep));
  rep->fail_row = rep->fail_col = -1;
  if (ldta != m || ldtb != n || ldc != m || ldy != m) return SYLV_EINVAL;
  // S = T + dT, Y = Y0
  int rc = copy2d<Hh>(m, m, TA, ldta, SA, m, st);
  if (!rc) { add_kernel<Hh><<<dim3(cdiv(m, 256), m), 256, 0, st>>>(m, m, SA, m, dTA, lddta); }
  if (!rc) rc = copy2d<Hh>(n, n, TB, ldtb, SB, n, st);
  if (!rc) { add_kernel<Hh><<<dim3(cdiv(n, 256), n), 256, 0, st>>>(n, n, SB, n, dTB, lddtb); }
  if (!rc) rc = copy2d<Hh>(m, n, Y0, ldy0, Y, ldy, st);
  if (rc) return rc;
  rc = refine_loop<Hh, Hh>(m, n, TA, TB, b_lower, SA, SB, C, Y, R, nullptr, nullptr, nullptr, 64, eps, max_iter, t, t,
                           part, red, ints, st, rep);
  if (rc) return rc;
  if (rep->status == SYLV_SINGULAR_EQUATION) return 0;
  // residual of the perturbed problem (refinement.py:141)
  rc = gemm<Hh>('N', 'N', m, n, m, Hh(1), SA, m, Y, ldy, Hh(0), R, m, st);
  if (!rc) rc = gemm<Hh>('N', 'N', m, n, n, Hh(1), Y, ldy, SB, n, Hh(1), R, m, st);
  if (rc) return rc;
  double nr[3], nA[3], nB[3], nC[3], nX[3];
  rc = read_reduce<Hh>(R, m, n, m, C, ldc, 1, part, red, nr, st);
  if (!rc) rc = read_reduce<Hh>(SA, m, m, m, nullptr, 0, 0, part, red, nA, st);
  if (!rc) rc = read_reduce<Hh>(SB, n, n, n, nullptr, 0, 0, part, red, nB, st);
  if (!rc) rc = read_reduce<Hh>((Hh*)C, m, n, ldc, nullptr, 0, 0, part, red, nC, st);
  if (!rc) rc = read_reduce<Hh>(Y, m, n, ldy, nullptr, 0, 0, part, red, nX, st);
  if (rc) return rc;
  double num = std::sqrt(nr[0]), den = std::sqrt(nC[0]) + std::sqrt(nX[0]) * (std::sqrt(nA[0]) + std::sqrt(nB[0]));
  rep->residual = den == 0.0 ? 0.0 : num / den;
  return 0;
}

int sylv_refine(int dtype, int m, int n, const void* TA, int ldta, const void* dTA, int lddta, const void* TB,
                int ldtb, const void* dTB, int lddtb, int b_lower, const void* C, int ldc, const void* Y0, int ldy0,
                double epsilon, int max_iter, void* Y, int ldy, void* ws, size_t ws_bytes, void* stream,
                sylv_report* rep) {
  if ((dtype != 1 && dtype != 3) || m < 1 || n < 1 || max_iter < 1 || !rep) return SYLV_EINVAL;
  int rc = ctx_init();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 1)
    return refine_entry<double>(m, n, (const double*)TA, ldta, (const double*)dTA, lddta, (const double*)TB, ldtb,
                                (const double*)dTB, lddtb, b_lower, (const double*)C, ldc, (const double*)Y0, ldy0,
                                epsilon, max_iter, (double*)Y, ldy, ws, ws_bytes, st, rep);
  return refine_entry<cdouble>(m, n, (const cdouble*)TA, ldta, (const cdouble*)dTA, lddta, (const cdouble*)TB, ldtb,
                               (const cdouble*)dTB, lddtb, b_lower, (const cdouble*)C, ldc, (const cdouble*)Y0, ldy0,
                               epsilon, max_iter, (cdouble*)Y, ldy, ws, ws_bytes, st, rep);
}

// ---- schur -------------------------------------------------------------------
template <class S>
static size_t schur_ws_bytes(int m) {
  Arena ar(nullptr, 0);
  SchurWs<S> w;
  SchurWs<S>::carve(ar, m, w);
  return ar.off + 256;
}
int sylv_schur_workspace_size(int dtype, int m, size_t* bytes) {
  if (!valid_dtype(dtype) || m < 1) return SYLV_EINVAL;
  *bytes = dtype == 0 ? schur_ws_bytes<float>(m)
                      : dtype == 1 ? schur_ws_bytes<double>(m)
                                   : dtype == 2 ? schur_ws_bytes<cfloat>(m) : schur_ws_bytes<cdouble>(m);
  return 0;
}
template <class S>
static int schur_entry(int m, void* A, int lda, void* U, int ldu, void* ws, size_t wsb, cudaStream_t st, int* info) {
  Arena ar(ws, wsb);
  SchurWs<S> w;
  SchurWs<S>::carve(ar, m, w);
  if (!ar.ok()) return SYLV_EWORKSPACE;
  SchurStats s{};
  int rc = schur_device<S>(m, (S*)A, lda, (S*)U, ldu, w, st, &s);
  if (rc) return rc;
  MSY_CK(host_sync(st));
  if (info) { info[0] = s.status; info[1] = s.sweeps; info[2] = s.small_calls; info[3] = s.windows; }
  if (getenv("MSY_SCHUR_TIMING"))
    fprintf(stderr,
            "schur m=%d: hess %.1f ms, scan %.1f, small %.1f, shift %.1f, sweep %.1f, aed %.1f | qr sweeps %d, "
            "aed windows %d deflating %d\n",
            m, s.ms_hess, s.ms_scan, s.ms_small, s.ms_shift, s.ms_sweep, s.ms_aed, s.ms_sweeps, s.aed_calls,
            s.aed_deflated);
  return 0;
}
int sylv_schur(int dtype, int m, void* A, int lda, void* U, int ldu, void* ws, size_t ws_bytes, void* stream,
               int* info) {
  if (!valid_dtype(dtype) || m < 1 || lda < m || ldu < m) return SYLV_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case 0: return schur_entry<float>(m, A, lda, U, ldu, ws, ws_bytes, st, info);
    case 1: return schur_entry<double>(m, A, lda, U, ldu, ws, ws_bytes, st, info);
    case 2: return schur_entry<cfloat>(m, A, lda, U, ldu, ws, ws_bytes, st, info);
    default: return schur_entry<cdouble>(m, A, lda, U, ldu, ws, ws_bytes, st, info);
  }
}

// ---- trsyl -----------------------------------------------------------------------
int sylv_trsyl_workspace_size(int dtype, int m, int n, size_t* bytes) {
  if (!valid_dtype(dtype) || m < 1 || n < 1) return SYLV_EINVAL;
  Arena ar(nullptr, 0);
  switch (dtype) {  // the left-looking partials are sized by the element type
    case 0: { TrsylWs<float> w; TrsylWs<float>::carve(ar, m, n, w); break; }
    case 1: { TrsylWs<double> w; TrsylWs<double>::carve(ar, m, n, w); break; }
    case 2: { TrsylWs<cfloat> w; TrsylWs<cfloat>::carve(ar, m, n, w); break; }
    default: { TrsylWs<cdouble> w; TrsylWs<cdouble>::carve(ar, m, n, w); break; }
  }
  ar.get<int>(8);
  ar.get<double>(3 * RED_BLOCKS + 16);
  *bytes = ar.off + 256;
  return 0;
}
template <class S>
static int trsyl_entry(int m, int n, const void* TA, int ldta, const void* TB, int ldtb, int lowerB, void* W, int ldw,
                       void* ws, size_t wsb, cudaStream_t st, int* info) {
  Arena ar(ws, wsb);
  TrsylWs<S> w;
  TrsylWs<S>::carve(ar, m, n, w);
  int* stat = ar.get<int>(8);
  double* part = ar.get<double>(3 * RED_BLOCKS + 16);
  if (!ar.ok()) return SYLV_EWORKSPACE;
  trsyl_status_init<<<1, 1, 0, st>>>(stat);
  int rc = trsyl<S>(m, n, (const S*)TA, ldta, (const S*)TB, ldtb, lowerB, (S*)W, ldw, w, stat, st);
  if (rc) return rc;
  int row = -1, col = -1;
  int ts = read_trsyl_status(stat, m, n, lowerB, &row, &col, st);
  if (ts < 0) return ts;
  if (ts == SYLV_OK) {
    double o[3];
    rc = read_reduce<S>((S*)W, m, n, ldw, nullptr, 0, 0, part, part + 3 * RED_BLOCKS, o, st);
    if (rc) return rc;
    if (!std::isfinite(o[0])) {
      ts = SYLV_NUMERIC_BREAKDOWN;
      rc = first_nonfinite_col<S>((S*)W, m, n, ldw, lowerB, stat + 4, &col, st);
      if (rc) return rc;
    }
  }
  if (info) { info[0] = ts; info[1] = row; info[2] = col; }
  return 0;
}
int sylv_trsyl(int dtype, int m, int n, const void* TA, int ldta, const void* TB, int ldtb, int b_lower, void* W,
               int ldw, void* ws, size_t ws_bytes, void* stream, int* info) {
  if (!valid_dtype(dtype) || m < 1 || n < 1 || ldta < m || ldtb < n || ldw < m) return SYLV_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case 0: return trsyl_entry<float>(m, n, TA, ldta, TB, ldtb, b_lower, W, ldw, ws, ws_bytes, st, info);
    case 1: return trsyl_entry<double>(m, n, TA, ldta, TB, ldtb, b_lower, W, ldw, ws, ws_bytes, st, info);
    case 2: return trsyl_entry<cfloat>(m, n, TA, ldta, TB, ldtb, b_lower, W, ldw, ws, ws_bytes, st, info);
    default: return trsyl_entry<cdouble>(m, n, TA, ldta, TB, ldtb, b_lower, W, ldw, ws, ws_bytes, st, info);
  }
}

// ---- orth (mgs_qr) ---------------------------------------------------------------
int sylv_orth_workspace_size(int dtype, int m, size_t* bytes) {
  if ((dtype != 1 && dtype != 3) || m < 1) return SYLV_EINVAL;
  *bytes = 256 + 64 * sizeof(int) + 16 * sizeof(double) + 3 * RED_BLOCKS * sizeof(double) + 1024;
  return 0;
}
template <class S>
static int orth_entry(int m, const void* U, int ldu, void* Q, int ldq, void* R, int ldr, void* ws, size_t wsb,
                      cudaStream_t st, int* info) {
  Arena ar(ws, wsb);
  int* flag = ar.get<int>(64);
  double* red = ar.get<double>(16);
  double* part = ar.get<double>(3 * RED_BLOCKS);
  if (!ar.ok()) return SYLV_EWORKSPACE;
  MSY_CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
  fill<double>(1, 1, INFINITY, red + 8, 1, st);
  int rc = orth_cholqr<S>(m, (const S*)U, ldu, (S*)Q, ldq, (S*)R, ldr, flag, red + 8, st);
  if (rc) return rc;
  double o[3];
  rc = read_reduce<S>((S*)U, m, m, ldu, nullptr, 0, 0, part, red, o, st);
  if (rc) return rc;
  int hflag;
  double hdiag;
  MSY_CK(d2h(&hflag, flag, sizeof(int), st));
  MSY_CK(d2h(&hdiag, red + 8, sizeof(double), st));
  MSY_CK(host_sync(st));
  if (info) info[0] = (hflag || hdiag <= m * tr<S>::u() * std::sqrt(o[0])) ? SYLV_RANK_DEFICIENT : SYLV_OK;
  return 0;
}
int sylv_orth(int dtype, int m, const void* U, int ldu, void* Q, int ldq, void* R, int ldr, void* ws,
              size_t ws_bytes, void* stream, int* info) {
  if ((dtype != 1 && dtype != 3) || m < 1 || ldu < m || ldq < m || ldr < m) return SYLV_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 1) return orth_entry<double>(m, U, ldu, Q, ldq, R, ldr, ws, ws_bytes, st, info);
  return orth_entry<cdouble>(m, U, ldu, Q, ldq, R, ldr, ws, ws_bytes, st, info);
}

// ---- gemm --------------------------------------------------------------------------
int sylv_gemm(int dtype, char opa, char opb, int m, int n, int k, const void* alpha, const void* A, int lda,
              const void* B, int ldb, const void* beta, void* C, int ldc, void* stream) {
  if (!valid_dtype(dtype) || m < 0 || n < 0 || k < 0) return SYLV_EINVAL;
  if ((opa != 'N' && opa != 'T' && opa != 'C') || (opb != 'N' && opb != 'T' && opb != 'C')) return SYLV_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case 0: return gemm<float>(opa, opb, m, n, k, *(const float*)alpha, (const float*)A, lda, (const float*)B, ldb,
                               *(const float*)beta, (float*)C, ldc, st);
    case 1: return gemm<double>(opa, opb, m, n, k, *(const double*)alpha, (const double*)A, lda, (const double*)B, ldb,
                                *(const double*)beta, (double*)C, ldc, st);
    case 2: return gemm<cfloat>(opa, opb, m, n, k, *(const cfloat*)alpha, (const cfloat*)A, lda, (const cfloat*)B,
                                ldb, *(const cfloat*)beta, (cfloat*)C, ldc, st);
    default: return gemm<cdouble>(opa, opb, m, n, k, *(const cdouble*)alpha, (const cdouble*)A, lda,
                                  (const cdouble*)B, ldb, *(const cdouble*)beta, (cdouble*)C, ldc, st);
  }
}

// ---- Hermitian fast path: entrywise division by the eigenvalue sums ---------------
// W[i, j] /= dA[i] + dB[j] (solve_hermitian, sylvester.py:181-196); the first exactly zero
// denominator in row-major order (np.argwhere(denom == 0)[0]) is reported in info[1..2].
template <class S>
__global__ void hdiv_kernel(int m, int n, const double* __restrict__ dA, const double* __restrict__ dB, S* W, int ldw,
                            int* first_zero) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  for (int jj = j; jj < n; jj += gridDim.y) {
    if (i >= m) continue;
    const double d = dA[i] + dB[jj];
    if (d == 0.0) atomicMin(first_zero, i * n + jj);
    S* w = W + i + (size_t)jj * ldw;
    *w = *w * S(1.0 / d);
  }
}
template <class S>
static int hdiv_entry(int m, int n, const double* dA, const double* dB, void* W, int ldw, void* ws, size_t wsb,
                      cudaStream_t st, int* info) {
  if (!ws || wsb < sizeof(int)) return SYLV_EWORKSPACE;
  int* fz = (int*)ws;
  first_nonfinite_init_kernel<<<1, 1, 0, st>>>(fz);
  MSY_LAUNCH_CK();
  hdiv_kernel<S><<<dim3(cdiv(m, 256), std::min(n, 65535)), 256, 0, st>>>(m, n, dA, dB, (S*)W, ldw, fz);
  MSY_LAUNCH_CK();
  int h = 0;
  MSY_CK(d2h(&h, fz, sizeof(int), st));
  if (info) {
    info[0] = h == 0x7fffffff ? SYLV_OK : SYLV_SINGULAR_EQUATION;
    info[1] = h == 0x7fffffff ? -1 : h / n;
    info[2] = h == 0x7fffffff ? -1 : h % n;
  }
  return 0;
}
int sylv_hdiv(int dtype, int m, int n, const double* dA, const double* dB, void* W, int ldw, void* ws,
              size_t ws_bytes, void* stream, int* info) {
  if ((dtype != 1 && dtype != 3) || m < 1 || n < 1 || ldw < m || !dA || !dB || !W) return SYLV_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 1) return hdiv_entry<double>(m, n, dA, dB, W, ldw, ws, ws_bytes, st, info);
  return hdiv_entry<cdouble>(m, n, dA, dB, W, ldw, ws, ws_bytes, st, info);
}

// ---- GMRES-IR Arnoldi step (krylov.cuh) ---------------------------------------------
template <class S>
static int krylov_entry(int N, void* V, int ldv, int j, void* w, void* h_host, void* ws, size_t wsb, cudaStream_t st) {
  const int G = krylov_grid<S>(N);
  if (G <= 0) return SYLV_ECUDA;
  Arena ar(ws, wsb);
  S* part = ar.get<S>((size_t)2 * G);
  S* hd = ar.get<S>((size_t)j + 2);
  if (!ar.ok()) return SYLV_EWORKSPACE;
  int rc = krylov_mgs<S>(N, (S*)V, ldv, j, (S*)w, hd, part, G, st);
  if (rc) return rc;
  MSY_CK(d2h(h_host, hd, sizeof(S) * (size_t)(j + 2), st));
  return 0;
}
int sylv_krylov_workspace_size(int dtype, int N, int j, size_t* bytes) {
  if (!valid_dtype(dtype) || N < 1 || j < -1 || !bytes) return SYLV_EINVAL;
  const size_t es = dtype == 0 ? 4 : (dtype == 3 ? 16 : 8);
  *bytes = es * (2 * 2 * 148 * 8 + (size_t)j + 2) + 1024;  // partials for up to 8 blocks/SM x 148 SMs, x2
  return 0;
}
int sylv_krylov_mgs(int dtype, int N, void* V, int ldv, int j, void* w, void* h, void* ws, size_t ws_bytes,
                    void* stream) {
  if (!valid_dtype(dtype) || N < 1 || j < -1 || ldv < N || !V || !w || !h) return SYLV_EINVAL;
  if ((size_t)(j + 2) * (dtype == 3 ? 16 : 8) > 4096) return SYLV_EINVAL;  // readback staging cap
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case 0: return krylov_entry<float>(N, V, ldv, j, w, h, ws, ws_bytes, st);
    case 1: return krylov_entry<double>(N, V, ldv, j, w, h, ws, ws_bytes, st);
    case 2: return krylov_entry<cfloat>(N, V, ldv, j, w, h, ws, ws_bytes, st);
    default: return krylov_entry<cdouble>(N, V, ldv, j, w, h, ws, ws_bytes, st);
  }
}

// ---- solve with caller-supplied Schur factors (the 2-GPU split: Schur(B) on another GPU) ----
int sylv_solve_factored(const sylv_params* p, const void* A, int lda, const void* B, int ldb, const void* C, int ldc,
                        void* X, int ldx, const void* TA, int ldta, const void* UA, int ldua, const void* TB, int ldtb,
                        const void* UB, int ldub, void* ws, size_t ws_bytes, void* stream, sylv_report* rep) {
  if (!p || !TA || !UA || !TB || !UB || ldta < p->m || ldua < p->m || ldtb < p->n || ldub < p->n) return SYLV_EINVAL;
  if (p->variant == SYLV_VARIANT_BS) return SYLV_EUNSUPPORTED;
  GivenFactors g{TA, UA, TB, UB, ldta, ldua, ldtb, ldub};
  t_given = &g;
  const int rc = sylv_solve(p, A, lda, B, ldb, C, ldc, X, ldx, ws, ws_bytes, stream, rep);
  t_given = nullptr;
  return rc;
}

