// trsyl.cuh -- T_A Y + Y T_B = W for (quasi-)triangular T_A (upper) and T_B (upper, or
// lower for the Lyapunov adjoint), in place on W.
//
// Replaces the reference's column recurrence `solve_sylv_tri` (pkg/src/mpsylv/sylvester.py:111-157):
// same equation, same ascending (T_B upper) / descending (T_B lower) column order,
// same typed failures -- an exactly singular diagonal pair -> SINGULAR_EQUATION
// at (row, col) (sylvester.py:141-143), non-finite values -> NUMERIC_BREAKDOWN
// (sylvester.py:147-149).  Real Schur factors may carry 2x2 diagonal blocks;
// they are solved as coupled 2x2/4x4 systems and never split across tiles.
//
// B200 design: the m x n unknown is tiled into NB x NB blocks (boundaries nudged
// so no 2x2 block straddles a tile edge).  Block (I,J) depends on the blocks below
// it in its column and before it in its row, so blocks on one anti-diagonal are
// independent.  One kernel launch per anti-diagonal d: every pending block applies
// the two rank-NB GEMM updates coming from diagonal d-1 (in registers, smem-tiled),
// and blocks on diagonal d then solve themselves in shared memory with an
// element-level wavefront over 1x1/2x2 units.  (m/NB + n/NB - 1) launches total.
#pragma once
#include "common.cuh"

namespace msy {

template <class S> struct TrsylCfg { static constexpr int NB = 64; };
template <> struct TrsylCfg<cdouble> { static constexpr int NB = 32; };

enum { TRS_OK = 0, TRS_SINGULAR = 1, TRS_BREAKDOWN = 2 };

// status: [0] = min key (crank*m + m-1-row) of a singular unit, INT_MAX if none
__global__ void trsyl_status_init(int* status) {
  status[0] = 0x7fffffff; status[1] = -1; status[2] = -1; status[3] = 0;
}

// boundaries: rb[0..nbi], cb[0..nbj]; nominal k*NB moved by +1 if it would split a 2x2 block
template <class S>
__global__ void trsyl_partition_kernel(int m, const S* TA, int lda, int n, const S* TB, int ldb, int lowerB, int NB,
                                       int* rb, int nbi, int* cb, int nbj) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k <= nbi) {
    int b = k == nbi ? m : k * NB;
    if (k > 0 && k < nbi && !iszero(TA[b + (size_t)(b - 1) * lda])) b++;
    rb[k] = b;
  }
  if (k <= nbj) {
    int b = k == nbj ? n : k * NB;
    if (k > 0 && k < nbj) {
      S c = lowerB ? TB[(b - 1) + (size_t)b * ldb] : TB[b + (size_t)(b - 1) * ldb];
      if (!iszero(c)) b++;
    }
    cb[k] = b;
  }
}

// solve the pq x pq Kronecker system in place (Gaussian elimination, partial pivoting);
// returns false on an exactly zero pivot
template <class S>
__device__ bool small_solve(int nsys, S M[4][4], S rhs[4]) {
  typedef typename tr<S>::R R;
  for (int c = 0; c < nsys; c++) {
    int p = c;
    R best = abs1(M[c][c]);
    for (int r = c + 1; r < nsys; r++)
      if (abs1(M[r][c]) > best) { best = abs1(M[r][c]); p = r; }
    if (best == R(0)) return false;
    if (p != c) {
      for (int q = 0; q < nsys; q++) { S t = M[c][q]; M[c][q] = M[p][q]; M[p][q] = t; }
      S t = rhs[c]; rhs[c] = rhs[p]; rhs[p] = t;
    }
    for (int r = c + 1; r < nsys; r++) {
      S f = M[r][c] / M[c][c];
      for (int q = c; q < nsys; q++) M[r][q] = M[r][q] - f * M[c][q];
      rhs[r] = rhs[r] - f * rhs[c];
    }
  }
  for (int c = nsys - 1; c >= 0; c--) {
    S s = rhs[c];
    for (int q = c + 1; q < nsys; q++) s = s - M[c][q] * rhs[q];
    rhs[c] = s / M[c][c];
  }
  return true;
}

template <class S>
__global__ void __launch_bounds__(512) trsyl_step_kernel(int m, int n, const S* __restrict__ TA, int lda,
                                                         const S* __restrict__ TB, int ldb, int lowerB, S* W, int ldw,
                                                         const int* __restrict__ rb, const int* __restrict__ cb, int nbi,
                                                         int nbj, int d, int* status) {
  constexpr int NB = TrsylCfg<S>::NB;
  constexpr int MT = (NB + 1 + 3) / 4;  // micro-tile grid (MT x MT threads, 4x4 each)
  constexpr int P = 4 * MT;             // padded tile edge
  const int I = blockIdx.y, J = blockIdx.x;
  const int rI = nbi - 1 - I, cJ = lowerB ? nbj - 1 - J : J;
  const int dd = rI + cJ;
  if (dd < d) return;
  const int i0 = rb[I], i1 = rb[I + 1], j0 = cb[J], j1 = cb[J + 1];
  const int bi = i1 - i0, bj = j1 - j0;
  if (bi <= 0 || bj <= 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* As = (S*)smem_raw;      // [k][i], ld P   (K up to NB+1)
  S* Bs = As + P * P;        // [k][j], ld P
  S* Ws = Bs + P * P;        // W block, [i + j*P]
  __shared__ int ru_start[NB + 2], ru_rank[NB + 2], cu_start[NB + 2], cu_rank[NB + 2];
  __shared__ int ru_of[NB + 2], cu_of[NB + 2];  // rank -> first row / column of the unit
  __shared__ int nru, ncu, s_fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tr_ = tid % MT, tc = tid / MT;
  const bool mt_act = tid < MT * MT;
  S acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b] = S(0);

  // ---- updates from diagonal d-1 ----
  if (d >= 1) {
    // A-part: W -= TA[I, I*] Y[I*, J], with rank(I*) = d-1-cJ
    int ra = d - 1 - cJ;
    if (ra >= 0 && ra < rI) {
      int Is = nbi - 1 - ra;
      int k0 = rb[Is], k1 = rb[Is + 1], bk = k1 - k0;
      for (int e = tid; e < P * P; e += nt) { As[e] = S(0); Bs[e] = S(0); }
      __syncthreads();
      for (int e = tid; e < bi * bk; e += nt) {
        int i = e % bi, k = e / bi;
        As[k * P + i] = TA[(i0 + i) + (size_t)(k0 + k) * lda];
      }
      for (int e = tid; e < bk * bj; e += nt) {
        int k = e % bk, j = e / bk;
        Bs[k * P + j] = W[(k0 + k) + (size_t)(j0 + j) * ldw];
      }
      __syncthreads();
      if (mt_act) {
        for (int k = 0; k < bk; k++) {
          S a[4], b[4];
#pragma unroll
          for (int q = 0; q < 4; q++) { a[q] = As[k * P + tr_ + MT * q]; b[q] = Bs[k * P + tc + MT * q]; }
#pragma unroll
          for (int x = 0; x < 4; x++)
#pragma unroll
            for (int y = 0; y < 4; y++) acc[x][y] = fmac(a[x], b[y], acc[x][y]);
        }
      }
      __syncthreads();
    }
    // B-part: W -= Y[I, J*] TB[J*, J], with rank(J*) = d-1-rI
    int cr = d - 1 - rI;
    if (cr >= 0 && cr < cJ) {
      int Js = lowerB ? nbj - 1 - cr : cr;
      int k0 = cb[Js], k1 = cb[Js + 1], bk = k1 - k0;
      for (int e = tid; e < P * P; e += nt) { As[e] = S(0); Bs[e] = S(0); }
      __syncthreads();
      for (int e = tid; e < bi * bk; e += nt) {
        int i = e % bi, k = e / bi;
        As[k * P + i] = W[(i0 + i) + (size_t)(k0 + k) * ldw];
      }
      for (int e = tid; e < bk * bj; e += nt) {
        int k = e % bk, j = e / bk;
        Bs[k * P + j] = TB[(k0 + k) + (size_t)(j0 + j) * ldb];
      }
      __syncthreads();
      if (mt_act) {
        for (int k = 0; k < bk; k++) {
          S a[4], b[4];
#pragma unroll
          for (int q = 0; q < 4; q++) { a[q] = As[k * P + tr_ + MT * q]; b[q] = Bs[k * P + tc + MT * q]; }
#pragma unroll
          for (int x = 0; x < 4; x++)
#pragma unroll
            for (int y = 0; y < 4; y++) acc[x][y] = fmac(a[x], b[y], acc[x][y]);
        }
      }
      __syncthreads();
    }
  }
  // ---- write back the updated W (or stage it for the leaf solve) ----
  const bool solve = (dd == d);
  if (mt_act) {
#pragma unroll
    for (int x = 0; x < 4; x++) {
      int i = tr_ + MT * x;
      if (i >= bi) continue;
#pragma unroll
      for (int y = 0; y < 4; y++) {
        int j = tc + MT * y;
        if (j >= bj) continue;
        S v = W[(i0 + i) + (size_t)(j0 + j) * ldw] - acc[x][y];
        if (solve) Ws[i + j * P] = v;
        else W[(i0 + i) + (size_t)(j0 + j) * ldw] = v;
      }
    }
  }
  if (!solve) return;
  // ---- leaf: TA_II Y + Y TB_JJ = W_IJ in shared memory ----
  for (int e = tid; e < bi * bi; e += nt) {
    int i = e % bi, k = e / bi;
    As[i + k * P] = TA[(i0 + i) + (size_t)(i0 + k) * lda];
  }
  for (int e = tid; e < bj * bj; e += nt) {
    int i = e % bj, k = e / bj;
    Bs[i + k * P] = TB[(j0 + i) + (size_t)(j0 + k) * ldb];
  }
  __syncthreads();
  if (tid == 0) {
    // row units from the bottom (rank 0 = bottom unit); 2x2 if As[i][i-1] != 0
    int cnt = 0, i = bi - 1;
    while (i >= 0) {
      int st = (i > 0 && !iszero(As[i + (i - 1) * P])) ? i - 1 : i;
      for (int q = st; q <= i; q++) { ru_start[q] = st; ru_rank[q] = cnt; }
      ru_of[cnt] = st;
      cnt++;
      i = st - 1;
    }
    nru = cnt;
    // column units in solve order (upper: left->right; lower: right->left)
    cnt = 0;
    if (!lowerB) {
      int j = 0;
      while (j < bj) {
        int len = (j + 1 < bj && !iszero(Bs[(j + 1) + j * P])) ? 2 : 1;
        for (int q = j; q < j + len; q++) { cu_start[q] = j; cu_rank[q] = cnt; }
        cu_of[cnt] = j;
        cnt++;
        j += len;
      }
    } else {
      int j = bj - 1;
      while (j >= 0) {
        int st = (j > 0 && !iszero(Bs[(j - 1) + j * P])) ? j - 1 : j;
        for (int q = st; q <= j; q++) { cu_start[q] = st; cu_rank[q] = cnt; }
        cu_of[cnt] = st;
        cnt++;
        j = st - 1;
      }
    }
    ncu = cnt;
    s_fail = 0;
  }
  __syncthreads();
  const int nsteps = nru + ncu - 1;
  for (int s = 0; s < nsteps; s++) {
    // phase 1: solve the units on anti-diagonal s (one thread per unit, indexed by row unit rows)
    for (int i = tid; i < bi; i += nt) {
      if (ru_start[i] != i) continue;  // one thread per row unit (its first row)
      int ra = ru_rank[i], cr = s - ra;
      if (cr < 0 || cr >= ncu) continue;
      int jst = cu_of[cr];
      int p = (i + 1 < bi && ru_start[i + 1] == i) ? 2 : 1;
      int q = (jst + 1 < bj && cu_start[jst + 1] == jst) ? 2 : 1;
      S M[4][4], rhs[4];
      int ns = p * q;
      for (int a = 0; a < 4; a++)
        for (int b = 0; b < 4; b++) M[a][b] = S(0);
      // unknown index u = r + p*c  (vec, column-major over the unit)
      for (int c = 0; c < q; c++)
        for (int r = 0; r < p; r++) {
          int uu = r + p * c;
          rhs[uu] = Ws[(i + r) + (jst + c) * P];
          for (int r2 = 0; r2 < p; r2++) M[uu][r2 + p * c] += As[(i + r) + (i + r2) * P];      // TA_RR Y
          for (int c2 = 0; c2 < q; c2++) M[uu][r + p * c2] += Bs[(jst + c2) + (jst + c) * P];  // Y TB_CC
        }
      if (!small_solve<S>(ns, M, rhs)) {
        // singular diagonal pair: report the first in reference order
        int jg = j0 + jst, ig = i0 + i + p - 1;
        int crank = lowerB ? (n - 1 - jg) : jg;
        atomicMin(&status[0], crank * m + (m - 1 - ig));  // decoded on the host
        for (int uu = 0; uu < ns; uu++) rhs[uu] = mk<S>(NAN, NAN);
      }
      for (int c = 0; c < q; c++)
        for (int r = 0; r < p; r++) Ws[(i + r) + (jst + c) * P] = rhs[r + p * c];
    }
    __syncthreads();
    // phase 2: pending entries take the contributions of the units just solved
    for (int e = tid; e < bi * bj; e += nt) {
      int i = e % bi, j = e / bi;
      int ra = ru_rank[i], cr = cu_rank[j];
      if (ra + cr <= s) continue;
      S v = Ws[i + j * P];
      // solved unit in my column unit: row rank s - cr (below me if < ra)
      int rs = s - cr;
      if (rs >= 0 && rs < ra) {
        int st = ru_of[rs];
        int len = (st + 1 < bi && ru_start[st + 1] == st) ? 2 : 1;
        for (int k = st; k < st + len; k++) v = v - As[i + k * P] * Ws[k + j * P];
      }
      int cs = s - ra;
      if (cs >= 0 && cs < cr) {
        int st = cu_of[cs];
        int len = (st + 1 < bj && cu_start[st + 1] == st) ? 2 : 1;
        for (int k = st; k < st + len; k++) v = v - Ws[i + k * P] * Bs[k + j * P];
      }
      Ws[i + j * P] = v;
    }
    __syncthreads();
  }
  for (int e = tid; e < bi * bj; e += nt) {
    int i = e % bi, j = e / bi;
    W[(i0 + i) + (size_t)(j0 + j) * ldw] = Ws[i + j * P];
  }
}

template <class S>
static size_t trsyl_smem() {
  constexpr int P = 4 * ((TrsylCfg<S>::NB + 1 + 3) / 4);
  return (size_t)3 * P * P * sizeof(S);
}

template <class S>
struct TrsylWs {
  int* rb;
  int* cb;
  static void carve(Arena& ar, int m, int n, TrsylWs& w) {
    w.rb = ar.get<int>(m / 1 + 2);
    w.cb = ar.get<int>(n / 1 + 2);
  }
};

// Solve in place; status (device, 4 ints) must be initialised by the caller with
// trsyl_status_init (several solves may share one status word).
template <class S>
int trsyl(int m, int n, const S* TA, int lda, const S* TB, int ldb, int lowerB, S* W, int ldw, TrsylWs<S>& w,
          int* status, cudaStream_t st) {
  constexpr int NB = TrsylCfg<S>::NB;
  static bool attr = false;
  if (!attr) {
    MSY_CK(cudaFuncSetAttribute(trsyl_step_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)trsyl_smem<S>()));
    attr = true;
  }
  const int nbi = cdiv(m, NB), nbj = cdiv(n, NB);
  trsyl_partition_kernel<S><<<cdiv(max(nbi, nbj) + 1, 128), 128, 0, st>>>(m, TA, lda, n, TB, ldb, lowerB, NB, w.rb,
                                                                          nbi, w.cb, nbj);
  MSY_LAUNCH_CK();
  for (int d = 0; d < nbi + nbj - 1; d++) {
    trsyl_step_kernel<S><<<dim3(nbj, nbi), 512, trsyl_smem<S>(), st>>>(m, n, TA, lda, TB, ldb, lowerB, W, ldw, w.rb,
                                                                       w.cb, nbi, nbj, d, status);
    MSY_LAUNCH_CK();
  }
  return 0;
}

}  // namespace msy
