/*
 * mpsylv_b200.h -- C ABI of the B200-native mixed-precision Sylvester solver.
 *
 * Drop-in boundary for the reference package `mpsylv` (Python, read-only at
 * /root/reference).  The reference has no FFI of its own (pure Python + numpy,
 * SURVEY.md section 2.2), so each entry point below replaces one Python
 * function of its hot path; a ctypes binding (the reference side would add it
 * exactly as paper_2503_03456_b200/_native.py does) is shown in INTEGRATION.md.
 *
 * Conventions
 *   - matrices are column-major device pointers with leading dimensions;
 *   - `dtype`: 0 = float (s), 1 = double (d), 2 = complex float (c),
 *     3 = complex double (z); complex values are interleaved (re, im);
 *   - `stream` is a cudaStream_t passed as void*;
 *   - the caller owns every buffer, including the workspace (query its size
 *     first); the library performs no device allocation on the solve path;
 *   - return value: SYLV_OK or a negative SYLV_E* code for API/CUDA errors.
 *     Typed numerical outcomes (the reference's exceptions and failure
 *     strings) are reported in `sylv_report.status` / `*info`.
 */
#ifndef MPSYLV_B200_H
#define MPSYLV_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* numerical status codes (sylv_report.status, *info) -- mirror mpsylv.errors
 * (pkg/src/mpsylv/errors.py:4-45) and the SolveReport.failure strings
 * (pkg/src/mpsylv/refinement.py:125-140,185-187,237-245) */
enum {
  SYLV_OK = 0,
  SYLV_SINGULAR_EQUATION = 1,  /* SingularEquationError(row, col)            */
  SYLV_NUMERIC_BREAKDOWN = 2,  /* NumericBreakdownError / "nan_breakdown"    */
  SYLV_ITERATION_LIMIT = 3,    /* IterationLimitError (Schur sweeps)         */
  SYLV_RANK_DEFICIENT = 4,     /* RankDeficiencyError (orthonormalisation)   */
  SYLV_SINGULAR_MATRIX = 5,    /* SingularMatrixError (LU)                   */
  SYLV_FORMAT_OVERFLOW = 6,    /* FormatOverflowError (entering u_l)         */
  SYLV_NON_CONVERGENCE = 7,    /* "non_convergence" failure string           */
};
/* API / runtime errors (negative return values) */
enum {
  SYLV_EINVAL = -1,     /* bad argument (DimensionError / ValueError)   */
  SYLV_EUNSUPPORTED = -2,
  SYLV_EWORKSPACE = -3, /* workspace too small                          */
  SYLV_EINTERNAL = -5,
  SYLV_ECUDA = -100,    /* -100 - cudaError_t                           */
};

enum { SYLV_KIND_GENERAL = 0, SYLV_KIND_LYAPUNOV = 1 };
/* SYLV_VARIANT_BS: the fp64 Bartels-Stewart comparator (sylvester.py:160-178):
 * Schur in binary64 (low_bits must be 64), F = U_A^H C U_B, one triangular solve,
 * X = U_A Y U_B^H; no refinement (iterations = 0). */
enum { SYLV_VARIANT_ORTH = 0, SYLV_VARIANT_INV = 1, SYLV_VARIANT_BS = 2 };
/* where a typed failure happened: inside a refinement correction solve, at the
 * initial (u_l) triangular solve, or as a non-finite iterate after an update */
enum { SYLV_STAGE_REFINEMENT = 0, SYLV_STAGE_INITIAL = 1, SYLV_STAGE_DIVERGED = 2 };

#define SYLV_MAX_NORMS 256

/* RefinementConfig + problem shape (pkg/src/mpsylv/refinement.py:47-75,
 * pkg/src/mpsylv/sylvester.py:47-90) */
typedef struct sylv_params {
  int m, n;
  int kind;                  /* SYLV_KIND_*; lyapunov requires B = A^H          */
  int complex_data;          /* 0: real (fp64 in/out), 1: complex128 in/out     */
  int variant;               /* SYLV_VARIANT_ORTH (mp_orth) / _INV (mp_inv)     */
  int low_bits;              /* u_l: 32 (binary32) or 64 (binary64)             */
  int correction_bits;       /* 64: reference (u_h) corrections; 32: fast mode  */
  int max_iter;              /* RefinementConfig.max_iter (>= 1)                */
  int y0_zero;               /* mp_orth(..., y0_zero=True)                      */
  double epsilon;            /* RefinementConfig.resolve_epsilon(m, n) (> 0)    */
} sylv_params;

/* SolveReport (pkg/src/mpsylv/refinement.py:78-92) plus diagnostics */
typedef struct sylv_report {
  int status;                /* SYLV_* numerical status                         */
  int fail_stage;            /* SYLV_STAGE_* when status is a typed failure     */
  int fail_row, fail_col;    /* SingularEquationError position                  */
  int iterations;            /* computed corrections                            */
  int converged;
  int n_norms;
  double correction_norms[SYLV_MAX_NORMS];
  double residual;           /* ||AX+XB-C||_F/(||C||+||X||(||A||+||B||)), fp64  */
  double backward_error;     /* ||AX+XB-C||_F/((||A||_F+||B||_F)||X||_F)        */
  double norm_x;
  int schur_sweeps_a, schur_sweeps_b;
  double ms_schur, ms_orth, ms_setup, ms_y0, ms_refine, ms_recover, ms_total;
} sylv_report;

/* library identity and diagnostics */
int sylv_version(void);
const char* sylv_status_string(int status);
/* number of kernels this library has launched in the process (bench evidence) */
unsigned long long sylv_launch_count(void);
/* measured arithmetic peak in TFLOP/s: kind 0 = FP32 FFMA, 1 = FP64 DFMA,
 * 2 = FP64 DMMA.8x8x4 (the roofline denominators of the path) */
int sylv_microbench(int kind, double* tflops, void* stream);
/* live kernel-class timer (bench roofline evidence): op 1 = clear + enable,
 * op 0 = disable, op 2 = read and clear.  Classes: 0 fp64 DMMA GEMM, 1 SIMT GEMM,
 * 2 Z application, 3 bulge chase, 4 trsyl step, 5 Hessenberg panel, 6 one-CTA
 * Schur, 7 AED.  On read, per class (arrays of ncls entries): launches, summed
 * event-interval milliseconds, summed algorithmic flops declared at the launch. */
int sylv_ktimer(int op, int ncls, long long* launches, double* ms, double* flops);

/* mp_orth / mp_inv (refinement.py:205-297): A m x m, B n x n, C and X m x n,
 * fp64 (complex_data = 0) or complex128 (complex_data = 1). */
int sylv_workspace_size(const sylv_params* p, size_t* bytes);
int sylv_solve(const sylv_params* p, const void* A, int lda, const void* B, int ldb, const void* C, int ldc,
               void* X, int ldx, void* ws, size_t ws_bytes, void* stream, sylv_report* rep);

/* Batched solve of `batch` independent equations sharing *p (config C4: 512 x
 * mp_orth at m = n = 512).  The reference solves them one by one through
 * mp_orth / mp_inv (refinement.py:205-297; "independent solves may run
 * concurrently"); here `lanes` of them run concurrently, each
 * lane with its own stream, host worker and workspace slice.  A, B, C, X are host
 * arrays of `batch` device pointers (column-major, leading dimensions shared);
 * reports is a host array of `batch` records.  lanes <= 0 selects the default
 * (32).  Each lane keeps its equation's work on one stream, so the process
 * should create its CUDA context with CUDA_DEVICE_MAX_CONNECTIONS >= lanes
 * (the Python package sets 32) or lanes share hardware queues.  The call
 * returns when every equation is done; `stream` is ordered before and after
 * the batch. */
int sylv_batched_workspace_size(const sylv_params* p, int lanes, size_t* bytes);
int sylv_solve_batched(const sylv_params* p, int batch, const void* const* A, int lda, const void* const* B, int ldb,
                       const void* const* C, int ldc, void* const* X, int ldx, int lanes, void* ws, size_t ws_bytes,
                       void* stream, sylv_report* reports);

/* solve_pert_sylv_tri_stat (refinement.py:95-141): stationary refinement of
 * (T_A + dT_A) Y + Y (T_B + dT_B) = C in binary64; T_A upper (quasi-)
 * triangular, T_B upper or lower (quasi-)triangular. dtype 1 or 3. */
int sylv_refine_workspace_size(int dtype, int m, int n, size_t* bytes);
int sylv_refine(int dtype, int m, int n, const void* TA, int ldta, const void* dTA, int lddta, const void* TB,
                int ldtb, const void* dTB, int lddtb, int b_lower, const void* C, int ldc, const void* Y0, int ldy0,
                double epsilon, int max_iter, void* Y, int ldy, void* ws, size_t ws_bytes, void* stream,
                sylv_report* rep);

/* schur (linalg.py:518-577): A (m x m) -> T (in place, (quasi-)upper triangular)
 * and U with A = U T U^H.  dtype 0..3.  info[0] = status, info[1] = sweeps. */
int sylv_schur_workspace_size(int dtype, int m, size_t* bytes);
int sylv_schur(int dtype, int m, void* A, int lda, void* U, int ldu, void* ws, size_t ws_bytes, void* stream,
               int* info);

/* solve_sylv_tri (sylvester.py:111-157): T_A Y + Y T_B = W in place on W.
 * info[0] = status (1 singular, 2 breakdown), info[1] = row, info[2] = col. */
int sylv_trsyl_workspace_size(int dtype, int m, int n, size_t* bytes);
int sylv_trsyl(int dtype, int m, int n, const void* TA, int ldta, const void* TB, int ldtb, int b_lower, void* W,
               int ldw, void* ws, size_t ws_bytes, void* stream, int* info);

/* mgs_qr replacement (linalg.py:252-273): Q = U R^{-1}, R upper with positive
 * real diagonal; dtype 1 or 3.  R (m x m) returned in R. info[0] = status. */
int sylv_orth_workspace_size(int dtype, int m, size_t* bytes);
int sylv_orth(int dtype, int m, const void* U, int ldu, void* Q, int ldq, void* R, int ldr, void* ws,
              size_t ws_bytes, void* stream, int* info);

/* gemm (linalg.py:125-154): C = alpha op(A) op(B) + beta C, op in 'N','T','C'.
 * alpha/beta point to host scalars of the matrix dtype. */
int sylv_gemm(int dtype, char opa, char opb, int m, int n, int k, const void* alpha, const void* A, int lda,
              const void* B, int ldb, const void* beta, void* C, int ldc, void* stream);

/* solve_hermitian (sylvester.py:181-196), its entrywise step: W[i,j] /= dA[i] + dB[j] for the
 * real eigenvalues dA (m) and dB (n) of the Hermitian coefficients (device arrays, double);
 * dtype 1 or 3.  ws: >= 4 bytes of device scratch.  info[0] = SYLV_SINGULAR_EQUATION with
 * info[1..2] = (i, j) of the first exactly zero denominator in row-major order, else SYLV_OK. */
int sylv_hdiv(int dtype, int m, int n, const double* dA, const double* dB, void* W, int ldw, void* ws,
              size_t ws_bytes, void* stream, int* info);

/* mp_orth / mp_inv with the low-precision Schur factors supplied by the caller (the
 * _low_precision_schur_pair step, refinement.py:190-197, done elsewhere -- e.g. Schur(B) on a
 * second GPU): TA, UA (m x m) and TB, UB (n x n) in the low precision of `p` (float for real,
 * complex64 for complex data when low_bits = 32), column-major.  Everything else as
 * sylv_solve; the workspace is sylv_workspace_size's. */
int sylv_solve_factored(const sylv_params* p, const void* A, int lda, const void* B, int ldb, const void* C, int ldc,
                        void* X, int ldx, const void* TA, int ldta, const void* UA, int ldua, const void* TB, int ldtb,
                        const void* UB, int ldub, void* ws, size_t ws_bytes, void* stream, sylv_report* report);

/* GMRES-IR inner solver (gmresir.py:112-205), one Arnoldi step in one launch: modified
 * Gram-Schmidt of w (N) against the columns 0..j of V (N x (j+2), column-major, ld ldv),
 * h[0..j] = the coefficients <v_i, w>, h[j+1] = ||w||_2 (real part), V[:, j+1] = w / ||w||
 * (unless 0 / non-finite); w is overwritten.  h: HOST array of j+2 scalars of the dtype
 * (j + 2 <= 256), filled before return (the call synchronises the stream).  j = -1: only the
 * norm (h[0]) and V[:, 0] = w / ||w||. */
int sylv_krylov_workspace_size(int dtype, int N, int j, size_t* bytes);
int sylv_krylov_mgs(int dtype, int N, void* V, int ldv, int j, void* w, void* h, void* ws, size_t ws_bytes,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPSYLV_B200_H */
