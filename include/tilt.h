/*
 * tilt.h — C ABI of libtilt, a B200-native (sm_100a) batched TILT solver.
 *
 * Method: Ren & Lin, "Linearized Alternating Direction Method with Adaptive Penalty and Warm
 * Starts for Fast Solving Transform Invariant Low-Rank Textures", arXiv 1205.5351
 * (/root/reference/PAPER.md, cited as P:<line>).
 *
 * Problem per patch (Eq. TILT_2/TILT_3):
 *     min_{A,E,tau} ||A||_* + lambda ||E||_1   s.t.   D o tau + J dtau = A + E
 * solved by Algorithm 1: outer linearisation in tau, LADMAP inner loop with adaptive
 * penalty (Eqs. A, E, Y, mu, rho), the W^TW projector with centre+area constraints
 * (P:654-749), variable warm starts (Eq. warm_start, Eq. Y_new_warmstart) and
 * a warm-started SVD inside the singular value thresholding (the SVD warm-start idea of §5,
 * realised as one-sided Jacobi seeded with the previous right singular vectors).
 *
 * Conventions:
 *  - Images: fp32 intensities, [n_images][H][W] row-major.
 *  - Box: int32 {x0, y0, w, h}; the window is m = h rows by n = w columns. All boxes of one call
 *    share (m, n).
 *  - tau: normalised coordinates (reading Z15): window centre c = (x0+(n-1)/2, y0+(m-1)/2),
 *    scale s = max(m,n)/2, u = (x - c_x)/s. Parameter order (h11, h12, h21, h22, h13, h23) for
 *    TILT_AFFINE (p = 6) and (..., h31, h32) for TILT_HOMOGRAPHY (p = 8) (reading Z16);
 *    identity = (1,0,0,1,0,0[,0,0]).
 *  - Patch matrices (A, E, D_hat, M): [m][n] row-major (pixel (i,j) -> i*n + j, reading Z1).
 *  - Jacobian planes: [p][m][n] row-major per parameter.
 *
 * Memory ownership: every array pointer passed to a *_batch call is CALLER-OWNED DEVICE memory
 * (cudaMalloc / torch CUDA tensors) unless the function name ends in _host. The library owns only
 * the workspace it allocates in tilt_create. Inputs are never written. Calls are asynchronous on
 * the handle's stream (tilt_set_stream); the caller synchronises. A handle is not thread-safe.
 * Exception: the multi-CTA path (windows above 128 x 128) creates, on its first call, a private
 * capture stream and up to two CUDA-graph executables of an SVT's device-side Jacobi sweep loop
 * (rebuilt when the call's arguments change); they are released by tilt_destroy.
 *
 * Errors: every entry point returns a tilt_status; no exception crosses the ABI. Per-patch
 * failures never abort a batch: they are reported in tilt_report.status and the patch keeps its
 * last tau / A / E.
 */
#ifndef TILT_H_
#define TILT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TILT_ABI_VERSION 1

typedef enum {
  TILT_OK = 0,
  TILT_E_ARG = 1,   /* shape / p mismatch, m or n above the handle's maxima, non-finite params,
                       B above max_batch, NULL required pointer */
  TILT_E_CUDA = 2,  /* a CUDA runtime call failed (message: tilt_last_error) */
  TILT_E_OOM = 3,   /* workspace allocation failed in tilt_create */
  TILT_E_UNSUPPORTED = 4
} tilt_status;

typedef enum { TILT_AFFINE = 0, TILT_HOMOGRAPHY = 1 } tilt_transform;

/* Per-patch status (tilt_report.status). */
typedef enum {
  TILT_PATCH_CONVERGED = 0,     /* an outer stop rule fired (reading Z9) */
  TILT_PATCH_MAX_OUTER = 1,     /* max_outer reached without a stop rule */
  TILT_PATCH_WINDOW_ESCAPE = 2, /* a bilinear 4-tap stencil left the image (reading Z2) */
  TILT_PATCH_SINGULAR_GRAM = 3, /* Cholesky of J^TJ + Q^TQ failed (J not full rank) */
  TILT_PATCH_ZERO_PATCH = 4,    /* ||D o tau||_F = 0 (normalisation of Alg. 1 Step 1 undefined) */
  TILT_PATCH_DIVERGED = 5,      /* NaN/Inf or objective > 1e12 */
  TILT_PATCH_BAD_BOX = 6        /* the patch's box is not win_w x win_h (every box of a call must have
                                   the call's window size); the patch is not solved, tau_out = tau0 */
} tilt_patch_status;

typedef enum { TILT_CONSTRAINTS_NONE = 0, TILT_CONSTRAINTS_CENTER_AREA = 1 } tilt_constraint_mode;

/* Solver parameters (host struct, passed by pointer, copied at the call). The paper states no
 * values; defaults (tilt_default_params) are DESIGN.md's readings Z3-Z9, Z14. */
typedef struct {
  float lambda;           /* <= 0 -> 1/sqrt(max(m,n)) (Z8) */
  float mu0_scale;        /* mu_0 = mu0_scale / sigma_1(D_hat), reset each inner loop (Z3, Z5) */
  float mu_max_ratio;     /* mu_max = mu_max_ratio * mu_0 (Z6) */
  float rho0;             /* Eq. rho, >= 1 */
  float eps1;             /* Eq. Cond1 tolerance */
  float eps2;             /* Eq. Cond2 / Eq. rho tolerance */
  float obj_tol;          /* outer stop: relative objective change (Z9) */
  float tau_tol;          /* outer stop: ||dtau||_inf (Z9) */
  int32_t max_inner;      /* inner iteration cap per outer iteration */
  int32_t max_outer;      /* outer iteration cap */
  int32_t constraint_mode;/* tilt_constraint_mode (Z10) */
  int32_t vws;            /* 1: variable warm start of A, E, Y */
  int32_t svd_warm;       /* 1: warm-start the Jacobi SVD with the previous V */
  int32_t pyramid_levels; /* 1 or 2 (Z18) */
  float jacobi_tol;       /* <= 0 -> 8 sqrt(m) 2^-24 (Z14) */
  int32_t jacobi_max_sweeps;
  /* test-only controls (0 / NULL in production) */
  int32_t fixed_inner_iters;  /* > 0: exactly this many inner iterations (no early stop) */
  int32_t fixed_outer_iters;  /* > 0: exactly this many outer iterations */
  const uint8_t* rho_replay;  /* device [B][max_outer][max_inner] or NULL (Z21): bit 0 = rho decision
                                 (1: rho0), bit 1 = end the inner loop after this iteration */
  float* trace;               /* device [B][max_outer][max_inner][4] (mu, crit1, crit2, rho) or NULL;
                                 the multi-CTA path adds 2 to the rho slot when the iteration took
                                 Algorithm 2's warm step (svd_mode 1) */
  /* window size of the call (all boxes share it; a patch whose box differs is reported
   * TILT_PATCH_BAD_BOX and not solved). 0: read back from boxes[0] with a stream sync;
   * > 0: taken as given. Host syncs: none on the CTA-per-patch kernels when win_h, win_w > 0 (the
   * call is then graph-capturable); the multi-CTA path (kernel_path 3, windows above 128 x 128 on
   * auto, svd_mode 1) drives its LADMAP / outer loops from the host and synchronises the stream to
   * read its active-problem counter once per LADMAP / outer iteration (an SVT's Jacobi sweeps run
   * as a device-side CUDA-graph loop), so it returns
   * TILT_E_UNSUPPORTED on a capturing stream; the same holds for win_h/win_w = 0. */
  int32_t win_h, win_w;
  /* kernel family: 0 = auto (the CTA-per-patch kernels up to 128 x 128, the multi-CTA path above:
   * at 200 x 200 it is 2.4x faster; the ADM inner entry stays on the CTA kernels up to 256),
   * 1 = CTA-per-patch kernels, 3 = multi-CTA path (m, n <= 1024: one problem spread over many
   * CTAs, block-cyclic Jacobi, hand-written batched GEMM and LU). 2 (a
   * warp-per-patch kernel, round 1) is retired: TILT_E_ARG. All compute the same method; they
   * differ in data layout, Jacobi ordering and how a problem maps to the GPU. */
  int32_t kernel_path;
  /* Newton-Schulz re-orthonormalisation of the carried V (reading Z14) after every ns_period-th
   * LADMAP SVT of an inner loop (and after the last one); <= 1: after every SVT. Default 4 (the
   * column scales are renormalised exactly every SVT; the slow orthogonality drift is corrected
   * every 4th; fixed-count parity is tested at 1 and 4). */
  int32_t ns_period;
  /* inner solver: 0 = LADMAP (the paper's), 1 = the ADM baseline of Zhang et al. as
   * restated in P:241-264 (three variables, mu_{k+1} = adm_rho mu_k unbounded, cold start every outer
   * iteration, dtau from the ADM). CTA kernels and the multi-CTA path (not the
   * retired warp-per-patch kernel; not with svd_mode 1). */
  int32_t inner_solver;
  float adm_rho;          /* ADM penalty growth (default 1.25) */
  float adm_tol;          /* ADM stop: ||D + J dtau - A - E||_F / ||D||_F < adm_tol (default 1e-6: the
                             fp32 residual floor is ~1e-7, as for eps1; the fp64 oracle reproduces
                             Table 1's ADM counts at 1e-7) */
  /* persistent-grid size of the CTA-per-patch solve: at most this many patches in flight per SM
   * (0: the occupancy limit). Fewer in-flight patches run faster each, which shortens the tail of
   * a batch whose per-patch work varies widely. */
  int32_t ctas_per_sm;
  /* 2-level pyramid only: 1 = the fine level's first inner loop starts from the coarse level's A, E,
   * Y replicated 2x2 and halved (reading Z26; needs vws); 0 = tau only (Z18). */
  int32_t pyramid_warm;
  /* SVT of the LADMAP iterations: 0 = warm one-sided Jacobi every iteration; 1 = LADMAP+SVDWS
   * (Algorithm 2): when ||M_k - M_{k-1}||_F < svd_ws_gate ||D||_F one Taylor step along
   * the Cayley curve from the previous SVD replaces the Jacobi SVT (reading Z27; multi-CTA path,
   * tilt_inner_batch, m >= n). */
  int32_t svd_mode;
  float svd_ws_gate;      /* default 2e-5 */
} tilt_params;

/* Per-patch report (device array written by tilt_solve_batch). */
typedef struct {
  int32_t status;         /* tilt_patch_status */
  int32_t stop_rule;      /* 0 none, 1 objective change, 2 dtau, 3 max_outer (Z9) */
  int32_t outer_iters;
  int32_t inner_iters;    /* LADMAP iterations summed over outer iterations */
  int32_t jacobi_sweeps;  /* Jacobi sweeps summed over the LADMAP SVTs */
  int32_t aux_sweeps;     /* Jacobi sweeps of the per-outer sigma_1(D_hat) SVDs (mu_0, Z3) */
  int32_t rank;           /* #{sigma_j(A) > 1e-3 sigma_1(A)} (Z19) */
  int32_t rank_band;      /* 1 if some sigma_j(A)/sigma_1(A) lies in [3e-4, 3e-3] */
  int32_t svt_rank;       /* #{sigma_j(M_K) > 1/mu_K} of the last SVT */
  int32_t sweep_cap_hits; /* SVTs that stopped at jacobi_max_sweeps */
  float objective;        /* ||A||_* + lambda ||E||_1 at the last inner exit */
  float crit1;            /* Cond1 value at the last inner exit */
  float crit2;            /* Cond2 value at the last inner exit */
  float patch_norm;       /* ||D o tau||_F at the last outer iteration */
  float dtau_inf;         /* ||dtau||_inf of the last outer iteration */
  float mu_last;          /* mu_K of the last SVT */
  int32_t jacobi_rotations; /* Jacobi rotations applied, summed over the LADMAP SVTs */
  int32_t kernel_path;      /* 1: CTA-per-patch kernel, 3: multi-CTA path */
  int32_t svd_warm_steps;   /* SVTs replaced by the Alg. 2 warm step (svd_mode 1) */
} tilt_report;

typedef struct {
  int32_t device;        /* CUDA device ordinal */
  void* stream;          /* cudaStream_t, NULL = legacy default stream */
  int32_t max_batch;     /* largest B of any call */
  int32_t max_m, max_n;  /* largest window (<= 1024 each; tilt_solve_batch serves windows up to
                            256 x 256, tilt_inner_batch / tilt_svt_batch up to 1024 x 1024) */
  int32_t max_p;         /* 6 or 8 */
  int64_t max_image_elems; /* largest n_images*H*W of a pyramid call (0: no pyramid workspace) */
} tilt_create_opts;

typedef struct tilt_handle tilt_handle;

/* Library / handle lifetime ------------------------------------------------------------------ */

int32_t tilt_abi_version(void);
const char* tilt_status_string(tilt_status s);
const char* tilt_patch_status_string(int32_t s);
/* Last CUDA error message of this thread (static storage). */
const char* tilt_last_error(void);
/* Fills *prm with the defaults (no GPU needed). */
tilt_status tilt_default_params(tilt_params* prm);

/* Allocates all device workspace (library-owned). *h is NULL on failure. */
tilt_status tilt_create(tilt_handle** h, const tilt_create_opts* o);
/* Frees the workspace; h may be NULL. */
tilt_status tilt_destroy(tilt_handle* h);
tilt_status tilt_set_stream(tilt_handle* h, void* stream);

/* The hot entry (north_star) --------------------------------------------------
 * Batched Algorithm 1 over B independent patches: a persistent CTA pool pops patch indices from a
 * device work queue (one patch per CTA at a time) and runs warp/Jacobian -> orthonormalise ->
 * LADMAP (warm Jacobi SVT) -> dtau until each patch retires.
 *   images      [n_images][H][W] fp32        patch_image [B] int32 (patch -> image)
 *   boxes       [B][4] int32                 tau0 [B][p] fp32 or NULL (identity)
 *   tau_out     [B][p] fp32                  A_out, E_out [B][m][n] fp32 or NULL
 *   Y_out       [B][m][n] fp32 or NULL (final multiplier Y~ = W^TW Y)
 *   rep         [B] tilt_report or NULL
 * A/E/Y are at the unit-normalised scale of D_hat (Alg. 1 Step 1). B = 0 is a no-op. */
tilt_status tilt_solve_batch(tilt_handle* h, const float* images, int32_t n_images, int32_t H,
                             int32_t W, const int32_t* patch_image, const int32_t* boxes,
                             const float* tau0, int32_t B, int32_t kind, const tilt_params* prm,
                             float* tau_out, float* A_out, float* E_out, float* Y_out,
                             tilt_report* rep);

/* Same as tilt_solve_batch with HOST buffers: copies the inputs to device workspace, solves and
 * copies tau/A/E/reports back, then synchronises the stream (end-to-end entry). */
tilt_status tilt_solve_batch_host(tilt_handle* h, const float* images, int32_t n_images, int32_t H,
                                  int32_t W, const int32_t* patch_image, const int32_t* boxes,
                                  const float* tau0, int32_t B, int32_t kind,
                                  const tilt_params* prm, float* tau_out, float* A_out,
                                  float* E_out, tilt_report* rep);

/* Step-level entries (parity tests, K1 roofline) ----------------------------------------------- */

/* K1: Alg. 1 Step 1 for B patches at the given tau: D_hat = D o tau / ||D o tau||_F and
 * J = d/dtau (D o tau / ||D o tau||_F) (quotient rule), bilinear sampling with the exact
 * interpolant derivative (Z2). win_h, win_w: window size of the call (all boxes share it); <= 0 ->
 * read from boxes[0] with a stream sync (> 0: no host sync, graph-capturable). Outputs: Dhat
 * [B][m][n], J [B][p][m][n] (may be NULL), norm [B] = ||D o tau||_F (may be NULL), status [B]
 * int32 (tilt_patch_status; may be NULL). */
tilt_status tilt_warp_batch(tilt_handle* h, const float* images, int32_t n_images, int32_t H,
                            int32_t W, const int32_t* patch_image, const int32_t* boxes,
                            const float* tau, int32_t B, int32_t kind, int32_t win_h, int32_t win_w,
                            float* Dhat, float* J, float* norm, int32_t* status);

/* K3 core: singular value thresholding S_eps(M) (Eqs. A_1, S_operator) of B matrices
 * [B][m][n] with per-matrix eps [B], by warm one-sided Jacobi. V_io [B][n][n] row-major: input
 * warm start (NULL -> identity) and output right singular vectors (may be NULL). Outputs:
 * A [B][m][n]; sigma [B][n] singular values of M (unsorted, Jacobi column order; may be NULL);
 * sweeps [B] int32 (may be NULL). m, n <= 1024 (above 256: the multi-CTA path, which allocates its
 * workspace on first use, B x ~(10 + p) m n floats). */
tilt_status tilt_svt_batch(tilt_handle* h, const float* M, int32_t B, int32_t m, int32_t n,
                           const float* eps, float* V_io, float* A, float* sigma, int32_t* sweeps);

/* K2: W^TW v = v - J (J^TJ + Q^TQ)^{-1} J^T v  (Eq. Jperpv; Eq. WTW_property)
 * for B problems. J [B][p][m][n]; Q [B][l][p] or NULL (l <= 3); v [B][m][n]. Outputs: Pv [B][m][n];
 * G^{-1}J^T v [B][p] (the Delta tau of Eq. Delta_tau, may be NULL); status [B] (may be NULL). */
tilt_status tilt_project_batch(tilt_handle* h, const float* J, const float* Q, int32_t l,
                               const float* v, int32_t B, int32_t m, int32_t n, int32_t p,
                               float* Pv, float* dtau, int32_t* status);

/* Inner loop only (Table 1's setting P:1001-1012): LADMAP on given D [B][m][n]
 * (not normalised) and J [B][p][m][n] with optional Q [B][l][p], cold start A_0 = D, E_0 = Y_0 = 0.
 * Uses prm (lambda, mu0_scale, mu_max_ratio, rho0, eps1, eps2, max_inner, fixed_inner_iters,
 * rho_replay [B][max_inner], trace [B][max_inner][4], Jacobi controls). Outputs A, E, Y [B][m][n]
 * (Y may be NULL) and rep [B] (inner_iters, jacobi_sweeps, objective, crit1, crit2, rank...).
 * m, n <= 1024: windows above 128 (or prm->kernel_path = 3) run on the multi-CTA path, which
 * synchronises the handle's stream once per LADMAP iteration (it reads an active-problem counter;
 * the Jacobi sweeps of an SVT loop on the device in a CUDA graph). Its workspace (B x ~(10 + p) m n floats, more with svd_mode 1) is made
 * by tilt_create when max_m or max_n exceeds 128, else on first use. */
tilt_status tilt_inner_batch(tilt_handle* h, const float* D, const float* J, const float* Q,
                             int32_t l, int32_t B, int32_t m, int32_t n, int32_t p,
                             const tilt_params* prm, float* A, float* E, float* Y,
                             tilt_report* rep);

/* Kernel family used by tilt_svt_batch: 0 = auto (CTA-per-patch up to 256 x 256, else multi-CTA),
 * 1 = CTA-per-patch, 3 = multi-CTA block-cyclic Jacobi (m, n <= 1024) (step parity of both);
 * 2 (warp-per-patch) is retired: TILT_E_ARG. */
tilt_status tilt_set_svt_path(tilt_handle* h, int32_t path);

/* Number of kernel launches issued by this handle since creation (for bench accounting). */
int64_t tilt_launch_count(const tilt_handle* h);


#ifdef __cplusplus
}
#endif

#endif /* TILT_H_ */
