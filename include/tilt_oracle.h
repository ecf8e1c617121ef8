/* tilt_oracle.h — the fp64 CPU oracle twin of tilt_solve_batch.
 *
 * TEST INFRASTRUCTURE, not the product: only tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline / reference arm load libtilt_oracle.so. It shares no code, header or table with the CUDA
 * path (include/tilt.h, paper_1205_5351_b200/csrc/) and follows Algorithm 1 + LADMAP step by step in
 * the paper's order (PAPER.md P:527-574, P:437-501 with errata E1, E2), in fp64, with its own
 * one-sided Jacobi SVD — the same algorithm and readings as oracle/tilt_oracle.py,
 * against which it is tested (tests/test_oracle_cpp.py).
 *
 * One call solves B independent patches with OpenMP over patches (a patch is sequential).
 */
#ifndef TILT_ORACLE_H_
#define TILT_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double lambda;        /* <= 0 -> 1/sqrt(max(m, n)) (reading Z8) */
  double mu0_scale;     /* mu0 = mu0_scale / sigma_1(D_hat) (Z3), reset every inner loop (Z5) */
  double mu_max_ratio;  /* mu_max = ratio * mu0 (Z6) */
  double rho0;          /* Eq. rho */
  double eps1, eps2;    /* Cond1, Cond2, strict (Z12) */
  double obj_tol;       /* outer stop: relative objective change (Z9) */
  double tau_tol;       /* outer stop: ||dtau||_inf (Z9) */
  int32_t max_inner, max_outer;
  int32_t constraints;  /* 1: centre + area rows Q (Z10); 0: none */
  int32_t vws;          /* 1: variable warm start */
  int32_t fixed_inner;  /* > 0: exactly this many inner iterations (test mode) */
  int32_t fixed_outer;  /* > 0: exactly this many outer iterations (test mode) */
} tilt_oracle_params;

/* Per-patch report: status as tilt.h's tilt_patch_status (0 converged, 1 max_outer, 2 window
 * escape, 3 singular Gram, 4 zero patch, 5 diverged); stop_rule 0 none / 1 objective / 2 dtau /
 * 3 max_outer (Z9); rank by reading Z19. */
typedef struct {
  int32_t status, stop_rule, outer_iters, inner_iters, rank, rank_band, jacobi_sweeps;
  double objective, crit1, crit2, patch_norm;
} tilt_oracle_report;

/* Defaults of DESIGN.md §2 (lambda -1, mu0_scale 1.25, mu_max_ratio 1e6, rho0 2, eps1 1e-6,
 * eps2 0.1, obj_tol 1e-5, tau_tol 1e-4, max_inner 1000, max_outer 50, constraints 1, vws 1). */
void tilt_oracle_default_params(tilt_oracle_params* p);

/* Algorithm 1 on B patches (host fp64 buffers, caller-owned):
 *   images [n_images][H][W] row-major intensities; patch_image [B]; boxes [B][4] = (x0, y0, w, h),
 *   every box of the call the same w = n, h = m; tau0 [B][p] in normalised coordinates (Z15) or
 *   NULL for identity; kind 0 affine (p = 6) / 1 homography (p = 8; parameter order Z16).
 * Outputs: tau_out [B][p]; A_out, E_out [B][m][n] row-major (may be NULL; zero for a patch without
 * a state); rep [B] (may be NULL). n_threads <= 0: all OpenMP threads.
 * Returns 0, or 1 for invalid arguments (sizes, kind, box size mismatch, NULL required pointer). */
int32_t tilt_oracle_solve_batch(const double* images, int32_t n_images, int32_t H, int32_t W,
                                const int32_t* patch_image, const int32_t* boxes, const double* tau0,
                                int32_t B, int32_t kind, const tilt_oracle_params* prm, double* tau_out,
                                double* A_out, double* E_out, tilt_oracle_report* rep, int32_t n_threads);

/* The oracle's singular value shrinkage S_eps(M) by its own one-sided Jacobi SVD
 * (fp64, round-robin pairs, tol 1e-14, <= 60 sweeps): M [m][n] row-major in, A [m][n] out,
 * sigma [min(m, n)] descending out (may be NULL). Returns the sweep count. */
int32_t tilt_oracle_svt(const double* M, int32_t m, int32_t n, double eps, double* A, double* sigma);

#ifdef __cplusplus
}
#endif

#endif /* TILT_ORACLE_H_ */
