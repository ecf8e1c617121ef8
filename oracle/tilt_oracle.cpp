// tilt_oracle.cpp — the fp64 CPU oracle twin of tilt_solve_batch (include/tilt_oracle.h).
//
// TEST INFRASTRUCTURE: a plain, slow, step-by-step transcription of
// Algorithm 1 + LADMAP with the readings of DESIGN.md §2 — the same
// computation as oracle/tilt_oracle.py, in C++17 fp64 with its own one-sided Jacobi SVD and OpenMP over
// patches. It shares no code with the CUDA path. Every function names the passage it follows.
#include "../include/tilt_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

enum { CONVERGED = 0, MAX_OUTER = 1, WINDOW_ESCAPE = 2, SINGULAR_GRAM = 3, ZERO_PATCH = 4, DIVERGED = 5 };
enum { STOP_NONE = 0, STOP_OBJECTIVE = 1, STOP_DTAU = 2, STOP_MAX_OUTER = 3 };

using Vec = std::vector<double>;

// T_eps(x) = sgn(x) max(|x| - eps, 0)  (Eq. E_1)
inline double shrink(double x, double eps) {
  const double a = std::fabs(x) - eps;
  return a > 0.0 ? (x > 0.0 ? a : -a) : 0.0;
}

double fro(const Vec& x) {
  double s = 0.0;
  for (double v : x) s += v * v;
  return std::sqrt(s);
}

// ---------------------------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi SVD of W (rows x cols, rows >= cols), column-major working copy
// (SURVEY.md §8(c) oracle step 5; the same rotations as oracle.jacobi_svd): round-robin ordering,
// t = sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)), zeta = (beta - alpha)/(2 gamma); a pair is skipped when
// |gamma| <= tol sqrt(alpha beta) or a column is zero to working precision; stop after a sweep
// without rotation. V may come in warm (the result is the same SVD). Returns the sweeps.
// ---------------------------------------------------------------------------------------------
int jacobi_svd(const Vec& Wcm, int rows, int cols, Vec& U, Vec& sigma, Vec& V, bool warm, double tol = 1e-14,
               int max_sweeps = 60) {
  Vec b(Wcm);
  if (!warm) {
    V.assign((size_t)cols * cols, 0.0);
    for (int j = 0; j < cols; ++j) V[(size_t)j * cols + j] = 1.0;
  } else {  // B = W V
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < rows; ++i) {
        double s = 0.0;
        for (int k = 0; k < cols; ++k) s += Wcm[(size_t)k * rows + i] * V[(size_t)j * cols + k];
        b[(size_t)j * rows + i] = s;
      }
  }
  const int nn = cols + (cols & 1), q = nn - 1;
  const double nb = std::max(fro(b), 1e-300);
  const double small = std::pow(cols * 2.220446049250313e-16 * nb, 2);
  int sweeps = 0;
  for (sweeps = 1; sweeps <= max_sweeps; ++sweeps) {
    bool rotated = false;
    for (int r = 0; r < q; ++r) {
      for (int k = 0; k < nn / 2; ++k) {
        const int i = k == 0 ? q : (r + k) % q;
        const int j = k == 0 ? r % q : ((r - k) % q + q) % q;
        if (i >= cols || j >= cols) continue;
        double* bi = &b[(size_t)i * rows];
        double* bj = &b[(size_t)j * rows];
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int e = 0; e < rows; ++e) {
          alpha += bi[e] * bi[e];
          beta += bj[e] * bj[e];
          gamma += bi[e] * bj[e];
        }
        if (!(std::fabs(gamma) > tol * std::sqrt(alpha * beta) && alpha > small && beta > small)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta > 0.0 ? 1.0 : (zeta < 0.0 ? -1.0 : 0.0)) / (std::fabs(zeta) + std::hypot(1.0, zeta));
        if (zeta == 0.0) t = 1.0;
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int e = 0; e < rows; ++e) {
          const double x = bi[e], y = bj[e];
          bi[e] = c * x - s * y;
          bj[e] = s * x + c * y;
        }
        double* vi = &V[(size_t)i * cols];
        double* vj = &V[(size_t)j * cols];
        for (int e = 0; e < cols; ++e) {
          const double x = vi[e], y = vj[e];
          vi[e] = c * x - s * y;
          vj[e] = s * x + c * y;
        }
      }
    }
    if (!rotated) break;
  }
  if (sweeps > max_sweeps) sweeps = max_sweeps;
  sigma.assign(cols, 0.0);
  for (int j = 0; j < cols; ++j) {
    double s = 0.0;
    for (int e = 0; e < rows; ++e) s += b[(size_t)j * rows + e] * b[(size_t)j * rows + e];
    sigma[j] = std::sqrt(s);
  }
  std::vector<int> order(cols);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sigma[x] > sigma[y]; });
  Vec s2(cols), V2((size_t)cols * cols);
  U.assign((size_t)rows * cols, 0.0);
  for (int o = 0; o < cols; ++o) {
    const int j = order[o];
    s2[o] = sigma[j];
    for (int e = 0; e < cols; ++e) V2[(size_t)o * cols + e] = V[(size_t)j * cols + e];
    if (sigma[j] > 0.0)
      for (int e = 0; e < rows; ++e) U[(size_t)o * rows + e] = b[(size_t)j * rows + e] / sigma[j];
  }
  sigma.swap(s2);
  V.swap(V2);
  return sweeps;
}

// S_eps(M) = U T_eps(Sigma) V^T (Eqs. A_1, S_operator) of a row-major m x n matrix; the
// carried V (of the transposed problem when m < n) warm-starts the next call
struct Svt {
  Vec V;
  bool have = false;
  int sweeps = 0;
  // returns A (row-major m x n) and the singular values of M (descending)
  void operator()(const Vec& M, int m, int n, double eps, Vec& A, Vec& sigma) {
    const bool tr = m < n;
    const int rows = tr ? n : m, cols = tr ? m : n;
    Vec W((size_t)rows * cols);  // column-major rows x cols of M (or M^T)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        if (!tr) W[(size_t)j * rows + i] = M[(size_t)i * n + j];
        else W[(size_t)i * rows + j] = M[(size_t)i * n + j];
      }
    Vec U;
    sweeps += jacobi_svd(W, rows, cols, U, sigma, V, have);
    have = true;
    A.assign((size_t)m * n, 0.0);
    for (int k = 0; k < cols; ++k) {
      const double h = shrink(sigma[k], eps);
      if (h == 0.0) continue;
      const double* u = &U[(size_t)k * rows];
      const double* v = &V[(size_t)k * cols];
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
          // W = U S V^T: (i, j) of M is W(i, j), or W(j, i) when transposed
          A[(size_t)i * n + j] += h * (tr ? u[j] * v[i] : u[i] * v[j]);
        }
    }
  }
};

// ---------------------------------------------------------------------------------------------
// D o tau and J_raw (Alg. 1 Step 1; readings Z2, Z15, Z16): bilinear value and the exact
// derivative of the bilinear interpolant from the same 4 taps, chained through the transform.
// ---------------------------------------------------------------------------------------------
int warp(const double* img, int Hh, int Ww, const int* box, const double* tau, int kind, Vec& d, Vec& jraw) {
  const int x0 = box[0], y0 = box[1], n = box[2], m = box[3], p = kind == 1 ? 8 : 6;
  const double s = std::max(m, n) / 2.0, cx = x0 + (n - 1) / 2.0, cy = y0 + (m - 1) / 2.0;
  const double h11 = tau[0], h12 = tau[1], h21 = tau[2], h22 = tau[3], h13 = tau[4], h23 = tau[5];
  const double h31 = kind == 1 ? tau[6] : 0.0, h32 = kind == 1 ? tau[7] : 0.0;
  d.assign((size_t)m * n, 0.0);
  jraw.assign((size_t)p * m * n, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      const double du = j - (n - 1) / 2.0, dv = i - (m - 1) / 2.0;
      const double w = 1.0 + (h31 * du + h32 * dv) / s;
      const double xs = cx + (h11 * du + h12 * dv + s * h13) / w;
      const double ys = cy + (h21 * du + h22 * dv + s * h23) / w;
      if (!std::isfinite(xs) || !std::isfinite(ys)) return WINDOW_ESCAPE;
      const double xf = std::floor(xs), yf = std::floor(ys);
      if (xf < 0 || xf + 1 > Ww - 1 || yf < 0 || yf + 1 > Hh - 1) return WINDOW_ESCAPE;
      const double fx = xs - xf, fy = ys - yf;
      const long xi = (long)xf, yi = (long)yf;
      const double i00 = img[yi * Ww + xi], i01 = img[yi * Ww + xi + 1];
      const double i10 = img[(yi + 1) * Ww + xi], i11 = img[(yi + 1) * Ww + xi + 1];
      const size_t o = (size_t)i * n + j;
      d[o] = (1 - fy) * ((1 - fx) * i00 + fx * i01) + fy * ((1 - fx) * i10 + fx * i11);
      const double dX = (1 - fy) * (i01 - i00) + fy * (i11 - i10);
      const double dY = (1 - fx) * (i10 - i00) + fx * (i11 - i01);
      const double u = du / s, v = dv / s, xn = (xs - cx) / s, yn = (ys - cy) / s;
      const double ix = s * dX, iy = s * dY;
      const size_t mn = (size_t)m * n;
      jraw[0 * mn + o] = ix * u / w;
      jraw[1 * mn + o] = ix * v / w;
      jraw[2 * mn + o] = iy * u / w;
      jraw[3 * mn + o] = iy * v / w;
      jraw[4 * mn + o] = ix / w;
      jraw[5 * mn + o] = iy / w;
      if (kind == 1) {
        jraw[6 * mn + o] = -(ix * xn + iy * yn) * u / w;
        jraw[7 * mn + o] = -(ix * xn + iy * yn) * v / w;
      }
    }
  return CONVERGED;
}

// Q (l = 3 rows): centre x, centre y and the shoelace area of tau(window corners), unit rows
// (reading Z10)
void constraints_q(const double* tau, int kind, int m, int n, double* q /* [3][p] */) {
  const int p = kind == 1 ? 8 : 6;
  const double h11 = tau[0], h12 = tau[1], h21 = tau[2], h22 = tau[3], h13 = tau[4], h23 = tau[5];
  const double h31 = kind == 1 ? tau[6] : 0.0, h32 = kind == 1 ? tau[7] : 0.0;
  const double big = std::max(m, n), cu = n / big, cv = m / big;
  const double cs[4][2] = {{-cu, -cv}, {cu, -cv}, {cu, cv}, {-cu, cv}};
  double px[4], py[4], gx[4][8], gy[4][8];
  for (int k = 0; k < 4; ++k) {
    const double u = cs[k][0], v = cs[k][1];
    const double w = h31 * u + h32 * v + 1.0;
    px[k] = (h11 * u + h12 * v + h13) / w;
    py[k] = (h21 * u + h22 * v + h23) / w;
    for (int e = 0; e < 8; ++e) gx[k][e] = gy[k][e] = 0.0;
    gx[k][0] = u / w; gx[k][1] = v / w; gx[k][4] = 1.0 / w;
    gy[k][2] = u / w; gy[k][3] = v / w; gy[k][5] = 1.0 / w;
    if (kind == 1) {
      gx[k][6] = -px[k] * u / w; gx[k][7] = -px[k] * v / w;
      gy[k][6] = -py[k] * u / w; gy[k][7] = -py[k] * v / w;
    }
  }
  double ga[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < 4; ++k) {
    const int l = (k + 1) % 4;
    for (int e = 0; e < p; ++e) ga[e] += 0.5 * (gx[k][e] * py[l] + px[k] * gy[l][e] - gx[l][e] * py[k] - px[l] * gy[k][e]);
  }
  double nga = 0.0;
  for (int e = 0; e < p; ++e) nga += ga[e] * ga[e];
  nga = std::sqrt(nga);
  for (int r = 0; r < 3; ++r)
    for (int e = 0; e < p; ++e) q[r * p + e] = 0.0;
  q[0 * p + 4] = 1.0;
  q[1 * p + 5] = 1.0;
  for (int e = 0; e < p; ++e) q[2 * p + e] = ga[e] / nga;
}

// W^T W v = v - J (J^T J + Q^T Q)^{-1} J^T v (Eq. Jperpv) by one Cholesky of
// the p x p Gram; delta_tau(r) = G^{-1} J^T r (Eq. Delta_tau, stacked least squares P:671-684)
struct Projector {
  int p = 0, mn = 0;
  const Vec* J = nullptr;  // [p][mn]
  double L[64];            // Cholesky factor (row-major lower)
  bool init(const Vec& j, int p_, int mn_, const double* q, int l) {
    J = &j;
    p = p_;
    mn = mn_;
    double G[64];
    for (int a = 0; a < p; ++a)
      for (int b = 0; b < p; ++b) {
        double s = 0.0;
        for (int o = 0; o < mn; ++o) s += j[(size_t)a * mn + o] * j[(size_t)b * mn + o];
        for (int r = 0; r < l; ++r) s += q[r * p + a] * q[r * p + b];
        G[a * 8 + b] = s;
      }
    for (int a = 0; a < p; ++a) {
      for (int b = 0; b <= a; ++b) {
        double s = G[a * 8 + b];
        for (int k = 0; k < b; ++k) s -= L[a * 8 + k] * L[b * 8 + k];
        if (a == b) {
          if (!(s > 0.0) || !std::isfinite(s)) return false;
          L[a * 8 + a] = std::sqrt(s);
        } else {
          L[a * 8 + b] = s / L[b * 8 + b];
        }
      }
    }
    return true;
  }
  void gsolve(const double* rhs, double* x) const {  // G x = rhs
    double y[8];
    for (int a = 0; a < p; ++a) {
      double s = rhs[a];
      for (int k = 0; k < a; ++k) s -= L[a * 8 + k] * y[k];
      y[a] = s / L[a * 8 + a];
    }
    for (int a = p - 1; a >= 0; --a) {
      double s = y[a];
      for (int k = a + 1; k < p; ++k) s -= L[k * 8 + a] * x[k];
      x[a] = s / L[a * 8 + a];
    }
  }
  void jt(const Vec& v, double* s) const {
    for (int a = 0; a < p; ++a) {
      double acc = 0.0;
      for (int o = 0; o < mn; ++o) acc += (*J)[(size_t)a * mn + o] * v[o];
      s[a] = acc;
    }
  }
  Vec apply(const Vec& v) const {
    double s[8], x[8];
    jt(v, s);
    gsolve(s, x);
    Vec out(v);
    for (int a = 0; a < p; ++a)
      for (int o = 0; o < mn; ++o) out[o] -= (*J)[(size_t)a * mn + o] * x[a];
    return out;
  }
  void delta_tau(const Vec& r, double* dt) const {
    double s[8];
    jt(r, s);
    gsolve(s, dt);
  }
};

struct InnerRes {
  int iters = 0;
  double mu = 0.0, crit1 = NAN, crit2 = NAN;
  Vec sigma_m;
};

// LADMAP (P:437-468 Eqs. A, E, Y, mu, rho; Cond1/2 P:489-497; Eq. newvars2 P:731-737 with errata
// E1: + dual step, E2: N_k from E_k); R reused for the next M
InnerRes ladmap(const Vec& dh, const Projector& proj, int m, int n, double lam, double mu0, double mu_max,
                const tilt_oracle_params& P, Vec& A, Vec& E, Vec& Y, Svt& svt) {
  const size_t mn = (size_t)m * n;
  InnerRes o;
  double denom = fro(proj.apply(dh));
  if (denom == 0.0) denom = 1.0;
  Vec v(mn);
  for (size_t i = 0; i < mn; ++i) v[i] = A[i] + E[i] - dh[i];
  Vec r = proj.apply(v);
  double mu = mu0;
  const int n_iter = P.fixed_inner > 0 ? P.fixed_inner : P.max_inner;
  Vec M(mn), A1, Nk(mn), E1(mn);
  for (int k = 0; k < n_iter; ++k) {
    for (size_t i = 0; i < mn; ++i) M[i] = A[i] - Y[i] / mu - r[i];
    svt(M, m, n, 1.0 / mu, A1, o.sigma_m);
    for (size_t i = 0; i < mn; ++i) v[i] = A1[i] + E[i] - dh[i];
    const Vec pa = proj.apply(v);
    for (size_t i = 0; i < mn; ++i) {
      Nk[i] = E[i] - Y[i] / mu - pa[i];
      E1[i] = shrink(Nk[i], lam / mu);
    }
    for (size_t i = 0; i < mn; ++i) v[i] = A1[i] + E1[i] - dh[i];
    r = proj.apply(v);
    double dA = 0.0, dE = 0.0, rr = 0.0;
    for (size_t i = 0; i < mn; ++i) {
      Y[i] += mu * r[i];
      rr += r[i] * r[i];
      dA += (A1[i] - A[i]) * (A1[i] - A[i]);
      dE += (E1[i] - E[i]) * (E1[i] - E[i]);
    }
    o.crit1 = std::sqrt(rr) / denom;
    o.crit2 = mu * std::sqrt(std::max(dA, dE)) / denom;
    A.swap(A1);
    E = E1;
    const bool rho_bit = o.crit2 < P.eps2;
    o.iters = k + 1;
    o.mu = mu;
    if (o.crit1 < P.eps1 && o.crit2 < P.eps2 && P.fixed_inner <= 0) return o;
    mu = std::min(mu_max, (rho_bit ? P.rho0 : 1.0) * mu);
  }
  return o;
}

// Algorithm 1 for one window
void tilt_one(const double* img, int Hh, int Ww, const int* box, const double* tau0, int kind,
              const tilt_oracle_params& P, double* tau_out, double* A_out, double* E_out, tilt_oracle_report* rep) {
  const int n = box[2], m = box[3], p = kind == 1 ? 8 : 6;
  const size_t mn = (size_t)m * n;
  const double lam = P.lambda > 0 ? P.lambda : 1.0 / std::sqrt((double)std::max(m, n));
  double tau[8] = {1, 0, 0, 1, 0, 0, 0, 0};
  if (tau0)
    for (int e = 0; e < p; ++e) tau[e] = tau0[e];
  Vec A, E, Y, d, jraw, dh, j;
  bool have = false, have_fprev = false;
  double f_prev = 0.0, f = NAN, nd = NAN, dtau_inf = NAN;
  int status = MAX_OUTER, stop_rule = STOP_NONE, inner = 0, outer = 0, sweeps = 0;
  InnerRes res;
  bool have_res = false;
  Svt svt;
  const int n_outer = P.fixed_outer > 0 ? P.fixed_outer : P.max_outer;
  for (int it = 0; it < n_outer; ++it) {
    const int st = warp(img, Hh, Ww, box, tau, kind, d, jraw);
    if (st != CONVERGED) {
      status = st;
      break;
    }
    nd = fro(d);
    if (nd == 0.0) {
      status = ZERO_PATCH;
      break;
    }
    // normalise (Step 1): D_hat = d/||d||, J = (J_raw - D_hat c^T)/||d||, c = D_hat^T J_raw
    dh.resize(mn);
    for (size_t o = 0; o < mn; ++o) dh[o] = d[o] / nd;
    j.assign((size_t)p * mn, 0.0);
    for (int a = 0; a < p; ++a) {
      double c = 0.0;
      for (size_t o = 0; o < mn; ++o) c += jraw[a * mn + o] * dh[o];
      for (size_t o = 0; o < mn; ++o) j[a * mn + o] = (jraw[a * mn + o] - c * dh[o]) / nd;
    }
    double q[24];
    const int l = P.constraints ? 3 : 0;
    if (l) constraints_q(tau, kind, m, n, q);
    Projector proj;
    if (!proj.init(j, p, (int)mn, q, l)) {
      status = SINGULAR_GRAM;
      break;
    }
    // mu0 = mu0_scale / sigma_1(D_hat) (Z3), every inner loop (Z5)
    Vec sv, dummyA;
    Svt s1;
    s1(dh, m, n, 0.0, dummyA, sv);
    const double mu0 = P.mu0_scale / sv[0];
    if (!have || !P.vws) {  // A_0 = D_hat, E_0 = Y_0 = 0 (Z4)
      A = dh;
      E.assign(mn, 0.0);
      Y.assign(mn, 0.0);
    } else {
      Y = proj.apply(Y);  // Y_0 = W^T W Y (Eq. Y_new_warmstart)
    }
    have = true;
    res = ladmap(dh, proj, m, n, lam, mu0, P.mu_max_ratio * mu0, P, A, E, Y, svt);
    have_res = true;
    inner += res.iters;
    // Step 3: dtau = G^{-1} J^T (A + E - D_hat); Step 4: tau += dtau
    Vec rr(mn);
    for (size_t o = 0; o < mn; ++o) rr[o] = A[o] + E[o] - dh[o];
    double dt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    proj.delta_tau(rr, dt);
    dtau_inf = 0.0;
    bool finite = true;
    for (int e = 0; e < p; ++e) {
      tau[e] += dt[e];
      dtau_inf = std::max(dtau_inf, std::fabs(dt[e]));
      finite = finite && std::isfinite(tau[e]);
    }
    double nuc = 0.0, l1 = 0.0;
    for (double s : res.sigma_m) nuc += shrink(s, 1.0 / res.mu);
    for (size_t o = 0; o < mn; ++o) l1 += std::fabs(E[o]);
    f = nuc + lam * l1;
    outer = it + 1;
    if (!std::isfinite(f) || f > 1e12 || !finite) {
      status = DIVERGED;
      break;
    }
    int rule = STOP_NONE;  // reading Z9
    if (have_fprev && std::fabs(f - f_prev) < P.obj_tol * std::fabs(f_prev)) rule = STOP_OBJECTIVE;
    else if (dtau_inf < P.tau_tol) rule = STOP_DTAU;
    f_prev = f;
    have_fprev = true;
    if (rule != STOP_NONE) {
      status = CONVERGED;
      stop_rule = rule;
      if (P.fixed_outer <= 0) break;
    } else {
      status = MAX_OUTER;
      stop_rule = STOP_MAX_OUTER;
    }
  }
  sweeps = svt.sweeps;
  for (int e = 0; e < p; ++e) tau_out[e] = tau[e];
  if (A_out)
    for (size_t o = 0; o < mn; ++o) A_out[o] = have ? A[o] : 0.0;
  if (E_out)
    for (size_t o = 0; o < mn; ++o) E_out[o] = have ? E[o] : 0.0;
  if (rep) {
    tilt_oracle_report r;
    std::memset(&r, 0, sizeof(r));
    r.status = status;
    r.stop_rule = stop_rule;
    r.outer_iters = outer;
    r.inner_iters = inner;
    r.jacobi_sweeps = sweeps;
    r.objective = f;
    r.crit1 = have_res ? res.crit1 : NAN;
    r.crit2 = have_res ? res.crit2 : NAN;
    r.patch_norm = nd;
    // reading Z19: relative rank of sigma(A) = T_{1/mu}(sigma(M_K)), band [3e-4, 3e-3]
    if (have_res) {
      Vec sa;
      for (double s : res.sigma_m) sa.push_back(shrink(s, 1.0 / res.mu));
      std::sort(sa.begin(), sa.end(), std::greater<double>());
      if (!sa.empty() && sa[0] > 0.0)
        for (double s : sa) {
          const double ratio = s / sa[0];
          r.rank += ratio > 1e-3;
          r.rank_band |= (ratio >= 3e-4 && ratio <= 3e-3);
        }
    }
    *rep = r;
  }
}

}  // namespace

extern "C" {

void tilt_oracle_default_params(tilt_oracle_params* p) {
  p->lambda = -1.0;
  p->mu0_scale = 1.25;
  p->mu_max_ratio = 1e6;
  p->rho0 = 2.0;
  p->eps1 = 1e-6;
  p->eps2 = 0.1;
  p->obj_tol = 1e-5;
  p->tau_tol = 1e-4;
  p->max_inner = 1000;
  p->max_outer = 50;
  p->constraints = 1;
  p->vws = 1;
  p->fixed_inner = 0;
  p->fixed_outer = 0;
}

int32_t tilt_oracle_solve_batch(const double* images, int32_t n_images, int32_t H, int32_t W,
                                const int32_t* patch_image, const int32_t* boxes, const double* tau0, int32_t B,
                                int32_t kind, const tilt_oracle_params* prm, double* tau_out, double* A_out,
                                double* E_out, tilt_oracle_report* rep, int32_t n_threads) {
  if (B < 0 || (B > 0 && (!images || !patch_image || !boxes || !tau_out || !prm))) return 1;
  if (kind != 0 && kind != 1) return 1;
  if (B == 0) return 0;
  const int n = boxes[2], m = boxes[3], p = kind == 1 ? 8 : 6;
  if (m < 2 || n < 2 || n_images < 1 || H < 2 || W < 2) return 1;
  for (int b = 0; b < B; ++b)
    if (boxes[4 * b + 2] != n || boxes[4 * b + 3] != m || patch_image[b] < 0 || patch_image[b] >= n_images) return 1;
  const size_t mn = (size_t)m * n;
#ifdef _OPENMP
  const int nt = n_threads > 0 ? n_threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
#endif
  for (int b = 0; b < B; ++b)
    tilt_one(images + (size_t)patch_image[b] * H * W, H, W, boxes + 4 * b, tau0 ? tau0 + (size_t)b * p : nullptr,
             kind, *prm, tau_out + (size_t)b * p, A_out ? A_out + b * mn : nullptr, E_out ? E_out + b * mn : nullptr,
             rep ? rep + b : nullptr);
  return 0;
}

int32_t tilt_oracle_svt(const double* M, int32_t m, int32_t n, double eps, double* A, double* sigma) {
  Vec Mv(M, M + (size_t)m * n), Av, sv;
  Svt svt;
  svt(Mv, m, n, eps, Av, sv);
  std::memcpy(A, Av.data(), Av.size() * sizeof(double));
  if (sigma) std::memcpy(sigma, sv.data(), sv.size() * sizeof(double));
  return svt.sweeps;
}

}  // extern "C"
