/* pvro.c — fp64 CPU ORACLE for the PVR super-resolution iteration.
 *
 * TEST INFRASTRUCTURE ONLY (see pvro.h): loaded by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs; never by the product.
 *
 * Plain, slow, obviously-correct loops in fp64, in the order of SURVEY.md §8(c)
 * (steps 0-11) and DESIGN.md §Readings. Every function cites the PAPER.md passage
 * (P:line) it restates. No blocking, no factorisation of the PSF, no reordering:
 * the forward model is a direct sum over (pixel, PSF sample, trilinear corner).
 * OpenMP runs patches in parallel; the adjoint accumulates with atomic adds.
 */
#include "pvro.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PVRO_MAX_STACKS 64
#define PVRO_MAX_PSF 20000

typedef struct {
  int W, H, K;
  double* y;          /* [K][H][W] */
  double G[12];       /* index -> world, row-major 3x4 */
  double theta;       /* slice thickness (through-plane FWHM) */
  /* PSF lattice (built at extract time, step 0) */
  double u[3], v[3], w[3];  /* in-plane unit axes and slice normal */
  double h[3];              /* lattice steps h_u, h_v, h_w (mm) */
  int S;
  int32_t* abc;             /* [S][3] */
  double* psi;              /* [S] */
  double dx, dy, sw;        /* pixel pitches, slice-profile sigma (volume-space PSF, mode 2) */
} ostack;

struct pvro_ctx {
  int n[3];
  double s, o[3];
  int n_stacks;
  ostack st[PVRO_MAX_STACKS];
  /* patches */
  int64_t M, P;
  int32_t* patch;    /* [M][7] stack, x0, y0, z0, sx, sy, sz */
  int64_t* pix0;     /* [M+1] first pixel of each patch */
  double* T;         /* [M][12] */
  int state;         /* 0 created, 1 stacks, 2 patched, 3 ready */
  /* parameters */
  double delta, tau_patch, c0, tau_live, tau_C, tau_obs, clamp, psf_mode, s2floor, nsigma;
  double lazy;       /* test-only: set_transforms skips the coverage pass (forward_range use) */
  double quality;    /* PSF lattice density factor q (1; 2 = f4 quality mode) */
  double em_rounds, em_tol;  /* f4 multi-round EM (1 round; 1e-6) */
  double patch_mixture;      /* f4 two-Gaussian patch classification (0) */
  uint8_t* mask;             /* f3: per-pixel patch mask [P] (NULL = all pixels) */
  /* iteration state */
  double* X;         /* [V] */
  double *p, *e, *kappa, *yhat;  /* [P] */
  double *pbar, *wpatch;         /* [M] */
  double *A, *C;                 /* [V] */
  double sigma2, c, m, lo, hi, s2min;
  int64_t t;
};

/* ------------------------------------------------------------------ */
/* Step 0: Taylor-series sinc: sinc(x) = 1 - x^2/3! + x^4/5! - ...
 * Reading Q4: cut the series once the next term is below an ABSOLUTE bound 1e-16
 * (the paper's "relative error" is undefined at the zero x = pi).               */
double pvro_sinc_taylor(double x) {
  double term = 1.0, sum = 1.0, x2 = x * x;
  for (int n = 0; n < 200; ++n) {
    double next = -term * x2 / ((2.0 * n + 2.0) * (2.0 * n + 3.0));
    if (fabs(next) < 1e-16) break;
    sum += next;
    term = next;
  }
  return sum;
}

static int lattice_count(double pitch, double s, double q) {
  /* Reading Q5: lattice step <= the HR voxel size / q, at least 2 steps per pitch
   * (q = 1 default; q = 2 the f4 quality mode). */
  int n = (int)ceil(q * pitch / s - 1e-9);
  return n < 2 ? 2 : n;
}

/* Step 0: PSF lattice ("sinc function for the in-plane and the slice
 * profile for the through-plane"). Readings Q1 (radial sinc(pi R)), Q2 (main
 * lobe R < 1), Q3 (Gaussian slice profile, FWHM = thickness, cut at nsigma),
 * Q5 (lattice discretisation). psi is normalised to sum 1.                     */
int pvro_psf_table(double dx, double dy, double theta, double s, double nsigma, int cap,
                   int32_t* abc, double* psi, double* hw_out) {
  return pvro_psf_table_q(dx, dy, theta, s, nsigma, 1.0, cap, abc, psi, hw_out);
}

int pvro_psf_table_q(double dx, double dy, double theta, double s, double nsigma, double q, int cap,
                     int32_t* abc, double* psi, double* hw_out) {
  if (!(dx > 0) || !(dy > 0) || !(theta > 0) || !(s > 0) || !(q >= 1)) return -1;
  int nu = lattice_count(dx, s, q), nv = lattice_count(dy, s, q), nw = lattice_count(theta, s, q);
  double hu = dx / nu, hv = dy / nv, hw = theta / nw;
  double sigw = theta / (2.0 * sqrt(2.0 * log(2.0)));
  int S = 0;
  double total = 0.0;
  for (int c = -1000; c <= 1000; ++c) {
    if (fabs(c * hw) > nsigma * sigw) continue;
    for (int b = -nv; b <= nv; ++b) {
      for (int a = -nu; a <= nu; ++a) {
        double R = sqrt((double)a * a / ((double)nu * nu) + (double)b * b / ((double)nv * nv));
        if (!(R < 1.0)) continue;
        if (S >= cap) return -2;
        double val = pvro_sinc_taylor(M_PI * R) * exp(-(c * hw) * (c * hw) / (2.0 * sigw * sigw));
        abc[3 * S + 0] = a;
        abc[3 * S + 1] = b;
        abc[3 * S + 2] = c;
        psi[S] = val;
        total += val;
        ++S;
      }
    }
  }
  for (int q = 0; q < S; ++q) psi[q] /= total;
  if (hw_out) {
    hw_out[0] = nu; hw_out[1] = nv; hw_out[2] = nw;
    hw_out[3] = hu; hw_out[4] = hv; hw_out[5] = hw; hw_out[6] = sigw;
  }
  return S;
}

/* Square patch windows along one axis ("size a and stride omega");
 * reading Q22: a last window is clamped to the edge so every pixel is covered. */
int pvro_windows(int dim, int size, int stride, int cap, int32_t* out) {
  if (size < 1 || size > dim || stride < 1 || stride > size) return -1;
  int n = 0, x = 0;
  for (; x + size <= dim; x += stride) {
    if (n >= cap) return -2;
    out[n++] = x;
  }
  if (out[n - 1] + size < dim) {
    if (n >= cap) return -2;
    out[n++] = dim - size;
  }
  return n;
}

/* P:202 p = G c / (G c + m (1 - c)), G = N(e; 0, sigma^2), evaluated in the
 * algebraically identical logistic form p = 1 / (1 + exp(z)),
 * z = ln(m (1-c) / c) + e^2 / (2 sigma^2) + 0.5 ln(2 pi sigma^2).              */
double pvro_posterior(double e, double sigma2, double c, double m) {
  if (c >= 1.0 || m <= 0.0) return 1.0;
  if (c <= 0.0) return 0.0;
  double z = log(m * (1.0 - c) / c) + e * e / (2.0 * sigma2) + 0.5 * log(2.0 * M_PI * sigma2);
  return 1.0 / (1.0 + exp(z));
}

/* One M-step + E-step (reading Q10/Q11). */
int pvro_em_round(int64_t n, const double* e, const uint8_t* live, const double* p_prev,
                  int64_t t, double c0, double sigma2_min, double* p_out, double* sigma2_out,
                  double* c_out, double* m_out) {
  double s_pe2 = 0.0, s_p = 0.0, emax = -INFINITY, emin = INFINITY;
  int64_t nl = 0;
  for (int64_t j = 0; j < n; ++j) {
    if (!live[j]) continue;
    s_pe2 += p_prev[j] * e[j] * e[j];
    s_p += p_prev[j];
    if (e[j] > emax) emax = e[j];
    if (e[j] < emin) emin = e[j];
    ++nl;
  }
  double sigma2 = s_p > 0.0 ? s_pe2 / s_p : 0.0;
  if (sigma2 < sigma2_min) sigma2 = sigma2_min;
  double c = (t <= 1) ? c0 : (nl > 0 ? s_p / (double)nl : c0);
  double spread = emax - emin;
  int degenerate = (nl == 0) || !(spread > sqrt(sigma2_min));
  double m = degenerate ? 0.0 : 1.0 / spread;  /* P:193 m = 1 / (max(e) - min(e)) */
  for (int64_t j = 0; j < n; ++j)
    p_out[j] = degenerate ? 1.0 : pvro_posterior(e[j], sigma2, c, m);
  if (sigma2_out) *sigma2_out = sigma2;
  if (c_out) *c_out = c;
  if (m_out) *m_out = m;
  return degenerate;
}

double pvro_em_loglik(int64_t n, const double* e, const uint8_t* live, double sigma2, double c, double m) {
  double ll = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    if (!live[j]) continue;
    const double G = exp(-e[j] * e[j] / (2.0 * sigma2)) / sqrt(2.0 * M_PI * sigma2);
    ll += log(c * G + (1.0 - c) * m);
  }
  return ll;
}

int pvro_em_rounds(int64_t n, const double* e, const uint8_t* live, const double* p_prev, int64_t t,
                   double c0, double sigma2_min, int rounds, double tol, double* p_out,
                   double* sigma2_out, double* c_out, double* m_out, double* ll_out) {
  double sigma2, c, m;
  const int degenerate = pvro_em_round(n, e, live, p_prev, t, c0, sigma2_min, p_out, &sigma2, &c, &m);
  double ll = degenerate ? NAN : pvro_em_loglik(n, e, live, sigma2, c, m), ll_prev = NAN;
  if (ll_out) ll_out[0] = ll;
  int r = 1;
  int64_t nl = 0;
  for (int64_t j = 0; j < n; ++j) nl += live[j] != 0;
  while (!degenerate && r < rounds && nl > 0) {
    if (r >= 2 && ll - ll_prev < tol * fabs(ll_prev)) break;
    double s_pe2 = 0.0, s_p = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (!live[j]) continue;
      s_pe2 += p_out[j] * e[j] * e[j];
      s_p += p_out[j];
    }
    sigma2 = s_p > 0.0 ? s_pe2 / s_p : 0.0;
    if (sigma2 < sigma2_min) sigma2 = sigma2_min;
    c = s_p / (double)nl;
    for (int64_t j = 0; j < n; ++j) p_out[j] = pvro_posterior(e[j], sigma2, c, m);
    ll_prev = ll;
    ll = pvro_em_loglik(n, e, live, sigma2, c, m);
    if (ll_out) ll_out[r] = ll;
    ++r;
  }
  if (sigma2_out) *sigma2_out = sigma2;
  if (c_out) *c_out = c;
  if (m_out) *m_out = m;
  return r;
}

static double gauss_pdf(double x, double mu, double s2) {
  return exp(-(x - mu) * (x - mu) / (2.0 * s2)) / sqrt(2.0 * M_PI * s2);
}

int pvro_patch_mixture(int64_t M, const double* pbar, const uint8_t* valid, int rounds, double tol,
                       double* r_out) {
  double n = 0.0, s1 = 0.0, s2 = 0.0, mx = -INFINITY, mn = INFINITY;
  for (int64_t s = 0; s < M; ++s) {
    r_out[s] = 0.0;
    if (!valid[s]) continue;
    n += 1.0;
    s1 += pbar[s];
    s2 += pbar[s] * pbar[s];
    if (pbar[s] > mx) mx = pbar[s];
    if (pbar[s] < mn) mn = pbar[s];
  }
  if (n <= 0.0) return 0;
  if (!(mx - mn > 1e-6)) {
    for (int64_t s = 0; s < M; ++s) r_out[s] = valid[s] ? 1.0 : 0.0;
    return 0;
  }
  double var = s2 / n - (s1 / n) * (s1 / n);
  if (var < 1e-6) var = 1e-6;
  double mu_in = mx, mu_out = mn, v_in = var, v_out = var, pi = 0.5, ll_prev = NAN;
  int r = 0;
  for (; r < rounds; ++r) {
    /* E-step with the current parameters, and the log-likelihood of those parameters */
    double sr = 0.0, srp = 0.0, srp2 = 0.0, so = 0.0, sop = 0.0, sop2 = 0.0, ll = 0.0;
    for (int64_t s = 0; s < M; ++s) {
      if (!valid[s]) continue;
      const double a = pi * gauss_pdf(pbar[s], mu_in, v_in), b = (1.0 - pi) * gauss_pdf(pbar[s], mu_out, v_out);
      const double rs = (a + b > 0.0) ? a / (a + b) : (pbar[s] >= 0.5 * (mu_in + mu_out) ? 1.0 : 0.0);
      r_out[s] = rs;
      ll += log(a + b > 0.0 ? a + b : 1e-300);
      sr += rs; srp += rs * pbar[s]; srp2 += rs * pbar[s] * pbar[s];
      so += 1.0 - rs; sop += (1.0 - rs) * pbar[s]; sop2 += (1.0 - rs) * pbar[s] * pbar[s];
    }
    if (r >= 1 && ll - ll_prev < tol * fabs(ll_prev)) { ++r; break; }
    ll_prev = ll;
    /* M-step */
    pi = sr / n;
    if (sr > 0.0) { mu_in = srp / sr; v_in = srp2 / sr - mu_in * mu_in; }
    if (so > 0.0) { mu_out = sop / so; v_out = sop2 / so - mu_out * mu_out; }
    if (v_in < 1e-6) v_in = 1e-6;
    if (v_out < 1e-6) v_out = 1e-6;
    if (pi <= 0.0 || pi >= 1.0) { ++r; break; }
  }
  return r;
}

/* P:207 pbar = sqrt((sum p^2) / N), N = number of (live) pixels of the patch. */
double pvro_patch_score(int64_t n, const double* p, const uint8_t* live) {
  double s = 0.0;
  int64_t N = 0;
  for (int64_t j = 0; j < n; ++j) {
    if (!live[j]) continue;
    s += p[j] * p[j];
    ++N;
  }
  return N > 0 ? sqrt(s / (double)N) : 0.0;
}

/* ------------------------------------------------------------------ */
/* Steps 9-10: SR update and edge-preserving regularisation.                  */
static const int D13[13][3] = {{1, 0, -1}, {0, 1, -1}, {1, 1, -1}, {1, -1, -1}, {1, 0, 0},
                               {0, 1, 0},  {1, 1, 0},  {1, -1, 0}, {1, 0, 1},   {0, 1, 1},
                               {1, 1, 1},  {1, -1, 1}, {0, 0, 1}};

int pvro_update_regularise(int nx, int ny, int nz, const double* X0, const double* A,
                           const double* C, double alpha, double lambda, double delta,
                           double tau_C, int clamp, double lo, double hi, double* X1,
                           double* X2) {
  int64_t V = (int64_t)nx * ny * nz;
  /* step 9: X1 = clip(X0 + alpha A / C) where C > tau_C, else X0 */
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < V; ++k) {
    if (C[k] > tau_C) {
      double x = X0[k] + alpha * A[k] / C[k];
      if (clamp) x = x < lo ? lo : (x > hi ? hi : x);
      X1[k] = x;
    } else {
      X1[k] = X0[k];
    }
  }
  /* step 10: X2_k = X1_k + alpha lambda sum_d [b_d(k)(X1_{k+d} - X1_k)
   *                                               + b_d(k-d)(X1_{k-d} - X1_k)],
   * b_d(k) = phi_d / sqrt(1 + phi_d ((X0_{k+d} - X0_k) / delta)^2), phi_d = 1/|d|_1,
   * b_d(k) = 0 unless k and k+d are both in the grid and both have C > tau_C.  */
#pragma omp parallel for schedule(static)
  for (int l = 0; l < nz; ++l) {
    for (int j = 0; j < ny; ++j) {
      for (int i = 0; i < nx; ++i) {
        int64_t k = ((int64_t)l * ny + j) * nx + i;
        if (!(C[k] > tau_C)) {
          X2[k] = X1[k];
          continue;
        }
        double sum = 0.0;
        for (int d = 0; d < 13; ++d) {
          double phi = 1.0 / (abs(D13[d][0]) + abs(D13[d][1]) + abs(D13[d][2]));
          for (int sgn = -1; sgn <= 1; sgn += 2) {
            int i2 = i + sgn * D13[d][0], j2 = j + sgn * D13[d][1], l2 = l + sgn * D13[d][2];
            if (i2 < 0 || i2 >= nx || j2 < 0 || j2 >= ny || l2 < 0 || l2 >= nz) continue;
            int64_t k2 = ((int64_t)l2 * ny + j2) * nx + i2;
            if (!(C[k2] > tau_C)) continue;
            /* b_d(k) for sgn = +1 uses (X0_{k+d} - X0_k); b_d(k-d) for sgn = -1 uses
               (X0_k - X0_{k-d}); both square the same neighbour difference. */
            double g = (X0[k2] - X0[k]) / delta;
            double b = phi / sqrt(1.0 + phi * g * g);
            sum += b * (X1[k2] - X1[k]);
          }
        }
        X2[k] = X1[k] + alpha * lambda * sum;
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* Problem-level API                                                           */
pvro_ctx* pvro_create(const int32_t dims[3], double spacing, const double origin[3]) {
  if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || !(spacing > 0)) return NULL;
  pvro_ctx* x = (pvro_ctx*)calloc(1, sizeof(pvro_ctx));
  for (int d = 0; d < 3; ++d) { x->n[d] = dims[d]; x->o[d] = origin[d]; }
  x->s = spacing;
  /* thresholds (reading Q24 / Q25): tau_C = 1e-6 (SURVEY.md:678); observed iff kappa > 0
     (SURVEY.md:652) with a 1e-2 floor against 1/kappa amplification of pixels >= 99% outside */
  x->delta = 150.0; x->tau_patch = 0.5; x->c0 = 0.9; x->tau_live = 0.99; x->tau_C = 1e-6;
  x->tau_obs = 0.01; x->clamp = 1; x->psf_mode = 0; x->s2floor = 1e-6; x->nsigma = 3.0; x->quality = 1.0;
  x->em_rounds = 1.0; x->em_tol = 1e-6; x->patch_mixture = 0.0;
  int64_t V = (int64_t)dims[0] * dims[1] * dims[2];
  x->X = (double*)calloc(V, sizeof(double));
  x->A = (double*)calloc(V, sizeof(double));
  x->C = (double*)calloc(V, sizeof(double));
  return x;
}

void pvro_destroy(pvro_ctx* x) {
  if (!x) return;
  for (int i = 0; i < x->n_stacks; ++i) { free(x->st[i].y); free(x->st[i].abc); free(x->st[i].psi); }
  free(x->patch); free(x->pix0); free(x->T); free(x->X); free(x->A); free(x->C);
  free(x->p); free(x->e); free(x->kappa); free(x->yhat); free(x->pbar); free(x->wpatch); free(x->mask);
  free(x);
}

int pvro_set_param(pvro_ctx* x, int key, double v) {
  switch (key) {
    case PVRO_DELTA: x->delta = v; break;
    case PVRO_TAU_PATCH: x->tau_patch = v; break;
    case PVRO_C0: x->c0 = v; break;
    case PVRO_TAU_LIVE: x->tau_live = v; break;
    case PVRO_TAU_C: x->tau_C = v; break;
    case PVRO_TAU_OBS: x->tau_obs = v; break;
    case PVRO_CLAMP: x->clamp = v; break;
    case PVRO_PSF_MODE: x->psf_mode = v; break;
    case PVRO_SIGMA2_FLOOR: x->s2floor = v; break;
    case PVRO_PSF_NSIGMA: x->nsigma = v; break;
    case PVRO_LAZY: x->lazy = v; break;
    case PVRO_PSF_QUALITY: x->quality = v; break;
    case PVRO_EM_ROUNDS: x->em_rounds = v; break;
    case PVRO_EM_TOL: x->em_tol = v; break;
    case PVRO_PATCH_MIXTURE: x->patch_mixture = v; break;
    default: return -1;
  }
  return 0;
}

static double norm3(const double* a) { return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

static int add_stack_impl(pvro_ctx* x, const float* sf, const double* sd, int W, int H, int K,
                          const double G[12], double thickness) {
  if (x->state > 1 || x->n_stacks >= PVRO_MAX_STACKS) return -1;
  if (W < 1 || H < 1 || K < 1 || !(thickness > 0)) return -1;
  ostack* st = &x->st[x->n_stacks];
  memset(st, 0, sizeof(*st));
  st->W = W; st->H = H; st->K = K; st->theta = thickness;
  memcpy(st->G, G, sizeof(st->G));
  int64_t L = (int64_t)W * H * K;
  st->y = (double*)malloc(L * sizeof(double));
  for (int64_t i = 0; i < L; ++i) st->y[i] = sf ? (double)sf[i] : sd[i];
  x->n_stacks++;
  x->state = 1;
  return x->n_stacks - 1;
}

int pvro_add_stack(pvro_ctx* x, const float* slices, int W, int H, int K, const double G[12],
                   double thickness) {
  return add_stack_impl(x, slices, NULL, W, H, K, G, thickness);
}

int pvro_add_stack_f64(pvro_ctx* x, const double* slices, int W, int H, int K, const double G[12],
                       double thickness) {
  return add_stack_impl(x, NULL, slices, W, H, K, G, thickness);
}

/* Stack frame: u = G[:,0]/dx, v = G[:,1]/dy, w = u x v (normalised) and its PSF. */
static int build_psf(pvro_ctx* x, ostack* st) {
  double c0[3] = {st->G[0], st->G[4], st->G[8]}, c1[3] = {st->G[1], st->G[5], st->G[9]};
  double dx = norm3(c0), dy = norm3(c1);
  if (!(dx > 0) || !(dy > 0)) return -1;
  for (int d = 0; d < 3; ++d) { st->u[d] = c0[d] / dx; st->v[d] = c1[d] / dy; }
  st->w[0] = st->u[1] * st->v[2] - st->u[2] * st->v[1];
  st->w[1] = st->u[2] * st->v[0] - st->u[0] * st->v[2];
  st->w[2] = st->u[0] * st->v[1] - st->u[1] * st->v[0];
  double nw = norm3(st->w);
  if (!(nw > 1e-12)) return -1;
  for (int d = 0; d < 3; ++d) st->w[d] /= nw;
  st->abc = (int32_t*)malloc(3 * PVRO_MAX_PSF * sizeof(int32_t));
  st->psi = (double*)malloc(PVRO_MAX_PSF * sizeof(double));
  st->dx = dx;
  st->dy = dy;
  st->sw = st->theta / (2.0 * sqrt(2.0 * log(2.0)));
  if (x->psf_mode == 2) { /* volume-space PSF (reading Q34): no patch-space lattice */
    st->S = 1;
    st->abc[0] = st->abc[1] = st->abc[2] = 0;
    st->psi[0] = 1.0;
    st->h[0] = st->h[1] = st->h[2] = 0.0;
    return 0;
  }
  if (x->psf_mode == 1) { /* test-only delta PSF: one sample at the pixel centre */
    st->S = 1;
    st->abc[0] = st->abc[1] = st->abc[2] = 0;
    st->psi[0] = 1.0;
    st->h[0] = st->h[1] = st->h[2] = 0.0;
    return 0;
  }
  double hw[7];
  st->S = pvro_psf_table_q(dx, dy, st->theta, x->s, x->nsigma, x->quality, PVRO_MAX_PSF, st->abc, st->psi, hw);
  st->h[0] = hw[3]; st->h[1] = hw[4]; st->h[2] = hw[5];
  return st->S > 0 ? 0 : -1;
}

static int64_t install_patches(pvro_ctx* x, int64_t M);

/* f3 multi-scale schedule: a context that has patches may extract new ones; the
 * patch table and per-pixel state are dropped, the stacks and X stay (set_transforms again). */
static void drop_patches(pvro_ctx* x) {
  if (x->state < 2) return;
  free(x->patch); free(x->pix0); free(x->T);
  free(x->p); free(x->e); free(x->kappa); free(x->yhat); free(x->pbar); free(x->wpatch); free(x->mask);
  x->patch = NULL; x->pix0 = NULL; x->T = NULL; x->p = x->e = x->kappa = x->yhat = NULL;
  x->pbar = x->wpatch = NULL; x->mask = NULL;
  for (int i = 0; i < x->n_stacks; ++i) { free(x->st[i].abc); free(x->st[i].psi); x->st[i].abc = NULL; x->st[i].psi = NULL; }
  x->M = x->P = 0;
  x->state = 1;
}

/* f3 (Eq. 3; reading Q32): an explicit patch table instead of
 * the square windows: rects [n][7] = (stack, x0, y0, z0, sx, sy, sz) inside their stacks, and
 * an optional per-pixel mask [sum sx sy sz] (patch-major; NULL = all pixels). Masked-out
 * pixels are never observations: their coverage kappa is 0 (so e = 0, p = 0, no splat). */
int64_t pvro_set_patches(pvro_ctx* x, int64_t n, const int32_t* rects, const uint8_t* mask) {
  if (x->state < 1 || n <= 0) return -1;
  for (int64_t s = 0; s < n; ++s) {
    const int32_t* r = &rects[7 * s];
    if (r[0] < 0 || r[0] >= x->n_stacks) return -1;
    const ostack* st = &x->st[r[0]];
    if (r[4] < 1 || r[5] < 1 || r[6] < 1 || r[1] < 0 || r[2] < 0 || r[3] < 0 || r[1] + r[4] > st->W ||
        r[2] + r[5] > st->H || r[3] + r[6] > st->K)
      return -1;
  }
  drop_patches(x);
  for (int i = 0; i < x->n_stacks; ++i)
    if (build_psf(x, &x->st[i]) != 0) return -1;
  x->patch = (int32_t*)malloc(7 * n * sizeof(int32_t));
  memcpy(x->patch, rects, 7 * n * sizeof(int32_t));
  const int64_t M = install_patches(x, n);
  if (mask) {
    x->mask = (uint8_t*)malloc(x->P);
    memcpy(x->mask, mask, x->P);
  }
  return M;
}

/* ---- f3 superpixels (reading Q33) ---- */
static int slic_quant(float y, float ymin, float ymax) {
  if (!(ymax > ymin)) return 0;
  const double t = ((double)y - (double)ymin) * 1023.0 / ((double)ymax - (double)ymin);
  return (int)floor(t + 0.5);
}

int pvro_slic(int W, int H, const float* img, float ymin, float ymax, int S, int m, int iters, int32_t* labels) {
  if (W < 1 || H < 1 || S < 2 || m < 1 || iters < 0) return -1;
  const int nxc = (W + S - 1) / S, nyc = (H + S - 1) / S, nc = nxc * nyc;
  int64_t* cx = (int64_t*)malloc(nc * sizeof(int64_t));
  int64_t* cy = (int64_t*)malloc(nc * sizeof(int64_t));
  int64_t* cI = (int64_t*)malloc(nc * sizeof(int64_t));
  int64_t* acc = (int64_t*)malloc(4 * nc * sizeof(int64_t));
  for (int j = 0; j < nyc; ++j)
    for (int i = 0; i < nxc; ++i) {
      const int k = j * nxc + i;
      const int px = i * S + S / 2 < W - 1 ? i * S + S / 2 : W - 1;
      const int py = j * S + S / 2 < H - 1 ? j * S + S / 2 : H - 1;
      cx[k] = 16 * (int64_t)px;
      cy[k] = 16 * (int64_t)py;
      cI[k] = 16 * (int64_t)slic_quant(img[(int64_t)py * W + px], ymin, ymax);
    }
  const int64_t S2 = (int64_t)S * S, m2 = (int64_t)m * m;
  for (int round = 0; round <= iters; ++round) {
    /* assignment */
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const int64_t I16 = 16 * (int64_t)slic_quant(img[(int64_t)y * W + x], ymin, ymax);
        const int ci = x / S, cj = y / S;
        int64_t best = INT64_MAX;
        int bk = -1;
        for (int dj = -1; dj <= 1; ++dj)
          for (int di = -1; di <= 1; ++di) {
            const int i = ci + di, j = cj + dj;
            if (i < 0 || i >= nxc || j < 0 || j >= nyc) continue;
            const int k = j * nxc + i;
            const int64_t dI = I16 - cI[k], dx = 16 * (int64_t)x - cx[k], dy = 16 * (int64_t)y - cy[k];
            const int64_t D = S2 * dI * dI + m2 * (dx * dx + dy * dy);
            if (D < best) { best = D; bk = k; }
          }
        labels[(int64_t)y * W + x] = bk;
      }
    if (round == iters) break;
    /* update */
    memset(acc, 0, 4 * nc * sizeof(int64_t));
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const int k = labels[(int64_t)y * W + x];
        acc[4 * k] += 1;
        acc[4 * k + 1] += x;
        acc[4 * k + 2] += y;
        acc[4 * k + 3] += slic_quant(img[(int64_t)y * W + x], ymin, ymax);
      }
    for (int k = 0; k < nc; ++k) {
      const int64_t n = acc[4 * k];
      if (n == 0) continue;
      cx[k] = (16 * acc[4 * k + 1] + n / 2) / n;
      cy[k] = (16 * acc[4 * k + 2] + n / 2) / n;
      cI[k] = (16 * acc[4 * k + 3] + n / 2) / n;
    }
  }
  free(cx); free(cy); free(cI); free(acc);
  return nc;
}

int64_t pvro_superpixel_patches(pvro_ctx* x, int S, int m, int iters, int gamma) {
  if (x->state < 1 || S < 2 || m < 1 || iters < 0 || gamma < 0) return -1;
  /* pass 0 counts (rects, pixels); pass 1 fills */
  int64_t nrect = 0, npix = 0;
  int32_t* rects = NULL;
  uint8_t* mask = NULL;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t r = 0, q = 0;
    for (int si = 0; si < x->n_stacks; ++si) {
      const ostack* st = &x->st[si];
      const int64_t HW = (int64_t)st->W * st->H;
      float ymin = INFINITY, ymax = -INFINITY;
      for (int64_t t = 0; t < HW * st->K; ++t) {
        const float v = (float)st->y[t];
        if (v < ymin) ymin = v;
        if (v > ymax) ymax = v;
      }
      float* img = (float*)malloc(HW * sizeof(float));
      int32_t* lab = (int32_t*)malloc(HW * sizeof(int32_t));
      for (int z = 0; z < st->K; ++z) {
        for (int64_t t = 0; t < HW; ++t) img[t] = (float)st->y[z * HW + t];
        const int nc = pvro_slic(st->W, st->H, img, ymin, ymax, S, m, iters, lab);
        for (int k = 0; k < nc; ++k) {
          int xmin = st->W, xmax = -1, ymn = st->H, ymx = -1;
          for (int yy = 0; yy < st->H; ++yy)
            for (int xx = 0; xx < st->W; ++xx)
              if (lab[(int64_t)yy * st->W + xx] == k) {
                if (xx < xmin) xmin = xx;
                if (xx > xmax) xmax = xx;
                if (yy < ymn) ymn = yy;
                if (yy > ymx) ymx = yy;
              }
          if (xmax < 0) continue;
          const int x0 = xmin - gamma > 0 ? xmin - gamma : 0, x1 = xmax + gamma < st->W - 1 ? xmax + gamma : st->W - 1;
          const int y0 = ymn - gamma > 0 ? ymn - gamma : 0, y1 = ymx + gamma < st->H - 1 ? ymx + gamma : st->H - 1;
          const int sx = x1 - x0 + 1, sy = y1 - y0 + 1;
          if (pass == 1) {
            int32_t* rr = &rects[7 * r];
            rr[0] = si; rr[1] = x0; rr[2] = y0; rr[3] = z; rr[4] = sx; rr[5] = sy; rr[6] = 1;
            for (int v = 0; v < sy; ++v)
              for (int u = 0; u < sx; ++u) {
                int hit = 0;
                for (int dv = -gamma; dv <= gamma && !hit; ++dv)
                  for (int du = -gamma; du <= gamma && !hit; ++du) {
                    const int xx = x0 + u + du, yy = y0 + v + dv;
                    if (xx >= 0 && xx < st->W && yy >= 0 && yy < st->H && lab[(int64_t)yy * st->W + xx] == k) hit = 1;
                  }
                mask[q + (int64_t)v * sx + u] = (uint8_t)hit;
              }
          }
          ++r;
          q += (int64_t)sx * sy;
        }
      }
      free(img);
      free(lab);
    }
    if (pass == 0) {
      nrect = r;
      npix = q;
      if (nrect == 0) return -1;
      rects = (int32_t*)malloc(7 * nrect * sizeof(int32_t));
      mask = (uint8_t*)malloc(npix);
    }
  }
  const int64_t M = pvro_set_patches(x, nrect, rects, mask);
  free(rects);
  free(mask);
  return M;
}

int64_t pvro_extract_patches(pvro_ctx* x, int size, int stride, int depth, int stride_z) {
  if (x->state < 1) return -1;
  drop_patches(x);
  for (int i = 0; i < x->n_stacks; ++i)
    if (build_psf(x, &x->st[i]) != 0) return -1;
  int64_t M = 0;
  int32_t *xs = (int32_t*)malloc(65536 * 4), *ys = (int32_t*)malloc(65536 * 4),
          *zs = (int32_t*)malloc(65536 * 4);
  for (int pass = 0; pass < 2; ++pass) {
    M = 0;
    for (int i = 0; i < x->n_stacks; ++i) {
      ostack* st = &x->st[i];
      int nxw = pvro_windows(st->W, size, stride, 65536, xs);
      int nyw = pvro_windows(st->H, size, stride, 65536, ys);
      int nzw = pvro_windows(st->K, depth, stride_z, 65536, zs);
      if (nxw < 0 || nyw < 0 || nzw < 0) { free(xs); free(ys); free(zs); return -1; }
      for (int a = 0; a < nzw; ++a)
        for (int b = 0; b < nyw; ++b)
          for (int c = 0; c < nxw; ++c) {
            if (pass == 1) {
              int32_t* pt = &x->patch[7 * M];
              pt[0] = i; pt[1] = xs[c]; pt[2] = ys[b]; pt[3] = zs[a];
              pt[4] = size; pt[5] = size; pt[6] = depth;
            }
            ++M;
          }
    }
    if (pass == 0) x->patch = (int32_t*)malloc(7 * (M > 0 ? M : 1) * sizeof(int32_t));
  }
  free(xs); free(ys); free(zs);
  return install_patches(x, M);
}

/* Patch table installed (x->patch holds M rows): pixel offsets and the per-pixel state. */
static int64_t install_patches(pvro_ctx* x, int64_t M) {
  x->M = M;
  x->pix0 = (int64_t*)malloc((M + 1) * sizeof(int64_t));
  x->pix0[0] = 0;
  for (int64_t s = 0; s < M; ++s)
    x->pix0[s + 1] = x->pix0[s] + (int64_t)x->patch[7 * s + 4] * x->patch[7 * s + 5] * x->patch[7 * s + 6];
  x->P = x->pix0[M];
  x->p = (double*)calloc(x->P, sizeof(double));
  x->e = (double*)calloc(x->P, sizeof(double));
  x->kappa = (double*)calloc(x->P, sizeof(double));
  x->yhat = (double*)calloc(x->P, sizeof(double));
  x->pbar = (double*)calloc(M, sizeof(double));
  x->wpatch = (double*)calloc(M, sizeof(double));
  x->T = (double*)calloc(12 * M, sizeof(double));
  x->state = 2;
  return M;
}

int64_t pvro_num_pixels(const pvro_ctx* x) { return x->P; }

int pvro_get_mask(const pvro_ctx* x, uint8_t* out) {
  if (x->state < 2) return -1;
  if (x->mask) memcpy(out, x->mask, x->P);
  else memset(out, 1, x->P);
  return 0;
}

int pvro_get_patches(const pvro_ctx* x, int32_t* out) {
  if (x->state < 2) return -1;
  memcpy(out, x->patch, 7 * x->M * sizeof(int32_t));
  return 0;
}

int pvro_get_psf(const pvro_ctx* x, int stack, int cap, int32_t* abc, double* psi) {
  if (x->state < 2 || stack < 0 || stack >= x->n_stacks) return -1;
  const ostack* st = &x->st[stack];
  if (cap < st->S) return -2;
  memcpy(abc, st->abc, 3 * st->S * sizeof(int32_t));
  memcpy(psi, st->psi, st->S * sizeof(double));
  return st->S;
}

/* Pixel j's observed value (stack view, not a copy). */
static double pixel_y(const pvro_ctx* x, const int32_t* pt, int u, int v, int z) {
  const ostack* st = &x->st[pt[0]];
  return st->y[((int64_t)(pt[3] + z) * st->H + (pt[2] + v)) * st->W + (pt[1] + u)];
}

/* Step 1: sample position x_jq = g(T_s(c_j + delta_q)) in continuous voxel index,
 * c_j = G (x0+u, y0+v, z0+z, 1), g(w) = (w - o) / s.                          */
static void sample_pos(const pvro_ctx* x, const int32_t* pt, const double* T, int u, int v,
                       int z, int q, double out[3]) {
  const ostack* st = &x->st[pt[0]];
  double col = pt[1] + u, row = pt[2] + v, sl = pt[3] + z;
  const int32_t* abc = &st->abc[3 * q];
  double c[3];
  for (int d = 0; d < 3; ++d)
    c[d] = st->G[4 * d + 0] * col + st->G[4 * d + 1] * row + st->G[4 * d + 2] * sl + st->G[4 * d + 3] +
           abc[0] * st->h[0] * st->u[d] + abc[1] * st->h[1] * st->v[d] + abc[2] * st->h[2] * st->w[d];
  for (int d = 0; d < 3; ++d) {
    double wd = T[4 * d + 0] * c[0] + T[4 * d + 1] * c[1] + T[4 * d + 2] * c[2] + T[4 * d + 3];
    out[d] = (wd - x->o[d]) / x->s;
  }
}

/* Step 1 (reading Q6): trilinear corners of a continuous index; corners outside
 * [0, n-1] are dropped. Returns the number of in-grid corners written.        */
static int trilinear(const pvro_ctx* x, const double pos[3], int64_t idx[8], double wt[8]) {
  int i0[3];
  double f[3];
  for (int d = 0; d < 3; ++d) {
    double fl = floor(pos[d]);
    i0[d] = (int)fl;
    f[d] = pos[d] - fl;
  }
  int n = 0;
  for (int cz = 0; cz < 2; ++cz)
    for (int cy = 0; cy < 2; ++cy)
      for (int cx = 0; cx < 2; ++cx) {
        int i = i0[0] + cx, j = i0[1] + cy, l = i0[2] + cz;
        if (i < 0 || i >= x->n[0] || j < 0 || j >= x->n[1] || l < 0 || l >= x->n[2]) continue;
        idx[n] = ((int64_t)l * x->n[1] + j) * x->n[0] + i;
        wt[n] = (cx ? f[0] : 1.0 - f[0]) * (cy ? f[1] : 1.0 - f[1]) * (cz ? f[2] : 1.0 - f[2]);
        ++n;
      }
  return n;
}

int pvro_set_transforms(pvro_ctx* x, const double* T, int64_t n) {
  if (x->state < 2) return -1;
  if (n != x->M) return -2;
  memcpy(x->T, T, 12 * n * sizeof(double));
  x->state = 3;
  if (x->lazy != 0.0) return 0; /* test-only: no coverage / EM reset (forward_range only) */
  /* coverage kappa (step 2) is geometry only: one forward pass on any volume */
  pvro_forward(x, x->X, x->yhat, x->kappa);
  /* EM reset: p_prev = 1, t = 0; live-y range for sigma2_min and the clamp (Q19) */
  double ymin = INFINITY, ymax = -INFINITY;
  for (int64_t s = 0; s < x->M; ++s) {
    const int32_t* pt = &x->patch[7 * s];
    int64_t j = x->pix0[s];
    for (int z = 0; z < pt[6]; ++z)
      for (int v = 0; v < pt[5]; ++v)
        for (int u = 0; u < pt[4]; ++u, ++j) {
          x->p[j] = 1.0;
          if (x->kappa[j] >= x->tau_live) {
            double yv = pixel_y(x, pt, u, v, z);
            if (yv < ymin) ymin = yv;
            if (yv > ymax) ymax = yv;
          }
        }
  }
  if (!(ymax >= ymin)) { ymin = 0.0; ymax = 0.0; }
  x->lo = ymin - 0.1 * fabs(ymin);
  x->hi = ymax + 0.1 * fabs(ymax);
  x->s2min = x->s2floor * (ymax - ymin) * (ymax - ymin);
  x->t = 0;
  for (int64_t s = 0; s < x->M; ++s) { x->pbar[s] = 1.0; x->wpatch[s] = 1.0; }
  return 0;
}

int pvro_set_volume(pvro_ctx* x, const double* X) {
  memcpy(x->X, X, (size_t)x->n[0] * x->n[1] * x->n[2] * sizeof(double));
  return 0;
}

int pvro_get_volume(const pvro_ctx* x, double* X) {
  memcpy(X, x->X, (size_t)x->n[0] * x->n[1] * x->n[2] * sizeof(double));
  return 0;
}

/* Steps 2-3 (Eq. 1): kappa_j = sum_q psi_q sum_{k in grid} t_k(x_jq);
 * observed iff kappa_j >= tau_obs; yhat_j = sum_k W_jk X_k,
 * W_jk = kappa_j^-1 sum_q psi_q t_k(x_jq) (each observed row sums to 1).      */
int pvro_forward(const pvro_ctx* x, const double* X, double* yhat, double* kappa) {
  return pvro_forward_range(x, X, 0, x->M, yhat, kappa);
}

/* ---- volume-space PSF (psf_mode 2; "fully flexible and accurate PSF", reading Q34) ----
 * The PSF of pixel j is evaluated at every HR voxel centre x_k: with delta = T_s^-1(x_k) - c_j
 * and its components (a, b, c) along the slice frame (u, v, w) in mm,
 *   psi(a, b, c) = sinc(pi R) exp(-c^2 / (2 sw^2)),  R = |(a / dx, b / dy)| < 1, |c| <= nsigma sw,
 * (sinc by the Taylor series of P:160, readings Q1-Q3); kappa_j = sum_{k in grid} psi /
 * sum_{k in Z^3} psi and W_jk = psi_jk / sum_{k in grid} psi. The voxels visited are those of the
 * index box holding the support's image under T_s. */
static double volpsf_weight(const ostack* st, double nsigma, const double d[3]) {
  double a = 0.0, b = 0.0, c = 0.0;
  for (int e = 0; e < 3; ++e) {
    a += st->u[e] * d[e];
    b += st->v[e] * d[e];
    c += st->w[e] * d[e];
  }
  double R = sqrt((a / st->dx) * (a / st->dx) + (b / st->dy) * (b / st->dy));
  if (!(R < 1.0) || fabs(c) > nsigma * st->sw) return 0.0;
  return pvro_sinc_taylor(M_PI * R) * exp(-c * c / (2.0 * st->sw * st->sw));
}

/* Pixel (u, v, z) of patch s: its world centre c_j, the inverse linear map of T_s, and the
 * voxel index box of its support. */
static void volpsf_pixel(const pvro_ctx* x, int64_t s, int u, int v, int z, double cw[3], double Ainv[9],
                         int lo[3], int hi[3], double nsigma) {
  const int32_t* pt = &x->patch[7 * s];
  const ostack* st = &x->st[pt[0]];
  const double* T = &x->T[12 * s];
  double col = pt[1] + u, row = pt[2] + v, sl = pt[3] + z;
  for (int d = 0; d < 3; ++d)
    cw[d] = st->G[4 * d] * col + st->G[4 * d + 1] * row + st->G[4 * d + 2] * sl + st->G[4 * d + 3];
  /* inverse of the 3x3 linear part of T (cofactors) */
  const double m00 = T[0], m01 = T[1], m02 = T[2], m10 = T[4], m11 = T[5], m12 = T[6], m20 = T[8], m21 = T[9],
               m22 = T[10];
  const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) + m02 * (m10 * m21 - m11 * m20);
  Ainv[0] = (m11 * m22 - m12 * m21) / det; Ainv[1] = (m02 * m21 - m01 * m22) / det; Ainv[2] = (m01 * m12 - m02 * m11) / det;
  Ainv[3] = (m12 * m20 - m10 * m22) / det; Ainv[4] = (m00 * m22 - m02 * m20) / det; Ainv[5] = (m02 * m10 - m00 * m12) / det;
  Ainv[6] = (m10 * m21 - m11 * m20) / det; Ainv[7] = (m01 * m20 - m00 * m21) / det; Ainv[8] = (m00 * m11 - m01 * m10) / det;
  /* support box corners (a, b, c) = (+-dx, +-dy, +-nsigma sw) mapped through T */
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int ia = -1; ia <= 1; ia += 2)
    for (int ib = -1; ib <= 1; ib += 2)
      for (int ic = -1; ic <= 1; ic += 2) {
        double p[3], q[3];
        for (int d = 0; d < 3; ++d)
          p[d] = cw[d] + ia * st->dx * st->u[d] + ib * st->dy * st->v[d] + ic * nsigma * st->sw * st->w[d];
        for (int d = 0; d < 3; ++d) q[d] = (T[4 * d] * p[0] + T[4 * d + 1] * p[1] + T[4 * d + 2] * p[2] + T[4 * d + 3] - x->o[d]) / x->s;
        for (int d = 0; d < 3; ++d) { if (q[d] < mn[d]) mn[d] = q[d]; if (q[d] > mx[d]) mx[d] = q[d]; }
      }
  for (int d = 0; d < 3; ++d) { lo[d] = (int)ceil(mn[d] - 1e-9); hi[d] = (int)floor(mx[d] + 1e-9); }
}

/* delta = T^-1(x_k) - c_j = Ainv (x_k - T(c_j)) */
static void volpsf_delta(const pvro_ctx* x, const double* T, const double cw[3], const double Ainv[9], int i, int j,
                         int l, double d[3]) {
  double tc[3], r[3];
  for (int e = 0; e < 3; ++e) tc[e] = T[4 * e] * cw[0] + T[4 * e + 1] * cw[1] + T[4 * e + 2] * cw[2] + T[4 * e + 3];
  const int k3[3] = {i, j, l};
  for (int e = 0; e < 3; ++e) r[e] = x->o[e] + x->s * k3[e] - tc[e];
  for (int e = 0; e < 3; ++e) d[e] = Ainv[3 * e] * r[0] + Ainv[3 * e + 1] * r[1] + Ainv[3 * e + 2] * r[2];
}

static int in_grid(const pvro_ctx* x, int i, int j, int l) {
  return i >= 0 && i < x->n[0] && j >= 0 && j < x->n[1] && l >= 0 && l < x->n[2];
}

static void volpsf_forward_patch(const pvro_ctx* x, const double* X, int64_t s, double* yhat, double* kappa) {
  const int32_t* pt = &x->patch[7 * s];
  const ostack* st = &x->st[pt[0]];
  const double* T = &x->T[12 * s];
  int64_t jj = x->pix0[s];
  for (int z = 0; z < pt[6]; ++z)
    for (int v = 0; v < pt[5]; ++v)
      for (int u = 0; u < pt[4]; ++u, ++jj) {
        double cw[3], Ainv[9], d[3];
        int lo[3], hi[3];
        volpsf_pixel(x, s, u, v, z, cw, Ainv, lo, hi, x->nsigma);
        double all = 0.0, in = 0.0, acc = 0.0;
        for (int l = lo[2]; l <= hi[2]; ++l)
          for (int j = lo[1]; j <= hi[1]; ++j)
            for (int i = lo[0]; i <= hi[0]; ++i) {
              volpsf_delta(x, T, cw, Ainv, i, j, l, d);
              const double w = volpsf_weight(st, x->nsigma, d);
              if (w == 0.0) continue;
              all += w;
              if (!in_grid(x, i, j, l)) continue;
              in += w;
              acc += w * X[((int64_t)l * x->n[1] + j) * x->n[0] + i];
            }
        double kap = all > 0.0 ? in / all : 0.0;
        if (x->mask && !x->mask[jj]) kap = 0.0;
        kappa[jj] = kap;
        yhat[jj] = (kap >= x->tau_obs) ? acc / in : 0.0;
      }
}

static void volpsf_adjoint_patch(const pvro_ctx* x, const double* r, int64_t s, double* out) {
  const int32_t* pt = &x->patch[7 * s];
  const ostack* st = &x->st[pt[0]];
  const double* T = &x->T[12 * s];
  int64_t jj = x->pix0[s];
  for (int z = 0; z < pt[6]; ++z)
    for (int v = 0; v < pt[5]; ++v)
      for (int u = 0; u < pt[4]; ++u, ++jj) {
        if (!(x->kappa[jj] >= x->tau_obs) || r[jj] == 0.0) continue;
        double cw[3], Ainv[9], d[3];
        int lo[3], hi[3];
        volpsf_pixel(x, s, u, v, z, cw, Ainv, lo, hi, x->nsigma);
        double in = 0.0;  /* row normaliser: sum of psi over the in-grid voxels */
        for (int l = lo[2]; l <= hi[2]; ++l)
          for (int j = lo[1]; j <= hi[1]; ++j)
            for (int i = lo[0]; i <= hi[0]; ++i) {
              if (!in_grid(x, i, j, l)) continue;
              volpsf_delta(x, T, cw, Ainv, i, j, l, d);
              in += volpsf_weight(st, x->nsigma, d);
            }
        for (int l = lo[2]; l <= hi[2]; ++l)
          for (int j = lo[1]; j <= hi[1]; ++j)
            for (int i = lo[0]; i <= hi[0]; ++i) {
              if (!in_grid(x, i, j, l)) continue;
              volpsf_delta(x, T, cw, Ainv, i, j, l, d);
              const double w = volpsf_weight(st, x->nsigma, d);
              if (w == 0.0) continue;
              const double add = w / in * r[jj];
#pragma omp atomic
              out[((int64_t)l * x->n[1] + j) * x->n[0] + i] += add;
            }
      }
}

/* Steps 2-3 for the pixels of one patch s (yhat, kappa indexed by global pixel). */
static void forward_patch(const pvro_ctx* x, const double* X, int64_t s, double* yhat, double* kappa) {
  if (x->psf_mode == 2) {
    volpsf_forward_patch(x, X, s, yhat, kappa);
    return;
  }
  const int32_t* pt = &x->patch[7 * s];
  const ostack* st = &x->st[pt[0]];
  const double* T = &x->T[12 * s];
  int64_t j = x->pix0[s];
  for (int z = 0; z < pt[6]; ++z)
    for (int v = 0; v < pt[5]; ++v)
      for (int u = 0; u < pt[4]; ++u, ++j) {
        double kap = 0.0, acc = 0.0;
        for (int q = 0; q < st->S; ++q) {
          double pos[3], wt[8];
          int64_t idx[8];
          sample_pos(x, pt, T, u, v, z, q, pos);
          int nc = trilinear(x, pos, idx, wt);
          for (int c = 0; c < nc; ++c) {
            kap += st->psi[q] * wt[c];
            acc += st->psi[q] * wt[c] * X[idx[c]];
          }
        }
        if (x->mask && !x->mask[j]) kap = 0.0;  /* f3: masked-out pixel (Q32) */
        kappa[j] = kap;
        yhat[j] = (kap >= x->tau_obs) ? acc / kap : 0.0;
      }
}

/* Forward of patches [first, first+count) only (yhat, kappa indexed by global pixel). */
int pvro_forward_range(const pvro_ctx* x, const double* X, int64_t first, int64_t count,
                       double* yhat, double* kappa) {
  if (x->state < 2 || first < 0 || first + count > x->M) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = first; s < first + count; ++s) forward_patch(x, X, s, yhat, kappa);
  return 0;
}

/* Coverage kappa (step 2) of a list of patches into the context (test hook for full-size
 * checks that never run the whole coverage pass: set_transforms with PVRO_LAZY). */
int pvro_coverage_subset(pvro_ctx* x, const int64_t* patches, int64_t n) {
  if (x->state < 3) return -1;
  for (int64_t i = 0; i < n; ++i)
    if (patches[i] < 0 || patches[i] >= x->M) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < n; ++i) forward_patch(x, x->X, patches[i], x->yhat, x->kappa);
  return 0;
}

/* Adjoint of step 3 for one patch: out_k += sum_j W_jk r_j over its observed pixels. */
static void adjoint_patch(const pvro_ctx* x, const double* r, int64_t s, double* out) {
  if (x->psf_mode == 2) {
    volpsf_adjoint_patch(x, r, s, out);
    return;
  }
  const int32_t* pt = &x->patch[7 * s];
  const ostack* st = &x->st[pt[0]];
  const double* T = &x->T[12 * s];
  int64_t j = x->pix0[s];
  for (int z = 0; z < pt[6]; ++z)
    for (int v = 0; v < pt[5]; ++v)
      for (int u = 0; u < pt[4]; ++u, ++j) {
        if (!(x->kappa[j] >= x->tau_obs) || r[j] == 0.0) continue;
        for (int q = 0; q < st->S; ++q) {
          double pos[3], wt[8];
          int64_t idx[8];
          sample_pos(x, pt, T, u, v, z, q, pos);
          int nc = trilinear(x, pos, idx, wt);
          for (int c = 0; c < nc; ++c) {
            double add = st->psi[q] * wt[c] / x->kappa[j] * r[j];
#pragma omp atomic
            out[idx[c]] += add;
          }
        }
      }
}

/* Adjoint of step 3 (north_star "backprojection"): out_k += sum_j W_jk r_j over the
 * observed pixels of patches [first, first+count). Requires kappa (set_transforms). */
int pvro_adjoint(const pvro_ctx* x, const double* r, int64_t first, int64_t count, double* out) {
  if (x->state < 3 || first < 0 || first + count > x->M) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = first; s < first + count; ++s) adjoint_patch(x, r, s, out);
  return 0;
}

/* The same adjoint over a list of patches. */
int pvro_adjoint_subset(const pvro_ctx* x, const double* r, const int64_t* patches, int64_t n, double* out) {
  if (x->state < 3) return -1;
  for (int64_t i = 0; i < n; ++i)
    if (patches[i] < 0 || patches[i] >= x->M) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < n; ++i) adjoint_patch(x, r, patches[i], out);
  return 0;
}

/* Init (SURVEY §8(c) Init): X = W^T y / W^T 1 where C0 > tau_C, else the mean
 * of the 26-neighbours with C0 > tau_C (one pass), else 0.                      */
int pvro_init_volume(pvro_ctx* x) {
  if (x->state < 3) return -1;
  int64_t V = (int64_t)x->n[0] * x->n[1] * x->n[2];
  double* r = (double*)malloc(x->P * sizeof(double));
  double* ones = (double*)malloc(x->P * sizeof(double));
  for (int64_t s = 0; s < x->M; ++s) {
    const int32_t* pt = &x->patch[7 * s];
    int64_t j = x->pix0[s];
    for (int z = 0; z < pt[6]; ++z)
      for (int v = 0; v < pt[5]; ++v)
        for (int u = 0; u < pt[4]; ++u, ++j) { r[j] = pixel_y(x, pt, u, v, z); ones[j] = 1.0; }
  }
  memset(x->A, 0, V * sizeof(double));
  memset(x->C, 0, V * sizeof(double));
  pvro_adjoint(x, r, 0, x->M, x->A);
  pvro_adjoint(x, ones, 0, x->M, x->C);
  free(r); free(ones);
  int nx = x->n[0], ny = x->n[1], nz = x->n[2];
#pragma omp parallel for schedule(static)
  for (int l = 0; l < nz; ++l)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t k = ((int64_t)l * ny + j) * nx + i;
        if (x->C[k] > x->tau_C) { x->X[k] = x->A[k] / x->C[k]; continue; }
        double sum = 0.0;
        int cnt = 0;
        for (int dl = -1; dl <= 1; ++dl)
          for (int dj = -1; dj <= 1; ++dj)
            for (int di = -1; di <= 1; ++di) {
              if (!di && !dj && !dl) continue;
              int i2 = i + di, j2 = j + dj, l2 = l + dl;
              if (i2 < 0 || i2 >= nx || j2 < 0 || j2 >= ny || l2 < 0 || l2 >= nz) continue;
              int64_t k2 = ((int64_t)l2 * ny + j2) * nx + i2;
              if (x->C[k2] > x->tau_C) { sum += x->A[k2] / x->C[k2]; ++cnt; }
            }
        x->X[k] = cnt ? sum / cnt : 0.0;
      }
  return 0;
}

/* Rigidity map (reading Q28): W^T (p pbar) / W^T 1 where W^T 1 > tau_C, else 0. */
int pvro_rigidity_map(const pvro_ctx* x, double* out) {
  if (x->state < 3) return -1;
  const int64_t V = (int64_t)x->n[0] * x->n[1] * x->n[2];
  double* r = (double*)malloc(x->P * sizeof(double));
  double* ones = (double*)malloc(x->P * sizeof(double));
  double* num = (double*)calloc(V, sizeof(double));
  double* den = (double*)calloc(V, sizeof(double));
  for (int64_t s = 0; s < x->M; ++s) {
    const int32_t* pt = &x->patch[7 * s];
    const int64_t n = (int64_t)pt[4] * pt[5] * pt[6];
    for (int64_t j = x->pix0[s]; j < x->pix0[s] + n; ++j) { r[j] = x->p[j] * x->pbar[s]; ones[j] = 1.0; }
  }
  pvro_adjoint(x, r, 0, x->M, num);
  pvro_adjoint(x, ones, 0, x->M, den);
  for (int64_t k = 0; k < V; ++k) out[k] = den[k] > x->tau_C ? num[k] / den[k] : 0.0;
  free(r); free(ones); free(num); free(den);
  return 0;
}

int pvro_set_weights(pvro_ctx* x, const double* p, const double* pbar) {
  if (x->state < 3) return -1;
  if (p) memcpy(x->p, p, x->P * sizeof(double));
  if (pbar) memcpy(x->pbar, pbar, x->M * sizeof(double));
  return 0;
}

/* ------------------------------------------------------------------ */
/* f1: rigid patch-to-volume registration (reading Q29).   */

double pvro_cc(int64_t n, const double* a, const double* b) {
  if (n < 2) return NAN;
  double ma = 0.0, mb = 0.0;
  for (int64_t i = 0; i < n; ++i) { ma += a[i]; mb += b[i]; }
  ma /= n;
  mb /= n;
  double sab = 0.0, saa = 0.0, sbb = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    sab += (a[i] - ma) * (b[i] - mb);
    saa += (a[i] - ma) * (a[i] - ma);
    sbb += (b[i] - mb) * (b[i] - mb);
  }
  if (!(saa > 0.0) || !(sbb > 0.0)) return NAN;
  return sab / sqrt(saa * sbb);
}

/* Rotation R = Rz(rz) Ry(ry) Rx(rx), angles in degrees (row-major 3x3). */
static void pose_rotation(const double* pose, double R[9]) {
  const double k = M_PI / 180.0;
  const double cx = cos(k * pose[3]), sx = sin(k * pose[3]);
  const double cy = cos(k * pose[4]), sy = sin(k * pose[4]);
  const double cz = cos(k * pose[5]), sz = sin(k * pose[5]);
  const double Rx[9] = {1, 0, 0, 0, cx, -sx, 0, sx, cx};
  const double Ry[9] = {cy, 0, sy, 0, 1, 0, -sy, 0, cy};
  const double Rz[9] = {cz, -sz, 0, sz, cz, 0, 0, 0, 1};
  double Ryx[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      Ryx[3 * i + j] = 0.0;
      for (int t = 0; t < 3; ++t) Ryx[3 * i + j] += Ry[3 * i + t] * Rx[3 * t + j];
    }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      R[3 * i + j] = 0.0;
      for (int t = 0; t < 3; ++t) R[3 * i + j] += Rz[3 * i + t] * Ryx[3 * t + j];
    }
}

/* World position of pixel (u, v, z) of patch s under T_s. */
static void patch_world(const pvro_ctx* x, int64_t s, double u, double v, double z, double out[3]) {
  const int32_t* pt = &x->patch[7 * s];
  const ostack* st = &x->st[pt[0]];
  const double* T = &x->T[12 * s];
  double c[3];
  for (int d = 0; d < 3; ++d)
    c[d] = st->G[4 * d] * (pt[1] + u) + st->G[4 * d + 1] * (pt[2] + v) + st->G[4 * d + 2] * (pt[3] + z) +
           st->G[4 * d + 3];
  for (int d = 0; d < 3; ++d) out[d] = T[4 * d] * c[0] + T[4 * d + 1] * c[1] + T[4 * d + 2] * c[2] + T[4 * d + 3];
}

/* Q29: the pose acts after T_s, rotating about the transformed patch centre. */
static void patch_centre(const pvro_ctx* x, int64_t s, double c[3]) {
  const int32_t* pt = &x->patch[7 * s];
  patch_world(x, s, 0.5 * (pt[4] - 1), 0.5 * (pt[5] - 1), 0.5 * (pt[6] - 1), c);
}

int pvro_compose_pose(const pvro_ctx* x, int64_t s, const double* pose, double* Tn) {
  if (x->state < 3 || s < 0 || s >= x->M) return -1;
  double R[9], c[3];
  pose_rotation(pose, R);
  patch_centre(x, s, c);
  const double* T = &x->T[12 * s];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) {
      Tn[4 * i + j] = 0.0;
      for (int t = 0; t < 3; ++t) Tn[4 * i + j] += R[3 * i + t] * T[4 * t + j];
    }
    double b = 0.0;
    for (int t = 0; t < 3; ++t) b += R[3 * i + t] * (T[4 * t + 3] - c[t]);
    Tn[4 * i + 3] = b + c[i] + pose[i];
  }
  return 0;
}

int pvro_patch_cc(const pvro_ctx* x, const double* Xl, int64_t s, const double* pose, int min_valid,
                  double* cc, int64_t* nvalid) {
  if (x->state < 3 || s < 0 || s >= x->M) return -1;
  const int32_t* pt = &x->patch[7 * s];
  const int64_t np = (int64_t)pt[4] * pt[5] * pt[6];
  double* ys = (double*)malloc(np * sizeof(double));
  double* xs = (double*)malloc(np * sizeof(double));
  double R[9], c[3];
  pose_rotation(pose, R);
  patch_centre(x, s, c);
  int64_t n = 0;
  for (int z = 0; z < pt[6]; ++z)
    for (int v = 0; v < pt[5]; ++v)
      for (int u = 0; u < pt[4]; ++u) {
        double w[3], m[3], g[3];
        patch_world(x, s, u, v, z, w);
        for (int i = 0; i < 3; ++i) {
          m[i] = R[3 * i] * (w[0] - c[0]) + R[3 * i + 1] * (w[1] - c[1]) + R[3 * i + 2] * (w[2] - c[2]) + c[i] +
                 pose[i];
          g[i] = (m[i] - x->o[i]) / x->s;
        }
        int64_t idx[8];
        double wt[8];
        const int nc = trilinear(x, g, idx, wt);
        double val = 0.0;
        for (int k = 0; k < nc; ++k) val += wt[k] * Xl[idx[k]];
        ys[n] = pixel_y(x, pt, u, v, z);
        xs[n] = val;
        ++n;
      }
  *nvalid = n;
  *cc = n >= min_valid ? pvro_cc(n, ys, xs) : NAN;
  free(ys);
  free(xs);
  return 0;
}

/* level L moves by 2^-L x (2 mm, 4 degrees) */

int pvro_register(const pvro_ctx* x, int levels, int iters, int min_valid, double* T_out, int32_t* status,
                  double* pose_out) {
  if (x->state < 3) return -1;
  const double* Xl = x->X;  /* Q29: levels are step sizes on the unblurred reconstruction */
  double* pose = (double*)calloc(6 * x->M, sizeof(double));
  for (int64_t s = 0; s < x->M; ++s) status[s] = 1;
  for (int L = 0; L < levels; ++L) {
    const double step_t = ldexp(2.0, -L), step_r = ldexp(4.0, -L);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t s = 0; s < x->M; ++s) {
      if (!status[s]) continue;
      double* p = &pose[6 * s];
      double cur;
      int64_t nv;
      pvro_patch_cc(x, Xl, s, p, min_valid, &cur, &nv);
      if (isnan(cur)) {
        if (L == 0) status[s] = 0;  /* unregistrable: transform left unchanged */
        continue;
      }
      for (int it = 0; it < iters; ++it) {
        double best = cur, q[6], qb[6];
        int bk = -1;
        for (int k = 0; k < 12; ++k) {
          memcpy(q, p, sizeof(q));
          const double step = (k / 2) < 3 ? step_t : step_r;
          q[k / 2] += (k % 2) ? -step : step;
          double cc;
          pvro_patch_cc(x, Xl, s, q, min_valid, &cc, &nv);
          if (!isnan(cc) && cc > best) { best = cc; bk = k; memcpy(qb, q, sizeof(qb)); }
        }
        if (bk < 0) break;
        memcpy(p, qb, sizeof(qb));
        cur = best;
      }
    }
  }
  for (int64_t s = 0; s < x->M; ++s) {
    if (status[s]) pvro_compose_pose(x, s, &pose[6 * s], &T_out[12 * s]);
    else memcpy(&T_out[12 * s], &x->T[12 * s], 12 * sizeof(double));
    if (pose_out) memcpy(&pose_out[6 * s], &pose[6 * s], 6 * sizeof(double));
  }
  free(pose);
  return 0;
}

/* One SR iteration = SURVEY §8(c) steps 1-11, in order. */
static int sr_step(pvro_ctx* x, double alpha, double lambda) {
  int64_t V = (int64_t)x->n[0] * x->n[1] * x->n[2];
  x->t += 1;
  /* steps 1-4: forward model and residual e = y - yhat on observed pixels */
  pvro_forward(x, x->X, x->yhat, x->kappa);
  uint8_t* live = (uint8_t*)malloc(x->P);
  for (int64_t s = 0; s < x->M; ++s) {
    const int32_t* pt = &x->patch[7 * s];
    int64_t j = x->pix0[s];
    for (int z = 0; z < pt[6]; ++z)
      for (int v = 0; v < pt[5]; ++v)
        for (int u = 0; u < pt[4]; ++u, ++j) {
          int obs = x->kappa[j] >= x->tau_obs;
          x->e[j] = obs ? pixel_y(x, pt, u, v, z) - x->yhat[j] : 0.0;
          live[j] = x->kappa[j] >= x->tau_live;
        }
  }
  /* steps 5-6: M-step (p_prev = p of the previous E-step) then E-step */
  double* pnew = (double*)malloc(x->P * sizeof(double));
  pvro_em_rounds(x->P, x->e, live, x->p, x->t, x->c0, x->s2min, (int)x->em_rounds, x->em_tol, pnew, &x->sigma2,
                 &x->c, &x->m, NULL);
  for (int64_t j = 0; j < x->P; ++j) x->p[j] = (x->kappa[j] >= x->tau_obs) ? pnew[j] : 0.0;
  free(pnew);
  /* step 7: patch score and weight (reading Q13; Q31 with the mixture) */
  uint8_t* pvalid = (uint8_t*)malloc(x->M);
  for (int64_t s = 0; s < x->M; ++s) {
    int64_t j0 = x->pix0[s], n = x->pix0[s + 1] - j0, nl = 0;
    for (int64_t j = j0; j < j0 + n; ++j) nl += live[j] != 0;
    x->pbar[s] = pvro_patch_score(n, &x->p[j0], &live[j0]);
    x->wpatch[s] = x->pbar[s] >= x->tau_patch ? x->pbar[s] : 0.0;
    pvalid[s] = nl > 0;
  }
  if (x->patch_mixture != 0.0) {
    double* r = (double*)malloc(x->M * sizeof(double));
    pvro_patch_mixture(x->M, x->pbar, pvalid, 50, 1e-6, r);
    for (int64_t s = 0; s < x->M; ++s) x->wpatch[s] = r[s] >= 0.5 ? r[s] : 0.0;
    free(r);
  }
  free(pvalid);
  free(live);
  /* step 8: A = W^T (w p e), C = W^T (w p) */
  double* rA = (double*)malloc(x->P * sizeof(double));
  double* rC = (double*)malloc(x->P * sizeof(double));
  for (int64_t s = 0; s < x->M; ++s)
    for (int64_t j = x->pix0[s]; j < x->pix0[s + 1]; ++j) {
      rA[j] = x->wpatch[s] * x->p[j] * x->e[j];
      rC[j] = x->wpatch[s] * x->p[j];
    }
  memset(x->A, 0, V * sizeof(double));
  memset(x->C, 0, V * sizeof(double));
  pvro_adjoint(x, rA, 0, x->M, x->A);
  pvro_adjoint(x, rC, 0, x->M, x->C);
  free(rA); free(rC);
  /* steps 9-11: update, regularise, commit */
  double* X1 = (double*)malloc(V * sizeof(double));
  double* X2 = (double*)malloc(V * sizeof(double));
  pvro_update_regularise(x->n[0], x->n[1], x->n[2], x->X, x->A, x->C, alpha, lambda, x->delta,
                         x->tau_C, x->clamp != 0, x->lo, x->hi, X1, X2);
  memcpy(x->X, X2, V * sizeof(double));
  free(X1); free(X2);
  return 0;
}

int pvro_sr_iterate(pvro_ctx* x, int n, double alpha, double lambda) {
  if (x->state < 3 || n < 0 || alpha < 0 || lambda < 0) return -1;
  for (int i = 0; i < n; ++i) sr_step(x, alpha, lambda);
  return 0;
}

int pvro_get_weights(const pvro_ctx* x, double* p, double* pbar, double* w) {
  if (x->state < 3) return -1;
  if (p) memcpy(p, x->p, x->P * sizeof(double));
  if (pbar) memcpy(pbar, x->pbar, x->M * sizeof(double));
  if (w) memcpy(w, x->wpatch, x->M * sizeof(double));
  return 0;
}

int pvro_get_taps(const pvro_ctx* x, double* e, double* kappa, double* A, double* C) {
  if (x->state < 3) return -1;
  int64_t V = (int64_t)x->n[0] * x->n[1] * x->n[2];
  if (e) memcpy(e, x->e, x->P * sizeof(double));
  if (kappa) memcpy(kappa, x->kappa, x->P * sizeof(double));
  if (A) memcpy(A, x->A, V * sizeof(double));
  if (C) memcpy(C, x->C, V * sizeof(double));
  return 0;
}

int pvro_get_em_state(const pvro_ctx* x, double* sigma2, double* c, double* m, int64_t* t,
                      double* lo, double* hi) {
  if (sigma2) *sigma2 = x->sigma2;
  if (c) *c = x->c;
  if (m) *m = x->m;
  if (t) *t = x->t;
  if (lo) *lo = x->lo;
  if (hi) *hi = x->hi;
  return 0;
}
