/* pvro.h — fp64 CPU ORACLE for the PVR super-resolution iteration.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product
 * (libpvr.so, paper_1611_07289_b200/) never includes, links or calls it, and this
 * tree includes nothing from the product: the two share no code, header, table or
 * constant generator.
 *
 * What it computes: SURVEY.md §8(c) steps 0-11 and the init, written as plain
 * fp64 loops in the paper's order (PAPER.md = /root/reference/PAPER.md):
 *   PSF table ............ P:158-160 (sinc in-plane, slice profile through-plane,
 *                          Taylor-series sinc); readings Q1-Q5 in DESIGN.md
 *   forward model ........ Eq. 1, P:53-58 (x_i = W_i y + n_i, W_i = D B T_i)
 *   residual, EM ......... P:189-209 (m = 1/(max e - min e), p = Gc/(Gc+m(1-c)),
 *                          pbar = sqrt(sum p^2 / N), patch exclusion)
 *   adjoint / SR update .. P:185 ("reintegrated into X using iterative
 *                          super-resolution with gradient descent")
 *   regulariser .......... P:97 (edge-preserving anisotropic diffusion; reading Q17)
 *   init ................. P:89 (empty voxels filled with the mean of neighbours)
 * Parity status per function is listed in DESIGN.md §Oracle; the PSF
 * discretisation (Q1-Q5), regulariser form (Q17) and patch rule (Q13) are
 * "parity unpinned" against the paper (the paper prints no numbers for them) and
 * are pinned only by closed forms / invariants of the readings themselves.
 *
 * Conventions (independent restatement of DESIGN.md §Geometry):
 *   volume voxel (i,j,l) -> world o + s*(i,j,l); data index (l*ny + j)*nx + i.
 *   stack slices float/double [K][H][W]; G: row-major 3x4, world = G*(col,row,slice,1).
 *   patch pixel order: patch-major, then slice z, row v, column u.
 *   T: row-major 3x4 per patch, world -> world; sample = T(c_j + delta_q).
 * All functions return 0 on success, a negative value on error.
 */
#ifndef PVRO_H
#define PVRO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct pvro_ctx pvro_ctx;

/* parameter keys (oracle-side numbering; the product has its own) */
enum {
  PVRO_DELTA = 0,        /* regulariser edge scale delta (default 150)              */
  PVRO_TAU_PATCH = 1,    /* patch inlier threshold on pbar (0.5)                     */
  PVRO_C0 = 2,           /* initial inlier proportion c at t = 1 (0.9)               */
  PVRO_TAU_LIVE = 3,     /* live pixel: kappa >= tau_live (0.99)                     */
  PVRO_TAU_C = 4,        /* voxel updated iff C > tau_C (1e-6)                       */
  PVRO_TAU_OBS = 5,      /* observed pixel: kappa >= tau_obs (0.01)                  */
  PVRO_CLAMP = 6,        /* 1: clamp X1 to [lo, hi] (default 1)                      */
  PVRO_PSF_MODE = 7,     /* 0: PVR PSF; 1: delta PSF (S = 1, delta_q = 0), test only;
                            2: volume-space PSF evaluation (reading Q34)          */
  PVRO_SIGMA2_FLOOR = 9, /* sigma2_min = floor * (ymax - ymin)^2 (1e-6)              */
  PVRO_PSF_NSIGMA = 10,  /* through-plane truncation in sigma_w (3)                  */
  PVRO_LAZY = 12,        /* test-only: set_transforms skips coverage (forward_range)  */
  PVRO_PSF_QUALITY = 13, /* PSF lattice density q: n = max(2, ceil(q pitch / s)) (1)   */
  PVRO_EM_ROUNDS = 14,   /* EM rounds per SR iteration, f4 multi-round EM (1)          */
  PVRO_EM_TOL = 15,      /* stop rounds when the log-likelihood gains < tol |LL| (1e-6) */
  PVRO_PATCH_MIXTURE = 16, /* 1: patch weights from a two-Gaussian mixture on pbar (0)    */
};

/* ---- scalar building blocks (pinned individually by tests/test_oracle_*.py) ---- */
double pvro_sinc_taylor(double x);                       /* sin(x)/x by its Taylor series */
/* PSF lattice of one stack. Writes up to cap entries: abc[3*q] = (a,b,c), psi[q].
   Returns S (number of samples) or <0. hw_out (nullable) = {n_u,n_v,n_w,h_u,h_v,h_w,sigma_w}. */
int pvro_psf_table(double dx, double dy, double theta, double s, double nsigma,
                   int cap, int32_t* abc, double* psi, double* hw_out);
/* Same with the lattice density factor q >= 1 (SURVEY 8(f) f4 "q = 2 PSF quality mode"). */
int pvro_psf_table_q(double dx, double dy, double theta, double s, double nsigma, double q, int cap,
                     int32_t* abc, double* psi, double* hw_out);
/* Square-window extraction along one axis (clamp-last reading Q22).
   Returns the number of windows, writes starts to out (cap entries). */
int pvro_windows(int dim, int size, int stride, int cap, int32_t* out);
/* EM: posterior of one residual (logistic form of P:202). */
double pvro_posterior(double e, double sigma2, double c, double m);
/* One EM round over n residuals: M-step with p_prev (t == 1 uses c = c0), then E-step.
   live[j] != 0 marks pixels in the statistics; p_out gets the posterior for every j.
   Returns 1 if the degenerate (zero-spread / no-live) path was taken, else 0. */
int pvro_em_round(int64_t n, const double* e, const uint8_t* live, const double* p_prev,
                  int64_t t, double c0, double sigma2_min, double* p_out,
                  double* sigma2_out, double* c_out, double* m_out);
/* f4 multi-round EM ("alternates (E) ... with (M) ... until
 * log-likelihood sum log P(e | sigma, c) increases by < 1e-6 or 20 EM rounds"; reading Q30).
 * Round 1 is pvro_em_round. Round r >= 2 (only while not degenerate, and not when round r-1
 * gained less than tol |LL_{r-2}| over round r-2): M-step sigma^2 = max(sum p e^2 / sum p,
 * sigma2_min), c = sum p / N over live pixels from the previous round's p (m = 1 / spread is
 * fixed by e), E-step p = posterior on every pixel. LL_r = sum_live log(c G(e) + (1-c) m).
 * ll_out [rounds] (may be NULL) receives LL_1 .. LL_R' ; returns R' (>= 1), the rounds run. */
int pvro_em_rounds(int64_t n, const double* e, const uint8_t* live, const double* p_prev, int64_t t,
                   double c0, double sigma2_min, int rounds, double tol, double* p_out,
                   double* sigma2_out, double* c_out, double* m_out, double* ll_out);
/* f4 two-Gaussian patch classification ("an inlier and outlier probability for each
 * y_s ... exclude it ... if classified as an outlier"; reading Q31): a 1D mixture
 * pi N(mu_in, s_in^2) + (1 - pi) N(mu_out, s_out^2) over the patch scores pbar of the valid
 * patches (valid[s] != 0: at least one live pixel), fitted by EM from mu_in = max, mu_out = min,
 * s_in^2 = s_out^2 = the scores' variance, pi = 1/2; rounds until the mixture log-likelihood
 * gains < tol |LL| (at most `rounds`); variances floored at 1e-6. r_out [M]: the inlier
 * posterior (0 for invalid patches; 1 for all valid ones when the scores are all equal to
 * 1e-6). Returns the rounds run. */
int pvro_patch_mixture(int64_t M, const double* pbar, const uint8_t* valid, int rounds, double tol,
                       double* r_out);
/* log-likelihood sum_live log(c G_sigma(e) + (1-c) m) of the mixture. */
double pvro_em_loglik(int64_t n, const double* e, const uint8_t* live, double sigma2, double c, double m);
/* pbar = sqrt(sum_{live} p^2 / N_live); 0 if N_live = 0. */
double pvro_patch_score(int64_t n, const double* p, const uint8_t* live);
/* SR update (step 9) + regulariser (step 10) on a bare grid, for the closed-form pins. */
int pvro_update_regularise(int nx, int ny, int nz, const double* X0, const double* A,
                           const double* C, double alpha, double lambda, double delta,
                           double tau_C, int clamp, double lo, double hi, double* X1_out,
                           double* X2_out);

/* ---- problem-level API (mirrors the product's call sequence) ---- */
pvro_ctx* pvro_create(const int32_t dims[3], double spacing, const double origin[3]);
void pvro_destroy(pvro_ctx*);
int pvro_set_param(pvro_ctx*, int key, double value);
int pvro_add_stack(pvro_ctx*, const float* slices, int W, int H, int K,
                   const double G[12], double thickness);
/* fp64 slices, for the exact fixed-point pins (tests only) */
int pvro_add_stack_f64(pvro_ctx*, const double* slices, int W, int H, int K,
                       const double G[12], double thickness);
int64_t pvro_extract_patches(pvro_ctx*, int size, int stride, int depth, int stride_z);
/* f3 superpixels (Eq. 3 P:140-145 "superpixels ... SLIC"; reading Q33): integer
 * SLIC on one slice (W x H floats, row-major) so that every decision is exact on any machine:
 * intensities quantised I = floor(1023 (y - ymin) / (ymax - ymin) + 0.5) (fp64; I = 0 if
 * ymax = ymin); cluster centres on the S-grid (cell (i, j) at min(i S + S/2, W-1),
 * min(j S + S/2, H-1)) in 1/16 units; each pixel picks, among the centres of its own and the 8
 * neighbouring grid cells, the smallest D = S^2 (16 I - cI)^2 + m^2 ((16 x - cx)^2 + (16 y - cy)^2)
 * (int64; ties to the lowest cluster index k = j ceil(W/S) + i); centres move to the rounded
 * means (c = (16 sum + n/2) / n; empty clusters stay); `iters` assign+update rounds, then a final
 * assignment. labels [H][W] = k. Returns the number of clusters ceil(W/S) ceil(H/S). */
int pvro_slic(int W, int H, const float* img, float ymin, float ymax, int S, int m, int iters, int32_t* labels);
/* Superpixel patches of all stacks (reading Q32, Q33): SLIC on every slice (the stack's own
 * intensity range), then per non-empty cluster (stack, slice, k order) the bounding box dilated
 * by gamma pixels (clipped to the slice) and the mask of pixels within Chebyshev distance
 * gamma of the cluster (dilation by a flat structuring element). Installs them as
 * pvro_set_patches does. Returns M or < 0. */
int64_t pvro_superpixel_patches(pvro_ctx*, int S, int m, int iters, int gamma);
/* The per-pixel patch mask [P] (1 everywhere when none was given). */
int pvro_get_mask(const pvro_ctx*, uint8_t* out);
/* f3 (reading Q32): explicit patch table rects [n][7] = (stack, x0, y0, z0,
 * sx, sy, sz) and an optional per-pixel mask (patch-major, NULL = all): masked-out pixels are
 * never observations (kappa = 0). Instead of pvro_extract_patches. Returns M or < 0. */
int64_t pvro_set_patches(pvro_ctx*, int64_t n, const int32_t* rects, const uint8_t* mask);
int64_t pvro_num_pixels(const pvro_ctx*);
/* patch table: 7 int32 per patch {stack, x0, y0, z0, sx, sy, sz} */
int pvro_get_patches(const pvro_ctx*, int32_t* out);
int pvro_get_psf(const pvro_ctx*, int stack, int cap, int32_t* abc, double* psi);
int pvro_set_transforms(pvro_ctx*, const double* T, int64_t n);
int pvro_set_volume(pvro_ctx*, const double* X);
int pvro_get_volume(const pvro_ctx*, double* X);
/* forward operator on an arbitrary volume: yhat[j] (0 if unobserved) and kappa[j] */
int pvro_forward(const pvro_ctx*, const double* X, double* yhat, double* kappa);
int pvro_forward_range(const pvro_ctx*, const double* X, int64_t first, int64_t count,
                       double* yhat, double* kappa);
/* adjoint operator: out[k] = sum_j W_jk r[j] over observed pixels of patches
   [first, first + count) (out is accumulated into, caller zeroes it) */
int pvro_adjoint(const pvro_ctx*, const double* r, int64_t first, int64_t count, double* out);
/* The adjoint over a list of patches (accumulates into out), and the coverage kappa of a list of
 * patches into the context: test hooks for full-size region-of-interest checks. */
int pvro_adjoint_subset(const pvro_ctx*, const double* r, const int64_t* patches, int64_t n, double* out);
int pvro_coverage_subset(pvro_ctx*, const int64_t* patches, int64_t n);
int pvro_init_volume(pvro_ctx*);
/* Rigidity map ("Integrating p and pbar into a 3D volume using the same PSF as for
 * the reconstruction"; reading Q28): out_k = [W^T (p pbar_s)]_k /
 * [W^T 1]_k where [W^T 1]_k > tau_C, else 0; W^T over the observed pixels of all patches with
 * the reconstruction's row normalisation 1/kappa; p, pbar of the last E-step (1 before any). */
int pvro_rigidity_map(const pvro_ctx*, double* out);
/* ---- f1: rigid patch-to-volume registration by cross correlation (
 * P:185-186 "individual 2D patches are continuously rigidly registered to the current 3D
 * reconstruction"; CC as the similarity; reading Q29). ---------------- */
/* Pearson correlation of n pairs (two-pass); NaN if n < 2 or either side is constant. */
double pvro_cc(int64_t n, const double* a, const double* b);
/* CC of patch s against volume Xl under pose (tx, ty, tz [mm], rx, ry, rz [deg]) applied
 * after the patch's transform T_s, about the transformed patch centre (Q29): over all the
 * patch's pixels, y_j against the trilinear sample of Xl at the pixel's mapped centre
 * (corners outside the grid dropped, i.e. zero, as in the forward model, Q6). *cc = NaN if
 * the patch has fewer than min_valid pixels or either side is constant; *nvalid = pixels. */
int pvro_patch_cc(const pvro_ctx*, const double* Xl, int64_t s, const double* pose, int min_valid,
                  double* cc, int64_t* nvalid);
/* Compose T_new = T_pose o T_s (3x4 row-major) for patch s. */
int pvro_compose_pose(const pvro_ctx*, int64_t s, const double* pose, double* T_new);
/* Register every patch against the current X: `levels` levels of step size 2^-L (2 mm,
 * 4 deg), L = 0 .. levels-1, on the unblurred X, compass search of at most `iters` moves per level over
 * the 12 coordinate moves +-step (best strict improvement, first index on ties), starting
 * from the identity pose. T_out [M][12]: the composed transforms; status [M]: 1 registered, 0
 * unregistrable (undefined CC at the start: transform left unchanged); pose_out [M][6]. */
int pvro_register(const pvro_ctx*, int levels, int iters, int min_valid, double* T_out, int32_t* status,
                  double* pose_out);
/* Test hook: overwrite the E-step state p [P] and pbar [M] (either may be NULL). */
int pvro_set_weights(pvro_ctx*, const double* p, const double* pbar);
int pvro_sr_iterate(pvro_ctx*, int n, double alpha, double lambda);
/* state after the last iteration: per-pixel p and e, per-patch pbar and w */
int pvro_get_weights(const pvro_ctx*, double* p, double* pbar, double* w);
int pvro_get_taps(const pvro_ctx*, double* e, double* kappa, double* A, double* C);
int pvro_get_em_state(const pvro_ctx*, double* sigma2, double* c, double* m, int64_t* t,
                      double* lo, double* hi);
#ifdef __cplusplus
}
#endif
#endif
