// kernels.cu — sm_100a kernels of the PVR SR iteration.
//
// Each kernel cites the PAPER.md passage (P:line) of the step it computes and the
// DESIGN.md reading (Qn) it follows. Positions and interpolation are fp32 (positions
// relative to an integer voxel base per patch); statistics are reduced in fp64.
#include <cfloat>
#include <cmath>

#include "device_util.cuh"
#include "pvr_internal.h"

namespace pvr {

// After k_em_reduce (and the optional cross-rank reduction) of the coverage partials:
// stats = {n_observed, n_live, samples_observed, max y, -min y} over live pixels.
__global__ void k_range_finish(double s2floor, EmDev* em) {
  double ymax = em->stats[3], ymin = -em->stats[4];
  if (!(ymax >= ymin)) { ymin = 0.0; ymax = 0.0; }
  em->ymin = ymin;
  em->ymax = ymax;
  em->lo = ymin - 0.1 * fabs(ymin);
  em->hi = ymax + 0.1 * fabs(ymax);
  em->s2min = s2floor * (ymax - ymin) * (ymax - ymin);
  em->t = 0;
  em->sigma2 = 0.0;
  em->c = 0.0;
  em->m = 0.0;
}

// Fixed-order reduction of the forward's per-block partials into em->stats (one CTA). The blocks
// claim groups dynamically, so the partials (and sigma^2, c, m) reproduce bit for bit only in
// PVR_PARAM_DETERMINISTIC mode, where every term sits on a fixed grid (reading Q35).
__global__ void k_em_reduce(const double* partials, int nblk, EmDev* em) {
  __shared__ double sh[5][32];
  double a[5] = {0.0, 0.0, 0.0, -DBL_MAX, -DBL_MAX};
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    for (int i = 0; i < 3; ++i) a[i] += partials[5 * b + i];
    a[3] = fmax(a[3], partials[5 * b + 3]);
    a[4] = fmax(a[4], partials[5 * b + 4]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    for (int i = 0; i < 3; ++i) a[i] += __shfl_xor_sync(0xffffffffu, a[i], o);
    a[3] = fmax(a[3], __shfl_xor_sync(0xffffffffu, a[3], o));
    a[4] = fmax(a[4], __shfl_xor_sync(0xffffffffu, a[4], o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
    for (int i = 0; i < 5; ++i) sh[i][wid] = a[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[5] = {0.0, 0.0, 0.0, -DBL_MAX, -DBL_MAX};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      for (int i = 0; i < 3; ++i) r[i] += sh[i][w];
      r[3] = fmax(r[3], sh[3][w]);
      r[4] = fmax(r[4], sh[4][w]);
    }
    for (int i = 0; i < 5; ++i) em->stats[i] = r[i];
  }
}

// E-step constants of (sigma^2, c, m): mode, logistic offset, uniform log term.
__device__ void set_mode(EmDev* em, bool degenerate) {
  const double sigma2 = em->sigma2, c = em->c, m = em->m;
  if (degenerate || c >= 1.0) {
    em->mode = 1;
  } else if (c <= 0.0) {
    em->mode = 2;
  } else {
    em->mode = 0;
    // P:202 in logistic form: p = 1 / (1 + exp(ln(m (1-c) / c) + e^2/(2 s2) + ln(2 pi s2)/2))
    em->logk = (float)(log(m * (1.0 - c) / c) + 0.5 * log(2.0 * M_PI * sigma2));
    em->inv2s2 = (float)(1.0 / (2.0 * sigma2));
    em->lnbm = (float)log((1.0 - c) * m);
  }
}

// a3 (reading Q10): sigma^2 = max(sum p e^2 / sum p, s2min),
// c = c0 at t = 1 else sum p / N, m = 1 / (max e - min e). Degenerate (no live pixel or
// spread <= sqrt(s2min)): p = 1 for every observed pixel.
__global__ void k_em_params(Params prm, EmDev* em) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  em->t += 1;
  const double spe2 = em->stats[0], sp = em->stats[1], nl = em->stats[2];
  const double emax = em->stats[3], emin = -em->stats[4];
  double sigma2 = sp > 0.0 ? spe2 / sp : 0.0;
  if (sigma2 < em->s2min) sigma2 = em->s2min;
  const double c = (em->t <= 1) ? (double)prm.c0 : (nl > 0.0 ? sp / nl : (double)prm.c0);
  const double spread = emax - emin;
  const bool degenerate = (nl <= 0.0) || !(spread > sqrt(em->s2min));
  const double m = degenerate ? 0.0 : 1.0 / spread;
  em->sigma2 = sigma2;
  em->c = c;
  em->m = m;
  set_mode(em, degenerate);
  em->degenerate = degenerate;
  em->done = degenerate;  // f4 rounds: nothing to iterate on the degenerate path
  em->ll_prev = NAN;
  em->rounds = 1;
}

// f4 multi-round EM, round >= 2 (reading Q30): stop when the last round gained
// less than tol |LL| over the round before (round >= 3); else the M-step from the last
// E-step's partials: sigma^2 = max(sum p e^2 / sum p, s2min), c = sum p / N (m fixed by e).
__global__ void k_em_round(Params prm, EmDev* em, int round, double tol) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || em->done) return;
  const double ll = em->stats2[2];
  if (round >= 3 && !(ll - em->ll_prev >= tol * fabs(em->ll_prev))) {
    em->done = 1;
    return;
  }
  em->ll_prev = ll;
  const double spe2 = em->stats2[0], sp = em->stats2[1], nl = em->stats[2];
  double sigma2 = sp > 0.0 ? spe2 / sp : 0.0;
  if (sigma2 < em->s2min) sigma2 = em->s2min;
  em->sigma2 = sigma2;
  em->c = nl > 0.0 ? sp / nl : em->c;
  set_mode(em, false);
  em->rounds = round;
}

// --------------------------------------------------------------------------------------
// a4: p_j (observed pixels; 0 elsewhere), pbar_s = sqrt(sum_live p^2 / N_live),
// w_s = pbar_s if pbar_s >= tau_patch else 0 (reading Q13). One CTA per patch; pixels read as
// float4 where the patch's pixel range is 16-byte aligned (every window of extract_patches with
// a width divisible by 4). ROUNDS (f4 multi-round EM, reading Q30) also forms the next M-step's
// partials {sum p e^2, sum p, LL}; the single-round default skips them and the log-likelihood's
// two transcendentals per pixel.
template <bool ROUNDS>
__device__ __forceinline__ void estep_pixel(float k, float ev, const Params& prm, int mode, float logk,
                                            float inv2s2, float lnbm, float& pv, double (&s)[5]) {
  float ll = 0.0f;
  pv = 0.0f;
  if (k >= prm.tau_obs) {
    if (mode == 1) {
      pv = 1.0f;
    } else if (mode == 0) {
      const float z = logk + ev * ev * inv2s2;
      pv = 1.0f / (1.0f + expf(z));
      if (ROUNDS) ll = lnbm + log1pf(expf(-z));  // ln(c G + (1 - c) m) = ln((1-c) m) + ln(1 + e^-z)
    }
  }
  if (k >= prm.tau_live) {
    s[0] += (double)pv * (double)pv;
    s[1] += 1.0;
    if (ROUNDS) {
      s[2] += (double)pv * (double)ev * (double)ev;
      s[3] += (double)pv;
      s[4] += (double)ll;
    }
  }
}

template <bool ROUNDS>
__global__ void __launch_bounds__(256) k_estep(const PatchDev* __restrict__ P, Params prm,
                                               EmDev* __restrict__ em,
                                               const float* __restrict__ kap,
                                               const float* __restrict__ e, float* __restrict__ p,
                                               float* __restrict__ pbar, float* __restrict__ w,
                                               int round, double* __restrict__ rpart,
                                               int32_t* __restrict__ nlive) {
  if (round >= 2 && em->done) return;  // f4 rounds converged: keep the last p, pbar, w
  const PatchDev& pt = P[blockIdx.x];
  const int npix = pt.sx * pt.sy * pt.sz;
  const int mode = em->mode;
  const float logk = em->logk, inv2s2 = em->inv2s2, lnbm = em->lnbm;
  // live-pixel sums: {sum p^2, N} for pbar, and {sum p e^2, sum p, LL} for the next M-step
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  float mx[1] = {0.0f};
  const int64_t j0 = pt.pix0;
  int q0 = 0;
  if ((j0 & 3) == 0) {  // aligned: float4 loads and stores over the multiple-of-4 body
    const int n4 = npix >> 2;
    const float4* k4 = reinterpret_cast<const float4*>(kap + j0);
    const float4* e4 = reinterpret_cast<const float4*>(e + j0);
    float4* p4 = reinterpret_cast<float4*>(p + j0);
    for (int q = threadIdx.x; q < n4; q += blockDim.x) {
      const float4 kk = __ldg(k4 + q), ee = __ldg(e4 + q);
      float4 pp;
      estep_pixel<ROUNDS>(kk.x, ee.x, prm, mode, logk, inv2s2, lnbm, pp.x, s);
      estep_pixel<ROUNDS>(kk.y, ee.y, prm, mode, logk, inv2s2, lnbm, pp.y, s);
      estep_pixel<ROUNDS>(kk.z, ee.z, prm, mode, logk, inv2s2, lnbm, pp.z, s);
      estep_pixel<ROUNDS>(kk.w, ee.w, prm, mode, logk, inv2s2, lnbm, pp.w, s);
      p4[q] = pp;
    }
    q0 = n4 << 2;
  }
  for (int q = q0 + threadIdx.x; q < npix; q += blockDim.x) {
    float pv;
    estep_pixel<ROUNDS>(kap[j0 + q], e[j0 + q], prm, mode, logk, inv2s2, lnbm, pv, s);
    p[j0 + q] = pv;
  }
  __shared__ double res[6];
  block_reduce_store<5, 1>(s, mx, res);
  if (threadIdx.x == 0) {
    const float pb = res[1] > 0.0 ? (float)sqrt(res[0] / res[1]) : 0.0f;
    pbar[blockIdx.x] = pb;
    w[blockIdx.x] = pb >= prm.tau_patch ? pb : 0.0f;
    if (nlive) nlive[blockIdx.x] = (int32_t)res[1];
    if (rpart) {
      // deterministic mode: each patch's sums on fixed grids (2^-4, 2^-24, 2^-10), so the sums
      // over patches are exact in fp64 and independent of their order and of the sharding
      const bool d = prm.det;
      rpart[3 * blockIdx.x] = d ? rint(res[2] * 16.0) / 16.0 : res[2];
      rpart[3 * blockIdx.x + 1] = d ? rint(res[3] * 16777216.0) / 16777216.0 : res[3];
      rpart[3 * blockIdx.x + 2] = d ? rint(res[4] * 1024.0) / 1024.0 : res[4];
    }
  }
}

// Deterministic reduction of the E-step partials into em->stats2 (one CTA).
__global__ void k_em_reduce3(const double* __restrict__ rpart, int64_t npatch, EmDev* em) {
  if (em->done) return;
  double a[3] = {0.0, 0.0, 0.0};
  for (int64_t b = threadIdx.x; b < npatch; b += blockDim.x)
    for (int i = 0; i < 3; ++i) a[i] += rpart[3 * b + i];
  float mx[1] = {0.0f};
  __shared__ double res[4];
  block_reduce_store<3, 1>(a, mx, res);
  if (threadIdx.x == 0)
    for (int i = 0; i < 3; ++i) em->stats2[i] = res[i];
}

// --------------------------------------------------------------------------------------
// f4 two-Gaussian patch classification (reading Q31; oracle/pvro.c
// pvro_patch_mixture): a 1D mixture pi N(mu_in, v_in) + (1 - pi) N(mu_out, v_out) on the
// patch scores of the valid patches (>= 1 live pixel), EM from mu_in = max, mu_out = min,
// v = the scores' variance, pi = 1/2, until the mixture LL gains < tol |LL|; the patch weight
// is the inlier posterior r_s if r_s >= 1/2, else 0. Rank-local sums are NCCL-summed between
// the kernels (engine.cu); single-CTA kernels: M is at most a few 1e5 patches.
__global__ void k_mix_init(const float* __restrict__ pbar, const int32_t* __restrict__ nlive, int64_t M,
                           EmDev* em) {
  double a[3] = {0.0, 0.0, 0.0};
  float mx[2] = {-FLT_MAX, -FLT_MAX};
  for (int64_t s = threadIdx.x; s < M; s += blockDim.x) {
    if (nlive[s] <= 0) continue;
    const double v = pbar[s];
    a[0] += 1.0;
    a[1] += v;
    a[2] += v * v;
    mx[0] = fmaxf(mx[0], (float)v);
    mx[1] = fmaxf(mx[1], (float)-v);
  }
  __shared__ double res[5];
  block_reduce_store<3, 2>(a, mx, res);
  if (threadIdx.x == 0)
    for (int i = 0; i < 5; ++i) em->mix_stats[i] = res[i];
}

__global__ void k_mix_params_init(EmDev* em) {
  if (threadIdx.x != 0) return;
  const double n = em->mix_stats[0], mx = em->mix_stats[3], mn = -em->mix_stats[4];
  em->mix_degenerate = !(n > 0.0) || !(mx - mn > 1e-6);
  em->mix_done = em->mix_degenerate;
  double var = n > 0.0 ? em->mix_stats[2] / n - (em->mix_stats[1] / n) * (em->mix_stats[1] / n) : 0.0;
  if (var < 1e-6) var = 1e-6;
  em->mix_mu[0] = mx;
  em->mix_mu[1] = mn;
  em->mix_v[0] = em->mix_v[1] = var;
  em->mix_pi = 0.5;
  em->mix_ll_prev = NAN;
}

__device__ __forceinline__ double gpdf(double x, double mu, double v) {
  return exp(-(x - mu) * (x - mu) / (2.0 * v)) / sqrt(2.0 * M_PI * v);
}

// E-step of one round with the current parameters: r_s into r, and the sums
// {sum r, sum r pbar, sum r pbar^2, sum (1-r), sum (1-r) pbar, sum (1-r) pbar^2, LL}.
__global__ void k_mix_round(const float* __restrict__ pbar, const int32_t* __restrict__ nlive, int64_t M,
                            EmDev* em, float* __restrict__ r) {
  if (em->mix_done) return;
  const double mu0 = em->mix_mu[0], mu1 = em->mix_mu[1], v0 = em->mix_v[0], v1 = em->mix_v[1];
  const double pi = em->mix_pi;
  double a[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t s = threadIdx.x; s < M; s += blockDim.x) {
    if (nlive[s] <= 0) continue;
    const double x = pbar[s];
    const double ai = pi * gpdf(x, mu0, v0), ao = (1.0 - pi) * gpdf(x, mu1, v1);
    const double rs = (ai + ao > 0.0) ? ai / (ai + ao) : (x >= 0.5 * (mu0 + mu1) ? 1.0 : 0.0);
    r[s] = (float)rs;
    a[0] += rs; a[1] += rs * x; a[2] += rs * x * x;
    a[3] += 1.0 - rs; a[4] += (1.0 - rs) * x; a[5] += (1.0 - rs) * x * x;
    a[6] += log(ai + ao > 0.0 ? ai + ao : 1e-300);
  }
  float mx[1] = {0.0f};
  __shared__ double res[8];
  block_reduce_store<7, 1>(a, mx, res);
  if (threadIdx.x == 0)
    for (int i = 0; i < 7; ++i) em->mix_stats[i] = res[i];
}

// Convergence test on the last E-step's LL, then the M-step.
__global__ void k_mix_update(EmDev* em, int round, double tol) {
  if (threadIdx.x != 0 || em->mix_done) return;
  const double* t = em->mix_stats;
  const double ll = t[6], n = t[0] + t[3];
  if (round >= 1 && !(ll - em->mix_ll_prev >= tol * fabs(em->mix_ll_prev))) {
    em->mix_done = 1;
    return;
  }
  em->mix_ll_prev = ll;
  const double pi = n > 0.0 ? t[0] / n : 0.0;
  if (t[0] > 0.0) { em->mix_mu[0] = t[1] / t[0]; em->mix_v[0] = t[2] / t[0] - em->mix_mu[0] * em->mix_mu[0]; }
  if (t[3] > 0.0) { em->mix_mu[1] = t[4] / t[3]; em->mix_v[1] = t[5] / t[3] - em->mix_mu[1] * em->mix_mu[1]; }
  if (em->mix_v[0] < 1e-6) em->mix_v[0] = 1e-6;
  if (em->mix_v[1] < 1e-6) em->mix_v[1] = 1e-6;
  em->mix_pi = pi;
  if (pi <= 0.0 || pi >= 1.0) em->mix_done = 1;
}

// w_s = r_s if r_s >= 1/2 else 0 (r_s = 1 on the degenerate path, 0 for invalid patches)
__global__ void k_mix_weights(const int32_t* __restrict__ nlive, int64_t M, const EmDev* __restrict__ em,
                              float* __restrict__ w) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < M; s += (int64_t)gridDim.x * blockDim.x) {
    float r = w[s];
    if (nlive[s] <= 0) r = 0.0f;
    else if (em->mix_degenerate) r = 1.0f;
    w[s] = r >= 0.5f ? r : 0.0f;
  }
}

// --------------------------------------------------------------------------------------
// a6 + a7 (P:185 update, reading Q16; P:97 edge-preserving regularisation, reading Q17):
// X1 = clip(X0 + alpha A / C) where C > tau_C; X2 = X1 + alpha lambda sum_{d in D13}
// [b_d(k)(X1_{k+d} - X1_k) + b_d(k-d)(X1_{k-d} - X1_k)], b from X0: the two terms of each
// axis pair d, -d are the 26 neighbours, each weighted by its own b.
// One CTA per 32 x 8 x 8 voxel tile: X0, A, C of the tile plus a 1-voxel halo are read once
// (a warp per halo row, lanes on the 32-aligned interior columns, two lanes on the halo
// columns), X1 and the covered flag c = [C > tau_C] are formed in shared memory, and every
// voxel of the tile sums its 26 neighbours from there as 13 axis pairs (d, -d) of equal weight.
// Tiles whose halo is entirely covered and in the grid (most of the volume) skip the
// per-neighbour coverage tests.
constexpr int kUX = 32, kUY = 8, kUZ = 8;
constexpr int kHX = kUX + 2, kHY = kUY + 2, kHZ = kUZ + 2;

__device__ __forceinline__ float rsqrt_ftz(float x) {  // x >= 1 here: no denormal handling
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// sum over the pair (d, -d) at shared offset O (weight W = |d|_1) of b (X1_n - X1_k),
// b = rsqrt(W (W + g^2)), g = (X0_n - X0_k) / delta
template <int O, int W, bool CHECK>
__device__ __forceinline__ void nb_pair(const float* c0, const float* c1, f2 X0p, f2 X1p, f2 id2, f2& sum) {
  const f2 d0 = sub2(pk(c0[-O], c0[O]), X0p);
  f2 t = fma2(mul2(d0, d0), id2, pk((float)W, (float)W));  // W + g^2
  if (W > 1) t = mul2s((float)W, t);
  const f2 b = pk(rsqrt_ftz(lo2(t)), rsqrt_ftz(hi2(t)));
  f2 dv = sub2(pk(c1[-O], c1[O]), X1p);
  if (CHECK) {  // neighbour uncovered / off-grid (NaN X1): no term
    const float v0 = lo2(dv) == lo2(dv) ? lo2(dv) : 0.0f, v1 = hi2(dv) == hi2(dv) ? hi2(dv) : 0.0f;
    dv = pk(v0, v1);
  }
  sum = fma2(b, dv, sum);
}

template <bool CHECK>
__device__ __forceinline__ float nb_sum(const float* c0, const float* c1, float x0, float x1, float id) {
  constexpr int X = 1, Y = kHX, Z = kHX * kHY;
  const f2 X0p = pk(x0, x0), X1p = pk(x1, x1), id2 = pk(id * id, id * id);
  f2 s = pk(0.0f, 0.0f);
  nb_pair<X, 1, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<Y, 1, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<Z, 1, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X + Y, 2, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X - Y, 2, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X + Z, 2, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X - Z, 2, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<Y + Z, 2, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<Y - Z, 2, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X + Y + Z, 3, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X + Y - Z, 3, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X - Y + Z, 3, CHECK>(c0, c1, X0p, X1p, id2, s);
  nb_pair<X - Y - Z, 3, CHECK>(c0, c1, X0p, X1p, id2, s);
  return lo2(s) + hi2(s);
}

__global__ void __launch_bounds__(256) k_update(const float* __restrict__ X0,
                                                const float2* __restrict__ AC, int3 n, int nxp,
                                                Params prm, const EmDev* __restrict__ em,
                                                float alpha, float lambda, float* __restrict__ X2,
                                                int zlo, int zhi) {
  __shared__ float s0[kHZ * kHY * kHX];  // X0
  __shared__ float s1[kHZ * kHY * kHX];  // X1, NaN where C <= tau_C (uncovered) or off-grid
  const float lo = (float)em->lo, hi = (float)em->hi;
  const int bx = blockIdx.x * kUX - 1, by = blockIdx.y * kUY - 1, bz = zlo + blockIdx.z * kUZ - 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool cov = true;
  // halo rows: a warp takes rows wid, wid + 8, ... on the 32 interior columns, and thread t <
  // 2 rows takes the halo column cell (row t / 2, side t % 2); every load is issued before any
  // is used (the load phase was latency-bound with one row's loads in flight per warp: 70% of
  // the kernel's stall samples)
  constexpr int kRows = kHY * kHZ, kRW = (kRows + 7) / 8;
  static_assert(2 * kRows <= 256, "one halo-column cell per thread");
  float rx0[kRW], ra[kRW], rc[kRW];
#pragma unroll
  for (int t = 0; t < kRW; ++t) {
    const int r = wid + 8 * t;
    rx0[t] = 0.0f; ra[t] = 0.0f; rc[t] = 0.0f;
    const int hz = r / kHY, hy = r - hz * kHY;
    const int j = by + hy, l = bz + hz, i = bx + lane + 1;
    if (r < kRows && (unsigned)j < (unsigned)n.y && (unsigned)l < (unsigned)n.z && (unsigned)i < (unsigned)n.x) {
      const int row = (l * n.y + j) * nxp;  // < 2^31 voxels
      rx0[t] = __ldg(X0 + row + i);
      const float2 ac = __ldg(AC + row + i);
      ra[t] = ac.x;
      rc[t] = ac.y;
    }
  }
  const int hr = threadIdx.x >> 1, hxh = (threadIdx.x & 1) ? kHX - 1 : 0;
  float hx0 = 0.0f, ha = 0.0f, hc = 0.0f;
  {
    const int hz = hr / kHY, hy = hr - hz * kHY;
    const int j = by + hy, l = bz + hz, i = bx + hxh;
    if (hr < kRows && (unsigned)j < (unsigned)n.y && (unsigned)l < (unsigned)n.z && (unsigned)i < (unsigned)n.x) {
      const int row = (l * n.y + j) * nxp;
      hx0 = __ldg(X0 + row + i);
      const float2 ac = __ldg(AC + row + i);
      ha = ac.x;
      hc = ac.y;
    }
  }
  // a6: X1 = clip(X0 + alpha A / C) where C > tau_C (>= 0), else NaN (uncovered;
  // off-grid cells read C = 0)
  auto x1_of = [&](float x0, float a, float c) {
    float x = __int_as_float(0x7fc00000);
    if (c > prm.tau_C) {
      x = fmaf(alpha * a, rcp_ftz(c), x0);
      if (prm.clamp) x = fminf(fmaxf(x, lo), hi);
    }
    return x;
  };
#pragma unroll
  for (int t = 0; t < kRW; ++t) {
    const int r = wid + 8 * t;
    if (r < kRows) {
      const float x1 = x1_of(rx0[t], ra[t], rc[t]);
      cov = cov && (x1 == x1);
      s0[r * kHX + lane + 1] = rx0[t];
      s1[r * kHX + lane + 1] = x1;
    }
  }
  if (hr < kRows) {
    const float h1 = x1_of(hx0, ha, hc);
    cov = cov && (h1 == h1);
    s0[hr * kHX + hxh] = hx0;
    s1[hr * kHX + hxh] = h1;
  }
  const bool allc = __syncthreads_and(cov);
  const float al = alpha * lambda;
  const float id = 1.0f / prm.delta;
  const int i = bx + 1 + lane, j = by + 1 + wid;
  if (i >= n.x || j >= n.y) return;
#pragma unroll 2
  for (int tz = 0; tz < kUZ; ++tz) {
    const int l = bz + 1 + tz;
    if (l >= zhi) break;  // this launch's planes [zlo, zhi) (a rank's slab, or all)
    const int c = ((tz + 1) * kHY + (wid + 1)) * kHX + lane + 1;
    const float x0 = s0[c], x1 = s1[c];
    float out;
    if (x1 != x1) {  // uncovered: X2 = X1 = X0
      out = x0;
    } else {
      // a7 (reading Q17): sum over the 26 neighbours d of b_d (X1_{k+d} - X1_k),
      // b_d = phi_d / sqrt(1 + phi_d ((X0_{k+d} - X0_k) / delta)^2), phi_d = 1/|d|_1
      const float sum = allc ? nb_sum<false>(s0 + c, s1 + c, x0, x1, id) : nb_sum<true>(s0 + c, s1 + c, x0, x1, id);
      out = fmaf(al, sum, x1);
    }
    X2[(l * n.y + j) * nxp + i] = out;
  }
}

// Init: X = A/C where C > tau_C, else mean of the covered 26-neighbours, else 0.
__global__ void __launch_bounds__(256) k_init_fill(const float2* __restrict__ AC, int3 n, int nxp,
                                                   Params prm, float* __restrict__ X) {
  const int64_t V = (int64_t)n.x * n.y * n.z;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < V;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k % n.x);
    const int j = (int)((k / n.x) % n.y);
    const int l = (int)(k / ((int64_t)n.x * n.y));
    const float2 ac = AC[((int64_t)l * n.y + j) * nxp + i];
    float* xo = X + ((int64_t)l * n.y + j) * nxp + i;
    if (ac.y > prm.tau_C) {
      *xo = ac.x / ac.y;
      continue;
    }
    float sum = 0.0f;
    int cnt = 0;
    for (int dl = -1; dl <= 1; ++dl)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          if (!di && !dj && !dl) continue;
          const int i2 = i + di, j2 = j + dj, l2 = l + dl;
          if (i2 < 0 || i2 >= n.x || j2 < 0 || j2 >= n.y || l2 < 0 || l2 >= n.z) continue;
          const float2 a2 = AC[((int64_t)l2 * n.y + j2) * nxp + i2];
          if (a2.y > prm.tau_C) {
            sum += a2.x / a2.y;
            ++cnt;
          }
        }
    *xo = cnt ? sum / (float)cnt : 0.0f;
  }
}

// f2 rigidity map (reading Q28): out = A / C where C > tau_C, else 0 (pitch nxp).
__global__ void __launch_bounds__(256) k_ratio(const float2* __restrict__ AC, int3 n, int nxp, float tau_C,
                                               float* __restrict__ out) {
  const int64_t V = (int64_t)nxp * n.y * n.z;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < V; k += (int64_t)gridDim.x * blockDim.x) {
    const float2 ac = AC[k];
    out[k] = ac.y > tau_C ? ac.x / ac.y : 0.0f;
  }
}

// set_transforms fast path (engine.cu: replan_on_device): recompute every group's voxel
// bounding box of an existing plan for the new geometry, with the host planner's rules
// (member_bbox / size_groups in engine.cu): fp64 member boxes over the lattice range's 8
// corners with a 1e-3 voxel margin; a forward group takes the smallest-area TMA box shape of
// the plan (shapes: the tensor maps already encoded) that holds its new footprint (x origin
// aligned to 4); backprojection groups get fresh odd pitches. A group without a shape or over
// the tile budget sets *fail (the host then replans from scratch).
// fp64 voxel bbox [lo, hi] of one member's PSF samples under the current transform (the host
// planner's member_bbox, engine.cu)
__device__ void replan_member_box(const MemberDev& m, const PatchDev& pt, const StackPsf& ps, int fwd, int (&lo)[3],
                                  int (&hi)[3]) {
  int Ulo, Uhi, Vlo, Vhi;
  if (fwd) {
    Ulo = ps.nu * m.u0 - ps.ru;
    Uhi = ps.nu * (m.u0 + m.tu - 1) + ps.ru + 1;
    Vlo = ps.nv * m.v0 - ps.rv;
    Vhi = ps.nv * (m.v0 + m.tv - 1) + ps.rv + 1;
  } else {
    Ulo = ps.nu * m.u0 - ps.ru;
    Uhi = (m.u0 + m.tu >= pt.sx) ? ps.nu * (pt.sx - 1) + ps.ru + 1 : ps.nu * (m.u0 + m.tu) - ps.ru;
    Vlo = ps.nv * m.v0 - ps.rv;
    Vhi = (m.v0 + m.tv >= pt.sy) ? ps.nv * (pt.sy - 1) + ps.rv + 1 : ps.nv * (m.v0 + m.tv) - ps.rv;
  }
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int c8 = 0; c8 < 8; ++c8) {
    const double U = (c8 & 1) ? Uhi - 1 : Ulo, V = (c8 & 2) ? Vhi - 1 : Vlo, C = (c8 & 4) ? m.c1 : m.c0;
    for (int d = 0; d < 3; ++d) {
      const double x = pt.t0d[d] + m.z * pt.Mzd[d] + U * pt.Qad[d] + V * pt.Qbd[d] + C * pt.Qcd[d];
      mn[d] = fmin(mn[d], x);
      mx[d] = fmax(mx[d], x);
    }
  }
  for (int d = 0; d < 3; ++d) {
    lo[d] = (int)floor(mn[d] - 1e-3);
    hi[d] = (int)floor(mx[d] + 1e-3) + 1;
  }
}

// backprojection tile box of a voxel bbox (the host planner's group(), engine.cu): even x
// origin, odd x / y pitches; returns its voxel count
__device__ int64_t replan_bp_box(int (&lo)[3], const int (&hi)[3], GroupDev& G) {
  lo[0] -= ((lo[0] % 2) + 2) % 2;
  for (int d = 0; d < 3; ++d) G.lo[d] = lo[d];
  G.dim[0] = (hi[0] - lo[0] + 1) | 1;
  G.dim[1] = (hi[1] - lo[1] + 1) | 1;
  G.dim[2] = hi[2] - lo[2] + 1;
  return (int64_t)G.dim[0] * G.dim[1] * G.dim[2];
}

__device__ int replan_interior(const int (&lo)[3], const int (&hi)[3], int3 n) {
  const int nn[3] = {n.x, n.y, n.z};
  for (int d = 0; d < 3; ++d)
    if (lo[d] < 0 || hi[d] > nn[d] - 1) return 0;
  return 1;
}

// Backprojection member: the whole PSF support of every pixel feeding its lines (its tile and
// one pixel around, all through-plane samples) is in the grid (engine.cu: size_groups)
__device__ int replan_support_interior(const MemberDev& m, const PatchDev& pt, const StackPsf& ps, int3 n) {
  MemberDev e = m;
  e.u0 = max(0, m.u0 - 1);
  e.tu = min(pt.sx, m.u0 + m.tu + 1) - e.u0;
  e.v0 = max(0, m.v0 - 1);
  e.tv = min(pt.sy, m.v0 + m.tv + 1) - e.v0;
  e.c0 = -ps.cmax;
  e.c1 = ps.cmax;
  int lo[3], hi[3];
  replan_member_box(e, pt, ps, 1, lo, hi);
  return replan_interior(lo, hi, n);
}

// Device re-plan of one plan for new transforms: same groups and order, new boxes. Forward:
// the smallest existing TMA box shape that holds the new footprint (else fail). Backprojection
// (`nappend` != NULL): a group whose box outgrew the tile budget is emptied (nm = 0) and its
// members appended as single-member groups at [ngroups + k] (k from *nappend, < cap); fail only
// if a single member does not fit or the capacity is exhausted.
__global__ void k_replan(const MemberDev* __restrict__ mem, GroupDev* __restrict__ grp, int ngroups, int cap,
                         const PatchDev* __restrict__ P, const StackPsf* __restrict__ psf, int fwd, int3 n,
                         int64_t vox_budget, const int* __restrict__ shapes, int nshape,
                         int* __restrict__ maxvox, int* __restrict__ fail, int* __restrict__ nappend,
                         int bp_mode) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  GroupDev G = grp[g];
  if (G.nm == 0) return;  // emptied by an earlier split
  int lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-(1 << 30), -(1 << 30), -(1 << 30)};
  int rim = 0, sup = 1;
  for (int i = G.m0; i < G.m0 + G.nm; ++i) {
    const MemberDev m = mem[i];
    const PatchDev& pt = P[m.patch];
    int ml[3], mh[3];
    replan_member_box(m, pt, psf[pt.stack], fwd, ml, mh);
    rim |= m.flags & kMemberRim;
    if (!fwd && bp_mode == kBpRim) sup &= replan_support_interior(m, pt, psf[pt.stack], n);
    for (int d = 0; d < 3; ++d) {
      lo[d] = min(lo[d], ml[d]);
      hi[d] = max(hi[d], mh[d]);
    }
  }
  G.interior = replan_interior(lo, hi, n);
  // backprojection tile precision (engine.cu: size_groups): exact for rim members and
  // footprints that leave the grid; the byte budget then buys half the cells
  G.exact = !fwd && (bp_mode >= kBpAll || (bp_mode == kBpRim && (rim || !sup)));
  // (deterministic mode: 4 B per cell in each of 6 planes of kBpDetPlane bytes)
  const int64_t cell_bytes = bp_mode == kBpDet ? 24 : G.exact ? 16 : 8;
  int64_t vox;
  if (fwd) {
    lo[0] -= ((lo[0] % 4) + 4) % 4;
    const int w = hi[0] - lo[0] + 1, h = hi[1] - lo[1] + 1;
    int best = -1, barea = 1 << 30;
    for (int k = 0; k < nshape; ++k) {
      const int sw = shapes[2 * k], sh = shapes[2 * k + 1];
      if (sw >= w && sh >= h && sw * sh < barea) { barea = sw * sh; best = k; }
    }
    if (best < 0) {
      atomicExch(fail, 1);
      best = G.tmap;
    }
    G.tmap = best;
    G.dim[0] = shapes[2 * best];
    G.dim[1] = shapes[2 * best + 1];
    for (int d = 0; d < 3; ++d) G.lo[d] = lo[d];
    G.dim[2] = hi[2] - lo[2] + 1;
    vox = (int64_t)((G.dim[0] * G.dim[1] + 31) & ~31) * G.dim[2];
  } else {
    vox = replan_bp_box(lo, hi, G);
    if (vox * cell_bytes > vox_budget && nappend && G.nm > 1) {
      for (int i = G.m0; i < G.m0 + G.nm; ++i) {
        const MemberDev m = mem[i];
        const PatchDev& pt = P[m.patch];
        int ml[3], mh[3];
        replan_member_box(m, pt, psf[pt.stack], 0, ml, mh);
        GroupDev S;
        S.m0 = i;
        S.nm = 1;
        S.tmap = 0;
        S.interior = replan_interior(ml, mh, n);
        // a split never lowers precision: the singles of an exact group stay exact
        S.exact = G.exact;
        const int64_t sv = replan_bp_box(ml, mh, S);
        const int k = atomicAdd(nappend, 1);
        if (sv * (bp_mode == kBpDet ? 24 : S.exact ? 16 : 8) > vox_budget ||
            (bp_mode == kBpDet && sv * 4 > kBpDetPlane) || ngroups + k >= cap) {
          atomicExch(fail, 1);
          continue;
        }
        atomicMax(maxvox, (int)sv);
        grp[ngroups + k] = S;
      }
      G.nm = 0;  // emptied: its members now live in the appended groups
      G.dim[0] = G.dim[1] = G.dim[2] = 0;
      vox = 0;
    }
  }
  if ((fwd ? vox : vox * cell_bytes) > vox_budget || (bp_mode == kBpDet && vox * 4 > kBpDetPlane))
    atomicExch(fail, 1);
  atomicMax(maxvox, (int)(vox < (1 << 30) ? vox : (1 << 30)));
  grp[g] = G;
}

// ---- deterministic mode (PVR_PARAM_DETERMINISTIC) -----------------------------------------
// Per patch: the maxima over its observed pixels of |rA| and rC (the backprojection's per-pixel
// inputs, the same formulas as k_lattice_bp's phase A), into em->det_max by atomicMax on the
// (non-negative) float bits: order-independent.
__global__ void k_bp_maxima(const PatchDev* __restrict__ P, Params prm, const float* __restrict__ kap,
                            const float* __restrict__ e, const float* __restrict__ p,
                            const float* __restrict__ w, const float* __restrict__ ys, int init,
                            EmDev* __restrict__ em) {
  const PatchDev& pt = P[blockIdx.x];
  const float ws = init == 1 ? 1.0f : (init == 2 ? 1.0f : w[blockIdx.x]);
  const float vs = init == 2 ? w[blockIdx.x] : 1.0f;
  if (ws == 0.0f) return;
  float mA = 0.0f, mC = 0.0f;
  const int npix = pt.sx * pt.sy * pt.sz;
  for (int q = threadIdx.x; q < npix; q += blockDim.x) {
    const int64_t j = pt.pix0 + q;
    const float k = kap[j];
    if (!(k >= prm.tau_obs)) continue;
    const int u = q % pt.sx, v = (q / pt.sx) % pt.sy, z = q / (pt.sx * pt.sy);
    const float pv = init ? 1.0f : p[j];
    const float val = init == 1 ? ys[pt.y0off + (int64_t)z * pt.HW + (int64_t)v * pt.W + u]
                                : init == 2 ? p[j] * vs : e[j];
    const float rC = ws * pv / k;
    mA = fmaxf(mA, fabsf(rC * val));
    mC = fmaxf(mC, rC);
  }
  mA = warp_max(mA);
  mC = warp_max(mC);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(reinterpret_cast<int*>(&em->det_max[0]), __float_as_int(mA));
    atomicMax(reinterpret_cast<int*>(&em->det_max[1]), __float_as_int(mC));
  }
}

// The global scales: the largest splat term maps to kDetTermMax units (tp <= 1).
__global__ void k_det_scales(EmDev* em) {
  if (threadIdx.x != 0) return;
  for (int q = 0; q < 2; ++q) em->det_scale[q] = em->det_max[q] > 0.0f ? kDetTermMax / (double)em->det_max[q] : 0.0;
}

// (A, C) = int64 totals / scale: {A hi, A lo 2^20 + lo2, C hi, C lo 2^20 + lo2} per voxel.
__global__ void k_det_to_float(const unsigned long long* __restrict__ ACd, int64_t Vp, const EmDev* __restrict__ em,
                               float2* __restrict__ AC) {
  const double iA = em->det_scale[0] > 0.0 ? 1.0 / em->det_scale[0] : 0.0;
  const double iC = em->det_scale[1] > 0.0 ? 1.0 / em->det_scale[1] : 0.0;
  const double l2 = 1.0 / (1048576.0 * 1048576.0);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < Vp; k += (int64_t)gridDim.x * blockDim.x) {
    const long long* v = reinterpret_cast<const long long*>(ACd + 4 * k);
    AC[k] = make_float2((float)(((double)v[0] + (double)v[1] * l2) * iA), (float)(((double)v[2] + (double)v[3] * l2) * iC));
  }
}

// One quantity of the interleaved, row-padded (A, C) volume into a contiguous [nz][ny][nx]
// array (pvr_get_confidence, the taps).
__global__ void k_unpack_ac(const float2* __restrict__ AC, int3 n, int nxp, int which, float* __restrict__ out) {
  const int64_t V = (int64_t)n.x * n.y * n.z;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < V; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = k / n.x;
    const float2 ac = AC[row * nxp + (k - row * n.x)];
    out[k] = which ? ac.y : ac.x;
  }
}

__global__ void k_scale(float* __restrict__ x, int64_t n, float f) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= f;
}

__global__ void k_fill(float* __restrict__ x, int64_t n, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

// --------------------------------------------------------------------------------------
// launchers

void launch_bp_maxima(cudaStream_t st, const PatchDev* P, int64_t npatch, Params prm, const float* kap,
                      const float* e, const float* p, const float* w, const float* ys, int init, EmDev* em) {
  if (npatch > 0) k_bp_maxima<<<(unsigned)npatch, 256, 0, st>>>(P, prm, kap, e, p, w, ys, init, em);
}

void launch_det_scales(cudaStream_t st, EmDev* em) { k_det_scales<<<1, 32, 0, st>>>(em); }

void launch_det_to_float(cudaStream_t st, const unsigned long long* ACd, int64_t Vp, const EmDev* em, float2* AC) {
  k_det_to_float<<<148 * 8, 256, 0, st>>>(ACd, Vp, em, AC);
}

void launch_unpack_ac(cudaStream_t st, const float2* AC, int3 dims, int nxp, int which, float* out) {
  k_unpack_ac<<<148 * 8, 256, 0, st>>>(AC, dims, nxp, which, out);
}

void launch_scale(cudaStream_t st, float* x, int64_t n, float f) {
  if (n > 0) k_scale<<<148 * 8, 256, 0, st>>>(x, n, f);
}

void launch_fill(cudaStream_t st, float* x, int64_t n, float v) {
  if (n > 0) k_fill<<<148 * 8, 256, 0, st>>>(x, n, v);
}

void launch_range_finish(cudaStream_t st, double s2floor, EmDev* em) {
  k_range_finish<<<1, 1, 0, st>>>(s2floor, em);
}

void launch_em_reduce(cudaStream_t st, const double* partials, int nblk, EmDev* em) {
  k_em_reduce<<<1, 1024, 0, st>>>(partials, nblk, em);
}

void launch_em_params(cudaStream_t st, Params prm, EmDev* em) {
  k_em_params<<<1, 32, 0, st>>>(prm, em);
}

void launch_estep(cudaStream_t st, const PatchDev* P, int64_t npatch, Params prm, EmDev* em,
                  const float* kap, const float* e, float* p, float* pbar, float* w, int round,
                  double* rpart, int32_t* nlive) {
  if (npatch <= 0) return;
  if (rpart)
    k_estep<true><<<(unsigned)npatch, 256, 0, st>>>(P, prm, em, kap, e, p, pbar, w, round, rpart, nlive);
  else
    k_estep<false><<<(unsigned)npatch, 256, 0, st>>>(P, prm, em, kap, e, p, pbar, w, round, rpart, nlive);
}

void launch_em_reduce3(cudaStream_t st, const double* rpart, int64_t npatch, EmDev* em) {
  k_em_reduce3<<<1, 1024, 0, st>>>(rpart, npatch, em);
}

void launch_mix_init(cudaStream_t st, const float* pbar, const int32_t* nlive, int64_t npatch, EmDev* em) {
  k_mix_init<<<1, 1024, 0, st>>>(pbar, nlive, npatch, em);
}
void launch_mix_params_init(cudaStream_t st, EmDev* em) { k_mix_params_init<<<1, 32, 0, st>>>(em); }
void launch_mix_round(cudaStream_t st, const float* pbar, const int32_t* nlive, int64_t npatch, EmDev* em, float* r) {
  k_mix_round<<<1, 1024, 0, st>>>(pbar, nlive, npatch, em, r);
}
void launch_mix_update(cudaStream_t st, EmDev* em, int round, double tol) {
  k_mix_update<<<1, 32, 0, st>>>(em, round, tol);
}
void launch_mix_weights(cudaStream_t st, const int32_t* nlive, int64_t npatch, const EmDev* em, float* w) {
  if (npatch > 0) k_mix_weights<<<(unsigned)((npatch + 255) / 256), 256, 0, st>>>(nlive, npatch, em, w);
}

void launch_em_round(cudaStream_t st, Params prm, EmDev* em, int round, double tol) {
  k_em_round<<<1, 32, 0, st>>>(prm, em, round, tol);
}

void launch_update(cudaStream_t st, const float* X0, const float2* AC, const int3 dims, int nxp,
                   Params prm, const EmDev* em, float alpha, float lambda, float* X2, int zlo, int zhi) {
  if (zhi <= zlo) return;
  const dim3 grid((dims.x + kUX - 1) / kUX, (dims.y + kUY - 1) / kUY, (zhi - zlo + kUZ - 1) / kUZ);
  k_update<<<grid, 256, 0, st>>>(X0, AC, dims, nxp, prm, em, alpha, lambda, X2, zlo, zhi);
}

void launch_replan(cudaStream_t st, const MemberDev* mem, GroupDev* grp, int ngroups, int cap, const PatchDev* P,
                   const StackPsf* psf, int fwd, int3 n, int64_t vox_budget, const int* shapes, int nshape,
                   int* maxvox, int* fail, int* nappend, int bp_mode) {
  if (ngroups > 0)
    k_replan<<<(ngroups + 255) / 256, 256, 0, st>>>(mem, grp, ngroups, cap, P, psf, fwd, n, vox_budget, shapes,
                                                     nshape, maxvox, fail, nappend, bp_mode);
}

void launch_ratio(cudaStream_t st, const float2* AC, const int3 dims, int nxp, float tau_C, float* out) {
  k_ratio<<<148 * 8, 256, 0, st>>>(AC, dims, nxp, tau_C, out);
}

void launch_init_fill(cudaStream_t st, const float2* AC, const int3 dims, int nxp, Params prm, float* X) {
  k_init_fill<<<148 * 16, 256, 0, st>>>(AC, dims, nxp, prm, X);
}

}  // namespace pvr
