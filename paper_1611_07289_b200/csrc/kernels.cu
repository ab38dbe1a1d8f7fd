// kernels.cu — sm_100a kernels of the PVR SR iteration.
//
// Each kernel cites the PAPER.md passage (P:line) of the step it computes and the
// DESIGN.md reading (Qn) it follows. Positions and interpolation are fp32 (positions
// relative to an integer voxel base per patch); statistics are reduced in fp64.
#include <cfloat>
#include <cmath>

#include "pvr_internal.h"

namespace pvr {

// --------------------------------------------------------------------------------------
// shared helpers

__device__ __forceinline__ void pixel_coords(const PatchDev& pt, int q, int& u, int& v, int& z) {
  int nxy = pt.sx * pt.sy;
  z = q / nxy;
  int r = q - z * nxy;
  v = r / pt.sx;
  u = r - v * pt.sx;
}

// Trilinear weights of a continuous local index r (relative to `base`), with corners
// outside [0, n-1] given weight 0 and their index clamped in-grid (reading Q6: out-of-grid
// corners are dropped, not redistributed). The in-grid set is a product set, so the
// in-grid mass of the 8 corners is (wx0+wx1)(wy0+wy1)(wz0+wz1).
struct Tri {
  int i0, j0, l0, i1, j1, l1;
  float wx0, wx1, wy0, wy1, wz0, wz1;
};

__device__ __forceinline__ void tri_axis(float r, int base, int n, int& a0, int& a1, float& w0,
                                         float& w1) {
  float fl = floorf(r);
  float f = r - fl;
  int i = base + (int)fl;
  w0 = (i >= 0 && i < n) ? 1.0f - f : 0.0f;
  w1 = (i + 1 >= 0 && i + 1 < n) ? f : 0.0f;
  a0 = min(max(i, 0), n - 1);
  a1 = min(max(i + 1, 0), n - 1);
}

__device__ __forceinline__ Tri tri_weights(float rx, float ry, float rz, const int32_t* base, int3 n) {
  Tri t;
  tri_axis(rx, base[0], n.x, t.i0, t.i1, t.wx0, t.wx1);
  tri_axis(ry, base[1], n.y, t.j0, t.j1, t.wy0, t.wy1);
  tri_axis(rz, base[2], n.z, t.l0, t.l1, t.wz0, t.wz1);
  return t;
}

__device__ __forceinline__ float tri_gather(const float* __restrict__ X, const Tri& t, int3 n) {
  const size_t sy = (size_t)n.x, sz = (size_t)n.x * n.y;
  const float* p00 = X + t.l0 * sz + t.j0 * sy;
  const float* p01 = X + t.l0 * sz + t.j1 * sy;
  const float* p10 = X + t.l1 * sz + t.j0 * sy;
  const float* p11 = X + t.l1 * sz + t.j1 * sy;
  float c00 = t.wx0 * __ldg(p00 + t.i0) + t.wx1 * __ldg(p00 + t.i1);
  float c01 = t.wx0 * __ldg(p01 + t.i0) + t.wx1 * __ldg(p01 + t.i1);
  float c10 = t.wx0 * __ldg(p10 + t.i0) + t.wx1 * __ldg(p10 + t.i1);
  float c11 = t.wx0 * __ldg(p11 + t.i0) + t.wx1 * __ldg(p11 + t.i1);
  return t.wz0 * (t.wy0 * c00 + t.wy1 * c01) + t.wz1 * (t.wy0 * c10 + t.wy1 * c11);
}

__device__ __forceinline__ void red_v2(float2* addr, float a, float c) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(c) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-reduce NS sums (double) and NM maxima (float) of a 256-thread block into out[].
template <int NS, int NM>
__device__ __forceinline__ void block_reduce_store(double (&s)[NS], float (&mx)[NM], double* out) {
  __shared__ double sh_s[8][NS > 0 ? NS : 1];
  __shared__ float sh_m[8][NM > 0 ? NM : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NS; ++i) s[i] = warp_sum(s[i]);
#pragma unroll
  for (int i = 0; i < NM; ++i) mx[i] = warp_max(mx[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) sh_s[wid][i] = s[i];
#pragma unroll
    for (int i = 0; i < NM; ++i) sh_m[wid][i] = mx[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int i = 0; i < NS; ++i) {
      double a = 0.0;
      for (int w = 0; w < nw; ++w) a += sh_s[w][i];
      out[i] = a;
    }
    for (int i = 0; i < NM; ++i) {
      float a = -FLT_MAX;
      for (int w = 0; w < nw; ++w) a = fmaxf(a, sh_m[w][i]);
      out[NS + i] = (double)a;
    }
  }
}

// --------------------------------------------------------------------------------------
// Coverage (set_transforms): kappa_j = sum_q psi_q sum_{k in grid}
// t_k(x_jq). Geometry only. Also the live-y range {min y, max y} and pixel counts.
__global__ void __launch_bounds__(kTile) k_coverage(const PatchDev* __restrict__ P,
                                                    const float4* __restrict__ psf,
                                                    const int2* __restrict__ tiles, int64_t ntiles,
                                                    const float* __restrict__ ys, int3 n, Params prm,
                                                    float* __restrict__ kap, double* partials) {
  double cnt[3] = {0.0, 0.0, 0.0};            // observed, live, PSF samples of observed
  float mx[2] = {-FLT_MAX, -FLT_MAX};         // max y, -min y over live
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int2 tl = tiles[t];
    const PatchDev& pt = P[tl.x];
    const int q = tl.y + threadIdx.x;
    if (q >= pt.sx * pt.sy * pt.sz) continue;
    int u, v, z;
    pixel_coords(pt, q, u, v, z);
    const float rx0 = pt.frac[0] + u * pt.Mu[0] + v * pt.Mv[0] + z * pt.Mz[0];
    const float ry0 = pt.frac[1] + u * pt.Mu[1] + v * pt.Mv[1] + z * pt.Mz[1];
    const float rz0 = pt.frac[2] + u * pt.Mu[2] + v * pt.Mv[2] + z * pt.Mz[2];
    float k = 0.0f;
    for (int s = 0; s < pt.S; ++s) {
      const float4 a = __ldg(&psf[pt.psf0 + s]);
      const float rx = rx0 + a.x * pt.Qa[0] + a.y * pt.Qb[0] + a.z * pt.Qc[0];
      const float ry = ry0 + a.x * pt.Qa[1] + a.y * pt.Qb[1] + a.z * pt.Qc[1];
      const float rz = rz0 + a.x * pt.Qa[2] + a.y * pt.Qb[2] + a.z * pt.Qc[2];
      const Tri tw = tri_weights(rx, ry, rz, pt.base, n);
      k += a.w * ((tw.wx0 + tw.wx1) * (tw.wy0 + tw.wy1) * (tw.wz0 + tw.wz1));
    }
    kap[pt.pix0 + q] = k;
    if (k >= prm.tau_obs) {
      cnt[0] += 1.0;
      cnt[2] += (double)pt.S;
    }
    if (k >= prm.tau_live) {
      const float y = ys[pt.y0off + (int64_t)z * pt.HW + (int64_t)v * pt.W + u];
      cnt[1] += 1.0;
      mx[0] = fmaxf(mx[0], y);
      mx[1] = fmaxf(mx[1], -y);
    }
  }
  block_reduce_store<3, 2>(cnt, mx, partials + (size_t)blockIdx.x * 5);
}

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

// --------------------------------------------------------------------------------------
// a1 + a2 (Eq. 1): yhat_j = kappa_j^-1 sum_q psi_q trilerp(X, x_jq),
// e_j = y_j - yhat_j on observed pixels (0 elsewhere), and the M-step sufficient
// statistics over live pixels {sum p_prev e^2, sum p_prev, N, max e, -min e}.
__global__ void __launch_bounds__(kTile) k_forward(const PatchDev* __restrict__ P,
                                                   const float4* __restrict__ psf,
                                                   const int2* __restrict__ tiles, int64_t ntiles,
                                                   const float* __restrict__ ys,
                                                   const float* __restrict__ X, int3 n, Params prm,
                                                   const float* __restrict__ kap,
                                                   const float* __restrict__ pprev,
                                                   float* __restrict__ e, double* partials) {
  double s[3] = {0.0, 0.0, 0.0};
  float mx[2] = {-FLT_MAX, -FLT_MAX};
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int2 tl = tiles[t];
    const PatchDev& pt = P[tl.x];
    const int q = tl.y + threadIdx.x;
    if (q >= pt.sx * pt.sy * pt.sz) continue;
    int u, v, z;
    pixel_coords(pt, q, u, v, z);
    const int64_t j = pt.pix0 + q;
    const float k = kap[j];
    float ev = 0.0f;
    if (k >= prm.tau_obs) {
      const float rx0 = pt.frac[0] + u * pt.Mu[0] + v * pt.Mv[0] + z * pt.Mz[0];
      const float ry0 = pt.frac[1] + u * pt.Mu[1] + v * pt.Mv[1] + z * pt.Mz[1];
      const float rz0 = pt.frac[2] + u * pt.Mu[2] + v * pt.Mv[2] + z * pt.Mz[2];
      float acc = 0.0f;
      for (int si = 0; si < pt.S; ++si) {
        const float4 a = __ldg(&psf[pt.psf0 + si]);
        const float rx = rx0 + a.x * pt.Qa[0] + a.y * pt.Qb[0] + a.z * pt.Qc[0];
        const float ry = ry0 + a.x * pt.Qa[1] + a.y * pt.Qb[1] + a.z * pt.Qc[1];
        const float rz = rz0 + a.x * pt.Qa[2] + a.y * pt.Qb[2] + a.z * pt.Qc[2];
        const Tri tw = tri_weights(rx, ry, rz, pt.base, n);
        acc += a.w * tri_gather(X, tw, n);
      }
      const float y = ys[pt.y0off + (int64_t)z * pt.HW + (int64_t)v * pt.W + u];
      ev = y - acc / k;
      if (k >= prm.tau_live) {
        const double pp = pprev[j];
        s[0] += pp * (double)ev * (double)ev;
        s[1] += pp;
        s[2] += 1.0;
        mx[0] = fmaxf(mx[0], ev);
        mx[1] = fmaxf(mx[1], -ev);
      }
    }
    e[j] = ev;
  }
  block_reduce_store<3, 2>(s, mx, partials + (size_t)blockIdx.x * 5);
}

// Deterministic reduction of the forward partials into em->stats (one CTA).
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
  if (degenerate || c >= 1.0) {
    em->mode = 1;
  } else if (c <= 0.0) {
    em->mode = 2;
  } else {
    em->mode = 0;
    // P:202 in logistic form: p = 1 / (1 + exp(ln(m (1-c) / c) + e^2/(2 s2) + ln(2 pi s2)/2))
    em->logk = (float)(log(m * (1.0 - c) / c) + 0.5 * log(2.0 * M_PI * sigma2));
    em->inv2s2 = (float)(1.0 / (2.0 * sigma2));
  }
}

// --------------------------------------------------------------------------------------
// a4: p_j (observed pixels; 0 elsewhere), pbar_s = sqrt(sum_live p^2 / N_live),
// w_s = pbar_s if pbar_s >= tau_patch else 0 (reading Q13). One CTA per patch.
__global__ void __launch_bounds__(256) k_estep(const PatchDev* __restrict__ P, Params prm,
                                               const EmDev* __restrict__ em,
                                               const float* __restrict__ kap,
                                               const float* __restrict__ e, float* __restrict__ p,
                                               float* __restrict__ pbar, float* __restrict__ w) {
  const PatchDev& pt = P[blockIdx.x];
  const int npix = pt.sx * pt.sy * pt.sz;
  const int mode = em->mode;
  const float logk = em->logk, inv2s2 = em->inv2s2;
  double s[2] = {0.0, 0.0};
  float mx[1] = {0.0f};
  for (int q = threadIdx.x; q < npix; q += blockDim.x) {
    const int64_t j = pt.pix0 + q;
    const float k = kap[j];
    float pv = 0.0f;
    if (k >= prm.tau_obs) {
      if (mode == 1) {
        pv = 1.0f;
      } else if (mode == 0) {
        const float ev = e[j];
        pv = 1.0f / (1.0f + expf(logk + ev * ev * inv2s2));
      }
    }
    p[j] = pv;
    if (k >= prm.tau_live) {
      s[0] += (double)pv * (double)pv;
      s[1] += 1.0;
    }
  }
  __shared__ double res[3];
  block_reduce_store<2, 1>(s, mx, res);
  if (threadIdx.x == 0) {
    const float pb = res[1] > 0.0 ? (float)sqrt(res[0] / res[1]) : 0.0f;
    pbar[blockIdx.x] = pb;
    w[blockIdx.x] = pb >= prm.tau_patch ? pb : 0.0f;
  }
}

// --------------------------------------------------------------------------------------
// a5 ("pixel-volume"): A_k += sum_s w_s sum_j W_jk p_j e_j and
// C_k += sum_s w_s sum_j W_jk p_j, with W_jk = psi_q t_k(x_jq) / kappa_j. init = 1 gives
// the initial-volume pass (p = w = 1, e := y). Direct form, global red.v2 per corner.
__global__ void __launch_bounds__(kTile) k_backproject(const PatchDev* __restrict__ P,
                                                       const float4* __restrict__ psf,
                                                       const int2* __restrict__ tiles,
                                                       int64_t ntiles, const float* __restrict__ ys,
                                                       int3 n, Params prm,
                                                       const float* __restrict__ kap,
                                                       const float* __restrict__ e,
                                                       const float* __restrict__ p,
                                                       const float* __restrict__ w, int init,
                                                       float2* __restrict__ AC) {
  const size_t sy = (size_t)n.x, sz = (size_t)n.x * n.y;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int2 tl = tiles[t];
    const PatchDev& pt = P[tl.x];
    const float ws = init ? 1.0f : w[tl.x];
    if (ws == 0.0f) continue;
    const int q = tl.y + threadIdx.x;
    if (q >= pt.sx * pt.sy * pt.sz) continue;
    int u, v, z;
    pixel_coords(pt, q, u, v, z);
    const int64_t j = pt.pix0 + q;
    const float k = kap[j];
    if (!(k >= prm.tau_obs)) continue;
    const float pv = init ? 1.0f : p[j];
    if (pv == 0.0f) continue;
    const float val = init ? ys[pt.y0off + (int64_t)z * pt.HW + (int64_t)v * pt.W + u] : e[j];
    const float rC = ws * pv / k;
    const float rA = rC * val;
    const float rx0 = pt.frac[0] + u * pt.Mu[0] + v * pt.Mv[0] + z * pt.Mz[0];
    const float ry0 = pt.frac[1] + u * pt.Mu[1] + v * pt.Mv[1] + z * pt.Mz[1];
    const float rz0 = pt.frac[2] + u * pt.Mu[2] + v * pt.Mv[2] + z * pt.Mz[2];
    for (int si = 0; si < pt.S; ++si) {
      const float4 a = __ldg(&psf[pt.psf0 + si]);
      const float rx = rx0 + a.x * pt.Qa[0] + a.y * pt.Qb[0] + a.z * pt.Qc[0];
      const float ry = ry0 + a.x * pt.Qa[1] + a.y * pt.Qb[1] + a.z * pt.Qc[1];
      const float rz = rz0 + a.x * pt.Qa[2] + a.y * pt.Qb[2] + a.z * pt.Qc[2];
      const Tri tw = tri_weights(rx, ry, rz, pt.base, n);
      const float cA = a.w * rA, cC = a.w * rC;
#pragma unroll
      for (int cz = 0; cz < 2; ++cz) {
        const float wz = cz ? tw.wz1 : tw.wz0;
        if (wz == 0.0f) continue;
        const size_t ol = (size_t)(cz ? tw.l1 : tw.l0) * sz;
#pragma unroll
        for (int cy = 0; cy < 2; ++cy) {
          const float wyz = wz * (cy ? tw.wy1 : tw.wy0);
          if (wyz == 0.0f) continue;
          const size_t oj = ol + (size_t)(cy ? tw.j1 : tw.j0) * sy;
          if (tw.wx0 != 0.0f) red_v2(AC + oj + tw.i0, cA * wyz * tw.wx0, cC * wyz * tw.wx0);
          if (tw.wx1 != 0.0f) red_v2(AC + oj + tw.i1, cA * wyz * tw.wx1, cC * wyz * tw.wx1);
        }
      }
    }
  }
}

// --------------------------------------------------------------------------------------
// a6 + a7 (P:185 update, reading Q16; P:97 edge-preserving regularisation, reading Q17):
// X1 = clip(X0 + alpha A / C) where C > tau_C; X2 = X1 + alpha lambda sum_{d in D13}
// [b_d(k)(X1_{k+d} - X1_k) + b_d(k-d)(X1_{k-d} - X1_k)], b from X0. Direct 27-point form.
__constant__ int c_D13[13][3] = {{1, 0, -1}, {0, 1, -1}, {1, 1, -1}, {1, -1, -1}, {1, 0, 0},
                                 {0, 1, 0},  {1, 1, 0},  {1, -1, 0}, {1, 0, 1},   {0, 1, 1},
                                 {1, 1, 1},  {1, -1, 1}, {0, 0, 1}};

__device__ __forceinline__ float sr_update(float x0, float2 ac, float alpha, float tauC, int clamp,
                                           float lo, float hi) {
  if (!(ac.y > tauC)) return x0;
  float x = x0 + alpha * ac.x / ac.y;
  if (clamp) x = fminf(fmaxf(x, lo), hi);
  return x;
}

__global__ void __launch_bounds__(256) k_update(const float* __restrict__ X0,
                                                const float2* __restrict__ AC, int3 n, Params prm,
                                                const EmDev* __restrict__ em, float alpha,
                                                float lambda, float* __restrict__ X2) {
  const int64_t V = (int64_t)n.x * n.y * n.z;
  const float lo = (float)em->lo, hi = (float)em->hi;
  const float inv_delta = 1.0f / prm.delta;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < V;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k % n.x);
    const int j = (int)((k / n.x) % n.y);
    const int l = (int)(k / ((int64_t)n.x * n.y));
    const float x0 = X0[k];
    const float2 ac = AC[k];
    const float x1 = sr_update(x0, ac, alpha, prm.tau_C, prm.clamp, lo, hi);
    if (!(ac.y > prm.tau_C)) {
      X2[k] = x1;
      continue;
    }
    float sum = 0.0f;
#pragma unroll
    for (int d = 0; d < 13; ++d) {
      const int dx = c_D13[d][0], dy = c_D13[d][1], dz = c_D13[d][2];
      const float phi = 1.0f / (float)(abs(dx) + abs(dy) + abs(dz));
#pragma unroll
      for (int sg = -1; sg <= 1; sg += 2) {
        const int i2 = i + sg * dx, j2 = j + sg * dy, l2 = l + sg * dz;
        if (i2 < 0 || i2 >= n.x || j2 < 0 || j2 >= n.y || l2 < 0 || l2 >= n.z) continue;
        const int64_t k2 = ((int64_t)l2 * n.y + j2) * n.x + i2;
        const float2 ac2 = AC[k2];
        if (!(ac2.y > prm.tau_C)) continue;
        const float x02 = X0[k2];
        const float x12 = sr_update(x02, ac2, alpha, prm.tau_C, prm.clamp, lo, hi);
        const float g = (x02 - x0) * inv_delta;
        const float b = phi * rsqrtf(1.0f + phi * g * g);
        sum += b * (x12 - x1);
      }
    }
    X2[k] = x1 + alpha * lambda * sum;
  }
}

// Init: X = A/C where C > tau_C, else mean of the covered 26-neighbours, else 0.
__global__ void __launch_bounds__(256) k_init_fill(const float2* __restrict__ AC, int3 n,
                                                   Params prm, float* __restrict__ X) {
  const int64_t V = (int64_t)n.x * n.y * n.z;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < V;
       k += (int64_t)gridDim.x * blockDim.x) {
    const float2 ac = AC[k];
    if (ac.y > prm.tau_C) {
      X[k] = ac.x / ac.y;
      continue;
    }
    const int i = (int)(k % n.x);
    const int j = (int)((k / n.x) % n.y);
    const int l = (int)(k / ((int64_t)n.x * n.y));
    float sum = 0.0f;
    int cnt = 0;
    for (int dl = -1; dl <= 1; ++dl)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          if (!di && !dj && !dl) continue;
          const int i2 = i + di, j2 = j + dj, l2 = l + dl;
          if (i2 < 0 || i2 >= n.x || j2 < 0 || j2 >= n.y || l2 < 0 || l2 >= n.z) continue;
          const float2 a2 = AC[((int64_t)l2 * n.y + j2) * n.x + i2];
          if (a2.y > prm.tau_C) {
            sum += a2.x / a2.y;
            ++cnt;
          }
        }
    X[k] = cnt ? sum / (float)cnt : 0.0f;
  }
}

__global__ void k_fill(float* __restrict__ x, int64_t n, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

// --------------------------------------------------------------------------------------
// launchers

void launch_fill(cudaStream_t st, float* x, int64_t n, float v) {
  if (n > 0) k_fill<<<148 * 8, 256, 0, st>>>(x, n, v);
}

static int grid_for(int64_t ntiles) {
  return (int)(ntiles < kStatBlocks ? (ntiles > 0 ? ntiles : 1) : kStatBlocks);
}

void launch_coverage(cudaStream_t st, const PatchDev* P, const float4* psf, const int2* tiles,
                     int64_t ntiles, const float* ystack, const int3 dims, Params prm, float* kap,
                     double* partials) {
  k_coverage<<<kStatBlocks, kTile, 0, st>>>(P, psf, tiles, ntiles, ystack, dims, prm, kap, partials);
}


void launch_range_finish(cudaStream_t st, double s2floor, EmDev* em) {
  k_range_finish<<<1, 1, 0, st>>>(s2floor, em);
}

void launch_forward(cudaStream_t st, const PatchDev* P, const float4* psf, const int2* tiles,
                    int64_t ntiles, const float* ystack, const float* X, const int3 dims,
                    Params prm, const float* kap, const float* p, float* e, double* partials) {
  k_forward<<<kStatBlocks, kTile, 0, st>>>(P, psf, tiles, ntiles, ystack, X, dims, prm, kap, p, e,
                                           partials);
}

void launch_em_reduce(cudaStream_t st, const double* partials, int nblk, EmDev* em) {
  k_em_reduce<<<1, 1024, 0, st>>>(partials, nblk, em);
}

void launch_em_params(cudaStream_t st, Params prm, EmDev* em) {
  k_em_params<<<1, 32, 0, st>>>(prm, em);
}

void launch_estep(cudaStream_t st, const PatchDev* P, int64_t npatch, Params prm, const EmDev* em,
                  const float* kap, const float* e, float* p, float* pbar, float* w) {
  if (npatch <= 0) return;
  k_estep<<<(unsigned)npatch, 256, 0, st>>>(P, prm, em, kap, e, p, pbar, w);
}

void launch_backproject(cudaStream_t st, const PatchDev* P, const float4* psf, const int2* tiles,
                        int64_t ntiles, const float* ystack, const int3 dims, Params prm,
                        const float* kap, const float* e, const float* p, const float* w, int init,
                        float2* AC) {
  k_backproject<<<grid_for(ntiles) * 4, kTile, 0, st>>>(P, psf, tiles, ntiles, ystack, dims, prm,
                                                        kap, e, p, w, init, AC);
}

void launch_update(cudaStream_t st, const float* X0, const float2* AC, const int3 dims, Params prm,
                   const EmDev* em, float alpha, float lambda, float* X2) {
  k_update<<<148 * 16, 256, 0, st>>>(X0, AC, dims, prm, em, alpha, lambda, X2);
}

void launch_init_fill(cudaStream_t st, const float2* AC, const int3 dims, Params prm, float* X) {
  k_init_fill<<<148 * 16, 256, 0, st>>>(AC, dims, prm, X);
}

}  // namespace pvr
