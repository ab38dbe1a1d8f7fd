// volpsf.cu — the volume-space PSF mode (PVR_PARAM_PSF_MODE = 2, "fully
// flexible and accurate PSF instead of approximated functions", reading Q34).
//
// The PSF of pixel j is evaluated at every HR voxel centre x_k inside its support instead of
// being sampled on a patch-space lattice and interpolated: with (a, b, c) the slice-frame
// components (mm) of T_s^-1(x_k) - c_j,
//   psi_jk = sinc(pi R) exp(-c^2 / (2 sw^2)),  R = |(a / dx, b / dy)| < 1,  |c| <= nsigma sw,
//   kappa_j = sum_{k in grid} psi_jk / sum_{k in Z^3} psi_jk,  W_jk = psi_jk / sum_{k in grid} psi_jk.
// One kernel, three passes: coverage (kappa and the row normaliser, once per set_transforms),
// forward (residual and EM statistics, as k_lattice_fwd<0>) and adjoint (red.global.add.v2
// of the pixel's (w p e, w p) W_jk into (A, C)). Direct form: each thread walks one pixel's
// support box (c3: ~270 voxels); positions are fp32 offsets from an integer voxel base per
// patch, the inverse map and the PSF constants come per patch from the host (fp64 -> fp32).
#include <cfloat>
#include <cmath>

#include "device_util.cuh"
#include "pvr_internal.h"

namespace pvr {

namespace {

// PSF value at slice-frame offsets (a, b, c) mm; 0 outside the support. The support test
// (R < 1, |c| <= nsigma sw) is an exact decision of the reading: a voxel within 1e-3 of its
// edge is decided again from fp64 offsets (the fp32 ones carry ~1e-5 of rounding), so the
// kernel includes the same voxels as the fp64 oracle.
__device__ __forceinline__ float vpsf(const VolPatch& V, float a, float b, float c, const double (&cd)[3],
                                      int i, int j, int l) {
  const float ra = a * V.idx, rb = b * V.idy;
  float R2 = ra * ra + rb * rb;
  if (fabsf(R2 - 1.0f) < 1e-3f || fabsf(fabsf(c) - V.cmax) < 1e-3f) {
    const double dx = i - cd[0], dy = j - cd[1], dz = l - cd[2];
    const double ad = V.Minvd[0] * dx + V.Minvd[1] * dy + V.Minvd[2] * dz;
    const double bd = V.Minvd[3] * dx + V.Minvd[4] * dy + V.Minvd[5] * dz;
    const double cd2 = V.Minvd[6] * dx + V.Minvd[7] * dy + V.Minvd[8] * dz;
    const double R2d = (ad / V.dxd) * (ad / V.dxd) + (bd / V.dyd) * (bd / V.dyd);
    if (!(sqrt(R2d) < 1.0) || fabs(cd2) > V.cmaxd) return 0.0f;
    R2 = fminf((float)R2d, 0.99999994f);
    c = (float)cd2;
  } else if (!(R2 < 1.0f) || fabsf(c) > V.cmax) {
    return 0.0f;
  }
  const float R = sqrtf(R2);
  const float s = R > 1e-4f ? sinpif(R) / (3.14159265358979f * R) : 1.0f - 1.6449341f * R2;
  return s * __expf(-c * c * V.i2s2);
}

template <int MODE>  // 0 forward, 1 coverage, 2 adjoint
__global__ void __launch_bounds__(256) k_volpsf(const VolPatch* __restrict__ VP, int64_t npatch, LatticeArgs a,
                                                const float* __restrict__ X, float* __restrict__ kap,
                                                float* __restrict__ vin, const float* __restrict__ pprev,
                                                float* __restrict__ e, double* __restrict__ partials,
                                                const float* __restrict__ w, const float* __restrict__ pv,
                                                int init, float2* __restrict__ AC) {
  double acc_s[3] = {0.0, 0.0, 0.0};
  float acc_m[2] = {-FLT_MAX, -FLT_MAX};
  const int3 n = a.n;
  for (int64_t s = blockIdx.x; s < npatch; s += gridDim.x) {
    const VolPatch V = VP[s];
    const int npix = V.sx * V.sy * V.sz;
    float ws = 1.0f, vs = 1.0f;
    if (MODE == 2) {
      ws = init ? 1.0f : w[s];
      vs = init == 2 ? w[s] : 1.0f;
      if (ws == 0.0f) continue;  // excluded patch
    }
    for (int q = threadIdx.x; q < npix; q += blockDim.x) {
      const int u = q % V.sx, v = (q / V.sx) % V.sy, z = q / (V.sx * V.sy);
      const int64_t j = V.pix0 + q;
      const float y = a.ys[V.y0off + (int64_t)z * V.HW + (int64_t)v * V.W + u];
      float rA = 0.0f, rC = 0.0f, norm = 1.0f;
      if (MODE == 0) {
        if (!(kap[j] >= a.prm.tau_obs)) {
          e[j] = 0.0f;
          continue;
        }
        norm = 1.0f / vin[j];
      } else if (MODE == 2) {
        const float k = kap[j];
        if (!(k >= a.prm.tau_obs)) continue;
        const float p = init ? 1.0f : pv[j];
        const float val = init == 1 ? y : init == 2 ? pv[j] * vs : e[j];
        rC = ws * p / vin[j];
        rA = rC * val;
        if (rA == 0.0f && rC == 0.0f) continue;
      }
      // pixel centre (index units, relative to the patch base) and its support box
      float c[3];
      double cd[3];
      int lo[3], hi[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        cd[d] = V.xcd[d] + u * V.Mud[d] + v * V.Mvd[d] + z * V.Mzd[d];
        c[d] = (float)cd[d];
        lo[d] = (int)ceilf(c[d] - V.h[d]);
        hi[d] = (int)floorf(c[d] + V.h[d]);
      }
      float all = 0.0f, in = 0.0f, acc = 0.0f;
      int cnt = 0;
      for (int l = lo[2]; l <= hi[2]; ++l) {
        const int gz = V.base[2] + l;
        const bool zin = (unsigned)gz < (unsigned)n.z;
        if (MODE != 1 && !zin) continue;
        const float dz = (float)l - c[2];
        for (int jj = lo[1]; jj <= hi[1]; ++jj) {
          const int gy = V.base[1] + jj;
          const bool yin = zin && (unsigned)gy < (unsigned)n.y;
          if (MODE != 1 && !yin) continue;
          const float dy = (float)jj - c[1];
          const int64_t row = ((int64_t)gz * n.y + gy) * a.nxp;
          for (int i = lo[0]; i <= hi[0]; ++i) {
            const int gx = V.base[0] + i;
            const bool xin = yin && (unsigned)gx < (unsigned)n.x;
            if (MODE != 1 && !xin) continue;
            const float dx = (float)i - c[0];
            const float pa = V.Minv[0] * dx + V.Minv[1] * dy + V.Minv[2] * dz;
            const float pb = V.Minv[3] * dx + V.Minv[4] * dy + V.Minv[5] * dz;
            const float pc = V.Minv[6] * dx + V.Minv[7] * dy + V.Minv[8] * dz;
            const float wt = vpsf(V, pa, pb, pc, cd, i, jj, l);
            if (wt == 0.0f) continue;
            if (MODE == 1) {
              all += wt;
              ++cnt;
              if (xin) in += wt;
            } else if (MODE == 0) {
              acc = fmaf(wt, X[row + gx], acc);
            } else {
              const float t = wt;
              asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(AC + row + gx), "f"(t * rA), "f"(t * rC)
                           : "memory");
            }
          }
        }
      }
      if (MODE == 1) {
        float k = all > 0.0f ? in / all : 0.0f;
        if (a.mask && !a.mask[j]) k = 0.0f;  // f3: masked-out pixel is never observed (Q32)
        kap[j] = k;
        vin[j] = in;
        if (k >= a.prm.tau_obs) {
          acc_s[0] += 1.0;
          acc_s[2] += (double)cnt;
        }
        if (k >= a.prm.tau_live) {
          acc_s[1] += 1.0;
          acc_m[0] = fmaxf(acc_m[0], y);
          acc_m[1] = fmaxf(acc_m[1], -y);
        }
      } else if (MODE == 0) {
        const float ev = y - acc * norm;
        e[j] = ev;
        if (kap[j] >= a.prm.tau_live) {
          const double pp = pprev[j];
          if (a.prm.det) {
            acc_s[0] += rint(pp * (double)ev * (double)ev * 16.0) * 0.0625;
            acc_s[1] += rint(pp * 16777216.0) * (1.0 / 16777216.0);
          } else {
            acc_s[0] += pp * (double)ev * (double)ev;
            acc_s[1] += pp;
          }
          acc_s[2] += 1.0;
          acc_m[0] = fmaxf(acc_m[0], ev);
          acc_m[1] = fmaxf(acc_m[1], -ev);
        }
      }
    }
  }
  if (MODE != 2) block_reduce_store<3, 2>(acc_s, acc_m, partials + (size_t)blockIdx.x * 5);
}

}  // namespace

void launch_volpsf(cudaStream_t st, int mode, const VolPatch* VP, int64_t npatch, const LatticeArgs& a,
                   const float* X, float* kap, float* vin, const float* pprev, float* e, double* partials,
                   const float* w, const float* p, int init, float2* AC) {
  if (mode == 0)
    k_volpsf<0><<<kStatBlocks, 256, 0, st>>>(VP, npatch, a, X, kap, vin, pprev, e, partials, w, p, init, AC);
  else if (mode == 1)
    k_volpsf<1><<<kStatBlocks, 256, 0, st>>>(VP, npatch, a, X, kap, vin, pprev, e, partials, w, p, init, AC);
  else
    k_volpsf<2><<<kStatBlocks, 256, 0, st>>>(VP, npatch, a, X, kap, vin, pprev, e, partials, w, p, init, AC);
}

}  // namespace pvr
