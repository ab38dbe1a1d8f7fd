// registration.cu — f1 (reading Q29): rigid
// patch-to-volume registration of every local patch against the current reconstruction X,
// maximising the cross correlation (CC) between the patch's pixels y_j and trilinear
// samples of X at the pixels' mapped centres (corners outside the grid read 0, Q6).
//
// Pose p = (tx, ty, tz [mm], rx, ry, rz [deg]) acts after the patch's transform T_s,
// rotating about the transformed patch centre c: x -> R (x - c) + c + t, R = Rz Ry Rx.
// Optimiser (same as oracle/pvro.c pvro_register): levels L = 0 .. levels-1 with steps
// 2^-L (2 mm, 4 deg); per level at most `iters` compass moves: evaluate the 12 coordinate
// moves +-step, take the best strict CC improvement (first index on ties), stop when none.
//
// One CTA per patch runs the whole search. The patch's centred intensities y - mean(y) sit
// in shared memory; thread 0 forms the 12 candidate pixel->voxel affine maps in fp64; every
// thread samples its pixels under all 12 maps (fp32 trilinear, 8 L1-cached loads each) and
// accumulates sum s, sum s^2, sum (y - mean y) s in fp32 over its few pixels; the block
// reduces in fp64 and thread 0 decides. CC = sum yc s / sqrt(sum yc^2 (sum s^2 - (sum s)^2/n)).
#include <cfloat>
#include <cmath>

#include "device_util.cuh"
#include "pvr_internal.h"

namespace pvr {

namespace {

constexpr int kRegThreads = 256;
constexpr int kCand = 12;

struct CandMap {  // voxel index g = A (u, v, z) + b
  float A[9], b[3];
};

__device__ void pose_rotation(const double* p, double R[9]) {
  double sx, cx, sy, cy, sz, cz;
  sincospi(p[3] / 180.0, &sx, &cx);
  sincospi(p[4] / 180.0, &sy, &cy);
  sincospi(p[5] / 180.0, &sz, &cz);
  // Rz Ry Rx
  const double Ryx[9] = {cy, sy * sx, sy * cx, 0.0, cx, -sx, -sy, cy * sx, cy * cx};
  const double Rz[9] = {cz, -sz, 0.0, sz, cz, 0.0, 0.0, 0.0, 1.0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[3 * i + j] = Rz[3 * i] * Ryx[j] + Rz[3 * i + 1] * Ryx[3 + j] + Rz[3 * i + 2] * Ryx[6 + j];
}

__device__ void cand_map(const RegPatch& P, const double* p, const RegArgs& a, CandMap& m) {
  double R[9];
  pose_rotation(p, R);
  const double is = 1.0 / a.s;
  for (int i = 0; i < 3; ++i) {
    m.A[3 * i + 0] = (float)((R[3 * i] * P.mu[0] + R[3 * i + 1] * P.mu[1] + R[3 * i + 2] * P.mu[2]) * is);
    m.A[3 * i + 1] = (float)((R[3 * i] * P.mv[0] + R[3 * i + 1] * P.mv[1] + R[3 * i + 2] * P.mv[2]) * is);
    m.A[3 * i + 2] = (float)((R[3 * i] * P.mz[0] + R[3 * i + 1] * P.mz[1] + R[3 * i + 2] * P.mz[2]) * is);
    const double w = R[3 * i] * (P.m0[0] - P.c[0]) + R[3 * i + 1] * (P.m0[1] - P.c[1]) +
                     R[3 * i + 2] * (P.m0[2] - P.c[2]) + P.c[i] + p[i];
    m.b[i] = (float)((w - a.o[i]) * is);
  }
}

// trilinear sample of X at voxel index g; corners outside the grid read 0 (Q6)
__device__ __forceinline__ float sample(const RegArgs& a, float gx, float gy, float gz) {
  const float fx0 = floorf(gx), fy0 = floorf(gy), fz0 = floorf(gz);
  const int i = (int)fx0, j = (int)fy0, l = (int)fz0;
  const float fx = gx - fx0, fy = gy - fy0, fz = gz - fz0;
  float v = 0.0f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int ii = i + (c & 1), jj = j + ((c >> 1) & 1), ll = l + (c >> 2);
    if ((unsigned)ii < (unsigned)a.n.x && (unsigned)jj < (unsigned)a.n.y && (unsigned)ll < (unsigned)a.n.z) {
      const float w = ((c & 1) ? fx : 1.0f - fx) * (((c >> 1) & 1) ? fy : 1.0f - fy) * ((c >> 2) ? fz : 1.0f - fz);
      v = fmaf(w, __ldg(a.X + ((size_t)ll * a.n.y + jj) * a.nxp + ii), v);
    }
  }
  return v;
}

// Block sum of NV doubles (every thread passes its NV partials; thread 0 gets the totals in out).
template <int NV>
__device__ void block_sum(double (&v)[NV], double* out, double (*sh)[NV]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[wid][k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < NV; ++k) {
      double t = 0.0;
      for (int w = 0; w < kRegThreads / 32; ++w) t += sh[w][k];
      out[k] = t;
    }
  __syncthreads();
}

__device__ __forceinline__ double cc_from(double n, double syy, double ss, double sss, double sys) {
  const double vs = sss - ss * ss / n;
  if (!(syy > 0.0) || !(vs > 0.0)) return NAN;
  return sys / sqrt(syy * vs);
}

// Evaluate NC candidate maps (in s_map) over the patch: CC per candidate into s_cc (thread 0).
template <int NC>
__device__ void eval_cands(const RegArgs& a, const RegPatch& P, const float* yc, int np, double syy,
                           const CandMap* s_map, double* s_cc, double (*sh)[3 * NC], double* s_tot) {
  float acc[3 * NC];
#pragma unroll
  for (int k = 0; k < 3 * NC; ++k) acc[k] = 0.0f;
  const int sxy = P.sx * P.sy;
  for (int j = threadIdx.x; j < np; j += kRegThreads) {
    const int z = j / sxy, r = j - z * sxy, v = r / P.sx, u = r - v * P.sx;
    const float fu = (float)u, fv = (float)v, fz = (float)z, y = yc[j];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const CandMap& m = s_map[k];
      const float gx = fmaf(m.A[0], fu, fmaf(m.A[1], fv, fmaf(m.A[2], fz, m.b[0])));
      const float gy = fmaf(m.A[3], fu, fmaf(m.A[4], fv, fmaf(m.A[5], fz, m.b[1])));
      const float gz = fmaf(m.A[6], fu, fmaf(m.A[7], fv, fmaf(m.A[8], fz, m.b[2])));
      const float sv = sample(a, gx, gy, gz);
      acc[3 * k] += sv;
      acc[3 * k + 1] = fmaf(sv, sv, acc[3 * k + 1]);
      acc[3 * k + 2] = fmaf(y, sv, acc[3 * k + 2]);
    }
  }
  double d[3 * NC];
#pragma unroll
  for (int k = 0; k < 3 * NC; ++k) d[k] = (double)acc[k];
  block_sum<3 * NC>(d, s_tot, sh);
  if (threadIdx.x == 0)
    for (int k = 0; k < NC; ++k) s_cc[k] = cc_from((double)np, syy, s_tot[3 * k], s_tot[3 * k + 1], s_tot[3 * k + 2]);
  __syncthreads();
}

// Dynamic shared memory: the patch's centred intensities (sx sy sz floats).
__global__ void __launch_bounds__(kRegThreads) k_register(RegArgs a, float* __restrict__ pose,
                                                         int32_t* __restrict__ status) {
  extern __shared__ float yc[];
  __shared__ CandMap s_map[kCand];
  __shared__ double sh[kRegThreads / 32][3 * kCand];
  __shared__ double s_tot[3 * kCand];
  __shared__ double s_cc[kCand];
  __shared__ double s_p[6], s_cur, s_syy;
  __shared__ int s_go;
  const int s = blockIdx.x;
  const RegPatch P = a.P[s];
  const int np = P.sx * P.sy * P.sz, sxy = P.sx * P.sy;
  // centred intensities
  double sy1[1] = {0.0};
  for (int j = threadIdx.x; j < np; j += kRegThreads) {
    const int z = j / sxy, r = j - z * sxy, v = r / P.sx, u = r - v * P.sx;
    const float y = a.ys[P.y0off + (int64_t)z * P.HW + (int64_t)v * P.W + u];
    yc[j] = y;
    sy1[0] += y;
  }
  {
    double (*sh1)[1] = reinterpret_cast<double (*)[1]>(sh);
    block_sum<1>(sy1, s_tot, sh1);
  }
  const float ybar = (float)(s_tot[0] / np);
  double syy[1] = {0.0};
  for (int j = threadIdx.x; j < np; j += kRegThreads) {
    const float c = yc[j] - ybar;
    yc[j] = c;
    syy[0] += (double)c * c;
  }
  {
    double (*sh1)[1] = reinterpret_cast<double (*)[1]>(sh);
    block_sum<1>(syy, s_tot, sh1);
  }
  if (threadIdx.x == 0) {
    s_syy = s_tot[0];
    for (int k = 0; k < 6; ++k) s_p[k] = 0.0;
    s_go = np >= a.min_valid;
  }
  __syncthreads();
  if (!s_go) {
    if (threadIdx.x == 0) status[s] = 0;
    return;
  }
  for (int L = 0; L < a.levels; ++L) {
    const double st_t = ldexp(2.0, -L), st_r = ldexp(4.0, -L);
    // CC at the current pose
    if (threadIdx.x == 0) cand_map(P, s_p, a, s_map[0]);
    __syncthreads();
    eval_cands<1>(a, P, yc, np, s_syy, s_map, s_cc, reinterpret_cast<double (*)[3]>(sh), s_tot);
    if (threadIdx.x == 0) {
      s_cur = s_cc[0];
      s_go = !isnan(s_cur);
      if (!s_go && L == 0) status[s] = 0;  // unregistrable: pose stays identity
    }
    __syncthreads();
    if (!s_go) {
      if (L == 0) return;
      continue;
    }
    for (int it = 0; it < a.iters; ++it) {
      if (threadIdx.x < kCand) {
        double q[6];
        for (int k = 0; k < 6; ++k) q[k] = s_p[k];
        const int c = threadIdx.x;
        q[c / 2] += ((c & 1) ? -1.0 : 1.0) * ((c / 2) < 3 ? st_t : st_r);
        cand_map(P, q, a, s_map[c]);
      }
      __syncthreads();
      eval_cands<kCand>(a, P, yc, np, s_syy, s_map, s_cc, sh, s_tot);
      if (threadIdx.x == 0) {
        double best = s_cur;
        int bk = -1;
        for (int k = 0; k < kCand; ++k)
          if (!isnan(s_cc[k]) && s_cc[k] > best) { best = s_cc[k]; bk = k; }
        s_go = bk >= 0;
        if (bk >= 0) {
          s_p[bk / 2] += ((bk & 1) ? -1.0 : 1.0) * ((bk / 2) < 3 ? st_t : st_r);
          s_cur = best;
        }
      }
      __syncthreads();
      if (!s_go) break;
    }
  }
  if (threadIdx.x == 0) {
    status[s] = 1;
    for (int k = 0; k < 6; ++k) pose[6 * s + k] = (float)s_p[k];
  }
}

// Tap: CC of (patch, pose) pairs, one CTA each (parity tests of the similarity).
__global__ void __launch_bounds__(kRegThreads) k_patch_cc(RegArgs a, const int32_t* __restrict__ which,
                                                         const float* __restrict__ poses,
                                                         double* __restrict__ out) {
  extern __shared__ float yc[];
  __shared__ CandMap s_map[1];
  __shared__ double sh[kRegThreads / 32][3];
  __shared__ double s_tot[3];
  __shared__ double s_cc[1];
  const RegPatch P = a.P[which[blockIdx.x]];
  const int np = P.sx * P.sy * P.sz, sxy = P.sx * P.sy;
  double sy1[1] = {0.0};
  for (int j = threadIdx.x; j < np; j += kRegThreads) {
    const int z = j / sxy, r = j - z * sxy, v = r / P.sx, u = r - v * P.sx;
    const float y = a.ys[P.y0off + (int64_t)z * P.HW + (int64_t)v * P.W + u];
    yc[j] = y;
    sy1[0] += y;
  }
  double (*sh1)[1] = reinterpret_cast<double (*)[1]>(sh);
  block_sum<1>(sy1, s_tot, sh1);
  const float ybar = (float)(s_tot[0] / np);
  double syy[1] = {0.0};
  for (int j = threadIdx.x; j < np; j += kRegThreads) {
    const float c = yc[j] - ybar;
    yc[j] = c;
    syy[0] += (double)c * c;
  }
  block_sum<1>(syy, s_tot, sh1);
  const double Syy = s_tot[0];
  if (threadIdx.x == 0) {
    double q[6];
    for (int k = 0; k < 6; ++k) q[k] = poses[6 * blockIdx.x + k];
    cand_map(P, q, a, s_map[0]);
  }
  __syncthreads();
  eval_cands<1>(a, P, yc, np, Syy, s_map, s_cc, sh, s_tot);
  if (threadIdx.x == 0) out[blockIdx.x] = np >= a.min_valid ? s_cc[0] : NAN;
}

}  // namespace

void launch_register(cudaStream_t st, const RegArgs& a, int nloc, int max_pix, float* pose, int32_t* status) {
  if (nloc <= 0) return;
  const int smem = max_pix * 4;
  cudaFuncSetAttribute(k_register, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_register<<<nloc, kRegThreads, smem, st>>>(a, pose, status);
}

void launch_patch_cc(cudaStream_t st, const RegArgs& a, int n, int max_pix, const int32_t* which,
                     const float* poses, double* out) {
  if (n <= 0) return;
  const int smem = max_pix * 4;
  cudaFuncSetAttribute(k_patch_cc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_patch_cc<<<n, kRegThreads, smem, st>>>(a, which, poses, out);
}

}  // namespace pvr
