// lattice.cu — the two hot loops of the SR iteration on the factorised PSF lattice.
//
// SURVEY.md §8(a) rows a1 (forward simulate, Eq. 1 P:53-58 with the P:158-160 PSF) and
// a5 (adjoint backprojection, P:185 / P:232 "pixel-volume"), plus the coverage kappa.
//
// The PSF of a stack is separable, psi(a,b,c) = ip(a,b) tp(c) (sinc in-plane times
// the slice profile), and its in-plane lattice is commensurate with the pixel pitch (reading
// Q5: pixel u's sample a sits at fine index U = n_u u + a). So the samples of all pixels of a
// patch slice lie on one affine lattice (U, V, c), and
//   forward:   yhat_j = kappa_j^-1 sum_{a,b} ip(a,b) T(n_u u + a, n_v v + b),
//              T(U, V) = sum_c tp(c) trilerp(X, x(U, V, c))
//   adjoint:   A += sum_{U,V,c} tp(c) L_A(U, V) splat(x(U, V, c)),
//              L_A(U, V) = sum_{(a,b): U = n_u u + a} ip(a,b) w p_j e_j / kappa_j
// which is exactly W (resp. W^T) of the direct sum over (pixel, sample), summed in another
// order; each lattice point is interpolated / splatted once instead of once per pixel that
// shares it (c3: 2.9e9 lattice points instead of 6.5e9 samples per pass).
//
// Backprojection accumulates a group's splats in a shared-memory fp32 (A, C) tile of the
// group's voxel bounding box, then flushes it with one coalesced red.global.add.v4.f32 per
// voxel pair. (A per-group int32 fixed-point tile was tried: native
// ATOMS.ADD is ~3x faster than the fp32 CAS loop, but the tile's dynamic range -- small-kappa
// pixels, trilinear tails -- cost ~4e-4 relative L2 on X, over the 1e-4 parity bar.)
#include <cfloat>
#include <cmath>

#include "device_util.cuh"
#include "pvr_internal.h"

namespace pvr {

namespace {

constexpr int kMaxIp = 81;   // (2 ru + 1)(2 rv + 1) <= 81 (n <= 5)
constexpr int kMaxTp = 256;  // 2 cmax + 1

struct Axis {
  int i0, i1;
  float w0, w1;
};

// Trilinear axis weights at continuous index off + r (grid [0, n)), with r a small fp32 local
// coordinate and off an integer origin (keeps the fractional part exact to ~1e-6 voxel).
// Out-of-grid corners get weight 0 and an in-grid (clamped) index (reading Q6: dropped, not
// redistributed).
__device__ __forceinline__ Axis axis_weights(float r, int off, int n) {
  float fl;
  const int i = mfloor(r, fl) + off;
  const float f = r - fl;
  Axis a;
  a.w0 = (i >= 0 && i < n) ? 1.0f - f : 0.0f;
  a.w1 = (i + 1 >= 0 && i + 1 < n) ? f : 0.0f;
  a.i0 = min(max(i, 0), n - 1);
  a.i1 = min(max(i + 1, 0), n - 1);
  return a;
}

// Member geometry shared by both kernels.
struct MemberGeom {
  float qa[3], qb[3], qc[3];
  int nu, nv, ru, rv, cmax, ntp, ip0, tp0;
};

// Voxel index of lattice point (U0, V0, c0) of slice z, formed in fp64 and split into an
// integer base and an fp32 fraction; the kernels then add small fp32 lattice offsets.
__device__ __forceinline__ void lattice_origin(const PatchDev& pt, int z, int U0, int V0, int c0,
                                               int (&base)[3], float (&frac)[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x = pt.t0d[d] + z * pt.Mzd[d] + U0 * pt.Qad[d] + V0 * pt.Qbd[d] + c0 * pt.Qcd[d];
    const double f = floor(x);
    base[d] = (int)f;
    frac[d] = (float)(x - f);
  }
}

__device__ __forceinline__ MemberGeom member_geom(const LatticeArgs& a, const PatchDev& pt, int z) {
  MemberGeom g;
  const StackPsf ps = a.psf[pt.stack];
  (void)z;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g.qa[d] = pt.Qa[d];
    g.qb[d] = pt.Qb[d];
    g.qc[d] = pt.Qc[d];
  }
  g.nu = ps.nu; g.nv = ps.nv; g.ru = ps.ru; g.rv = ps.rv; g.cmax = ps.cmax;
  g.ntp = 2 * ps.cmax + 1; g.ip0 = ps.ip0; g.tp0 = ps.tp0;
  return g;
}

// ------------------------------------------------------------------------------------------
// Forward (MODE 0) and coverage (MODE 1).
//   MODE 0: out = e (residual, 0 if unobserved); stats {sum p e^2, sum p, n_live | max e, -min e}
//   MODE 1: out = kappa;                         stats {n_obs, n_live, samples | max y, -min y}
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_lattice_fwd(LatticeArgs a, const float* __restrict__ X,
                                                          const float* __restrict__ kap,
                                                          const float* __restrict__ pprev,
                                                          float* __restrict__ out,
                                                          double* __restrict__ partials) {
  extern __shared__ float sT[];  // lattice values T(U, V) of the current member
  __shared__ float s_ip[kMaxIp], s_tp[kMaxTp];
  double acc_s[3] = {0.0, 0.0, 0.0};
  float acc_m[2] = {-FLT_MAX, -FLT_MAX};
  const int3 n = a.n;
  const size_t nxy = (size_t)n.x * n.y;

  for (int g = blockIdx.x; g < a.ngroups; g += gridDim.x) {
    const GroupDev G = a.grp[g];
    for (int mi = G.m0; mi < G.m0 + G.nm; ++mi) {
      const MemberDev m = a.mem[mi];
      const PatchDev& pt = a.P[m.patch];
      const MemberGeom mg = member_geom(a, pt, m.z);
      const int nip = (2 * mg.ru + 1) * (2 * mg.rv + 1);
      __syncthreads();  // previous member's readers of sT / tables are done
      for (int i = threadIdx.x; i < nip; i += kThreads) s_ip[i] = a.tab[mg.ip0 + i];
      for (int i = threadIdx.x; i < mg.ntp; i += kThreads) s_tp[i] = a.tab[mg.tp0 + i];
      // lattice points needed by the tile's pixels: U in [nu u0 - ru, nu (u0 + tu - 1) + ru]
      const int LU = mg.nu * (m.tu - 1) + 2 * mg.ru + 1;
      const int LV = mg.nv * (m.tv - 1) + 2 * mg.rv + 1;
      const int U0 = mg.nu * m.u0 - mg.ru, V0 = mg.nv * m.v0 - mg.rv;
      int ob[3];
      float of[3];
      lattice_origin(pt, m.z, U0, V0, -mg.cmax, ob, of);
      const int bx = ob[0], by = ob[1], bz = ob[2];
      __syncthreads();
      for (int i = threadIdx.x; i < LU * LV; i += kThreads) {
        const float U = (float)(i % LU), V = (float)(i / LU);
        float rx = of[0] + U * mg.qa[0] + V * mg.qb[0];
        float ry = of[1] + U * mg.qa[1] + V * mg.qb[1];
        float rz = of[2] + U * mg.qa[2] + V * mg.qb[2];
        float acc = 0.0f;
        for (int c = 0; c < mg.ntp; ++c) {
          const Axis ax = axis_weights(rx, bx, n.x);
          const Axis ay = axis_weights(ry, by, n.y);
          const Axis az = axis_weights(rz, bz, n.z);
          float v;
          if (MODE == 1) {
            v = (ax.w0 + ax.w1) * (ay.w0 + ay.w1) * (az.w0 + az.w1);
          } else {
            const float* p00 = X + az.i0 * nxy + (size_t)ay.i0 * n.x;
            const float* p01 = X + az.i0 * nxy + (size_t)ay.i1 * n.x;
            const float* p10 = X + az.i1 * nxy + (size_t)ay.i0 * n.x;
            const float* p11 = X + az.i1 * nxy + (size_t)ay.i1 * n.x;
            const float c00 = ax.w0 * __ldg(p00 + ax.i0) + ax.w1 * __ldg(p00 + ax.i1);
            const float c01 = ax.w0 * __ldg(p01 + ax.i0) + ax.w1 * __ldg(p01 + ax.i1);
            const float c10 = ax.w0 * __ldg(p10 + ax.i0) + ax.w1 * __ldg(p10 + ax.i1);
            const float c11 = ax.w0 * __ldg(p11 + ax.i0) + ax.w1 * __ldg(p11 + ax.i1);
            v = az.w0 * (ay.w0 * c00 + ay.w1 * c01) + az.w1 * (ay.w0 * c10 + ay.w1 * c11);
          }
          acc += s_tp[c] * v;
          rx += mg.qc[0];
          ry += mg.qc[1];
          rz += mg.qc[2];
        }
        sT[i] = acc;
      }
      __syncthreads();
      if (threadIdx.x < m.tu * m.tv) {
        const int du = threadIdx.x % m.tu, dv = threadIdx.x / m.tu;
        const int u = m.u0 + du, v = m.v0 + dv;
        const int w2 = 2 * mg.ru + 1;
        float s = 0.0f;
        for (int b = 0; b <= 2 * mg.rv; ++b) {
          const float* row = sT + (mg.nv * dv + b) * LU + mg.nu * du;
          for (int aa = 0; aa < w2; ++aa) s += s_ip[b * w2 + aa] * row[aa];
        }
        const int64_t j = pt.pix0 + ((int64_t)m.z * pt.sy + v) * pt.sx + u;
        const float y = a.ys[pt.y0off + (int64_t)m.z * pt.HW + (int64_t)v * pt.W + u];
        if (MODE == 1) {
          out[j] = s;
          if (s >= a.prm.tau_obs) {
            acc_s[0] += 1.0;
            acc_s[2] += (double)pt.S;
          }
          if (s >= a.prm.tau_live) {
            acc_s[1] += 1.0;
            acc_m[0] = fmaxf(acc_m[0], y);
            acc_m[1] = fmaxf(acc_m[1], -y);
          }
        } else {
          const float k = kap[j];
          float ev = 0.0f;
          if (k >= a.prm.tau_obs) {
            ev = y - s / k;
            if (k >= a.prm.tau_live) {
              const double pp = pprev[j];
              acc_s[0] += pp * (double)ev * (double)ev;
              acc_s[1] += pp;
              acc_s[2] += 1.0;
              acc_m[0] = fmaxf(acc_m[0], ev);
              acc_m[1] = fmaxf(acc_m[1], -ev);
            }
          }
          out[j] = ev;
        }
      }
    }
  }
  block_reduce_store<3, 2>(acc_s, acc_m, partials + (size_t)blockIdx.x * 5);
}

// ------------------------------------------------------------------------------------------
// Backprojection (a5) / initial backprojection (init = 1: p = w = 1, e := y).
struct Owned {  // a member's owned lattice range and the pixel range it reads
  int Ulo, Uhi, Vlo, Vhi;   // owned fine-lattice range [lo, hi)
  int plu, phu, plv, phv;   // pixel range [pl, ph] feeding it (clipped to the patch)
};

__device__ __forceinline__ Owned owned_range(const MemberDev& m, const PatchDev& pt, const MemberGeom& g) {
  // tiles partition U in [-ru, nu (sx - 1) + ru]: a tile owns [nu u0 - ru, nu (u0 + tu) - ru),
  // the last one up to nu (sx - 1) + ru inclusive
  Owned o;
  o.Ulo = g.nu * m.u0 - g.ru;
  o.Uhi = (m.u0 + m.tu >= pt.sx) ? g.nu * (pt.sx - 1) + g.ru + 1 : g.nu * (m.u0 + m.tu) - g.ru;
  o.Vlo = g.nv * m.v0 - g.rv;
  o.Vhi = (m.v0 + m.tv >= pt.sy) ? g.nv * (pt.sy - 1) + g.rv + 1 : g.nv * (m.v0 + m.tv) - g.rv;
  o.plu = max(0, -floor_div(-(o.Ulo - g.ru), g.nu));
  o.phu = min(pt.sx - 1, floor_div(o.Uhi - 1 + g.ru, g.nu));
  o.plv = max(0, -floor_div(-(o.Vlo - g.rv), g.nv));
  o.phv = min(pt.sy - 1, floor_div(o.Vhi - 1 + g.rv, g.nv));
  return o;
}

__global__ void __launch_bounds__(kThreads) k_lattice_bp(LatticeArgs a, int tile_words,
                                                         const float* __restrict__ kap,
                                                         const float* __restrict__ e,
                                                         const float* __restrict__ p,
                                                         const float* __restrict__ w, int init,
                                                         float2* __restrict__ AC) {
  extern __shared__ float4 smem4[];
  float* acc = reinterpret_cast<float*>(smem4);                   // [tile_words] (A, C) fp32
  float2* R = reinterpret_cast<float2*>(acc + tile_words);        // per-pixel (rA, rC)
  __shared__ float s_ip[kMaxIp], s_tp[kMaxTp];
  __shared__ float s_red[2][32];
  __shared__ float s_scale[2];
  const int3 n = a.n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  for (int g = blockIdx.x; g < a.ngroups; g += gridDim.x) {
    const GroupDev G = a.grp[g];
    const bool tiled = G.dim[0] > 0;
    const int dx = G.dim[0], dy = G.dim[1], dz = G.dim[2];
    const int nvox = dx * dy * dz;
    __syncthreads();  // previous group's flush is done with acc / R / tables
    // ---- phase A: per-pixel (rA, rC) of every member into R; group maxima for the scale
    float mA = 0.0f, mC = 0.0f;
    int roff = 0;
    for (int mi = G.m0; mi < G.m0 + G.nm; ++mi) {
      const MemberDev m = a.mem[mi];
      const PatchDev& pt = a.P[m.patch];
      const MemberGeom mg = member_geom(a, pt, m.z);
      const Owned o = owned_range(m, pt, mg);
      const int rw = o.phu - o.plu + 1, rh = o.phv - o.plv + 1;
      const float ws = init ? 1.0f : w[m.patch];
      for (int i = threadIdx.x; i < rw * rh; i += kThreads) {
        const int u = o.plu + i % rw, v = o.plv + i / rw;
        const int64_t j = pt.pix0 + ((int64_t)m.z * pt.sy + v) * pt.sx + u;
        float rA = 0.0f, rC = 0.0f;
        const float k = kap[j];
        if (ws != 0.0f && k >= a.prm.tau_obs) {
          const float pv = init ? 1.0f : p[j];
          const float val = init ? a.ys[pt.y0off + (int64_t)m.z * pt.HW + (int64_t)v * pt.W + u] : e[j];
          rC = ws * pv / k;
          rA = rC * val;
        }
        R[roff + i] = make_float2(rA, rC);
        mA = fmaxf(mA, fabsf(rA));
        mC = fmaxf(mC, rC);
      }
      roff += rw * rh;
    }
    mA = warp_max(mA);
    mC = warp_max(mC);
    if (lane == 0) {
      s_red[0][wid] = mA;
      s_red[1][wid] = mC;
    }
    {  // PSF tables of the group's stack (all members share it) and the tile reset
      const PatchDev& pt0 = a.P[a.mem[G.m0].patch];
      const MemberGeom mg = member_geom(a, pt0, 0);
      const int nip = (2 * mg.ru + 1) * (2 * mg.rv + 1);
      for (int i = threadIdx.x; i < nip; i += kThreads) s_ip[i] = a.tab[mg.ip0 + i];
      for (int i = threadIdx.x; i < mg.ntp; i += kThreads) s_tp[i] = a.tab[mg.tp0 + i];
      if (tiled)
        for (int i = threadIdx.x; i < (nvox >> 1); i += kThreads) smem4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float xA = 0.0f, xC = 0.0f;
      for (int i = 0; i < (kThreads >> 5); ++i) {
        xA = fmaxf(xA, s_red[0][i]);
        xC = fmaxf(xC, s_red[1][i]);
      }
      s_scale[0] = xA;
      s_scale[1] = xC;
    }
    __syncthreads();
    if (s_scale[0] == 0.0f && s_scale[1] == 0.0f) continue;  // nothing to splat (excluded patches)
    // ---- phase B: splat every owned lattice point of every member
    roff = 0;
    for (int mi = G.m0; mi < G.m0 + G.nm; ++mi) {
      const MemberDev m = a.mem[mi];
      const PatchDev& pt = a.P[m.patch];
      const MemberGeom mg = member_geom(a, pt, m.z);
      const Owned o = owned_range(m, pt, mg);
      const int rw = o.phu - o.plu + 1, rh = o.phv - o.plv + 1;
      const int nU = o.Uhi - o.Ulo, nV = o.Vhi - o.Vlo;
      const int w2 = 2 * mg.ru + 1;
      // local origin: tiled -> relative to the group bbox; global -> relative to voxel 0
      int ob[3];
      float of[3];
      lattice_origin(pt, m.z, o.Ulo, o.Vlo, -mg.cmax, ob, of);
      const int ox = ob[0] - (tiled ? G.lo[0] : 0);
      const int oy = ob[1] - (tiled ? G.lo[1] : 0);
      const int oz = ob[2] - (tiled ? G.lo[2] : 0);
      // lanes of a warp take lattice columns P apart (P coprime to nU) so that their
      // trilinear corners do not collide in the shared atomics
      int P = 5;
      while (nU % P == 0) P += 2;
      const int ex = tiled ? dx : n.x, ey = tiled ? dy : n.y, ez = tiled ? dz : n.z;
      for (int i = threadIdx.x; i < nU * nV; i += kThreads) {
        const int iu = ((i % nU) * P) % nU, iv = i / nU;
        const int U = o.Ulo + iu, V = o.Vlo + iv;
        float LA = 0.0f, LC = 0.0f;
        for (int b = -mg.rv; b <= mg.rv; ++b) {
          const int vn = V - b;
          if (vn < mg.nv * o.plv || vn > mg.nv * o.phv || (vn - mg.nv * o.plv) % mg.nv) continue;
          const int v = vn / mg.nv;
          for (int aa = -mg.ru; aa <= mg.ru; ++aa) {
            const int un = U - aa;
            if (un < mg.nu * o.plu || un > mg.nu * o.phu || (un - mg.nu * o.plu) % mg.nu) continue;
            const int u = un / mg.nu;
            const float wt = s_ip[(b + mg.rv) * w2 + (aa + mg.ru)];
            const float2 r = R[roff + (v - o.plv) * rw + (u - o.plu)];
            LA += wt * r.x;
            LC += wt * r.y;
          }
        }
        if (LA == 0.0f && LC == 0.0f) continue;
        const float fU = (float)iu, fV = (float)iv;
        float rx = of[0] + fU * mg.qa[0] + fV * mg.qb[0];
        float ry = of[1] + fU * mg.qa[1] + fV * mg.qb[1];
        float rz = of[2] + fU * mg.qa[2] + fV * mg.qb[2];
        for (int c = 0; c < mg.ntp; ++c) {
          const float t = s_tp[c];
          const float vA = LA * t, vC = LC * t;
          // validity against the grid: in tiled mode the bbox is clipped to the grid and
          // contains every in-grid corner, so "in [0, e)" is the same test
          const Axis ax = axis_weights(rx, ox, ex);
          const Axis ay = axis_weights(ry, oy, ey);
          const Axis az = axis_weights(rz, oz, ez);
          if (tiled) {
            const int r00 = (az.i0 * dy + ay.i0) * dx, r01 = (az.i0 * dy + ay.i1) * dx;
            const int r10 = (az.i1 * dy + ay.i0) * dx, r11 = (az.i1 * dy + ay.i1) * dx;
            const float w00 = az.w0 * ay.w0, w01 = az.w0 * ay.w1, w10 = az.w1 * ay.w0, w11 = az.w1 * ay.w1;
            const float a0 = vA * ax.w0, a1 = vA * ax.w1, c0 = vC * ax.w0, c1 = vC * ax.w1;
#define PVR_SPLAT(ROW, WYZ)                                          \
  {                                                                  \
    float* q0 = acc + 2 * ((ROW) + ax.i0);                           \
    float* q1 = acc + 2 * ((ROW) + ax.i1);                           \
    atomicAdd(q0, a0 * (WYZ));                                       \
    atomicAdd(q0 + 1, c0 * (WYZ));                                   \
    atomicAdd(q1, a1 * (WYZ));                                       \
    atomicAdd(q1 + 1, c1 * (WYZ));                                   \
  }
            PVR_SPLAT(r00, w00)
            PVR_SPLAT(r01, w01)
            PVR_SPLAT(r10, w10)
            PVR_SPLAT(r11, w11)
#undef PVR_SPLAT
          } else {
            const size_t sy = (size_t)a.nxp, sz = (size_t)a.nxp * n.y;
            const float wz[2] = {az.w0, az.w1}, wy[2] = {ay.w0, ay.w1}, wx[2] = {ax.w0, ax.w1};
            const int iz[2] = {az.i0, az.i1}, iy[2] = {ay.i0, ay.i1}, ix[2] = {ax.i0, ax.i1};
#pragma unroll
            for (int cz = 0; cz < 2; ++cz)
#pragma unroll
              for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                for (int cx = 0; cx < 2; ++cx) {
                  const float wt = wz[cz] * wy[cy] * wx[cx];
                  if (wt != 0.0f) red_v2(AC + iz[cz] * sz + iy[cy] * sy + ix[cx], vA * wt, vC * wt);
                }
          }
          rx += mg.qc[0];
          ry += mg.qc[1];
          rz += mg.qc[2];
        }
      }
      roff += rw * rh;
    }
    if (!tiled) continue;
    __syncthreads();
    // ---- phase C: flush the tile, one red.v4 per (even, odd) voxel pair along x
    const int hx = dx >> 1;
    for (int i = threadIdx.x; i < hx * dy * dz; i += kThreads) {
      const int px = i % hx, rest = i / hx;
      const int yy = rest % dy, zz = rest / dy;
      const float4 q = smem4[(zz * dy + yy) * hx + px];
      if (q.x == 0.0f && q.y == 0.0f && q.z == 0.0f && q.w == 0.0f) continue;
      float2* dst = AC + ((size_t)(G.lo[2] + zz) * n.y + (G.lo[1] + yy)) * a.nxp + G.lo[0] + 2 * px;
      red_v4(dst, q.x, q.y, q.z, q.w);
    }
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------
static void configure() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_lattice_bp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_lattice_fwd<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k_lattice_fwd<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  done = true;
}

// t_bytes: shared T buffer of one member (LU x LV floats, from the plan)
void launch_coverage(cudaStream_t st, const LatticeArgs& a, int t_bytes, float* kap, double* partials) {
  configure();
  k_lattice_fwd<1><<<kStatBlocks, kThreads, t_bytes, st>>>(a, nullptr, nullptr, nullptr, kap, partials);
}

void launch_forward(cudaStream_t st, const LatticeArgs& a, int t_bytes, const float* X, const float* kap,
                    const float* p, float* e, double* partials) {
  configure();
  k_lattice_fwd<0><<<kStatBlocks, kThreads, t_bytes, st>>>(a, X, kap, p, e, partials);
}

void launch_backproject(cudaStream_t st, const LatticeArgs& a, int tile_bytes, int r_bytes,
                        const float* kap, const float* e, const float* p, const float* w, int init,
                        float2* AC) {
  if (a.ngroups <= 0) return;
  configure();
  const int smem = tile_bytes + r_bytes;
  const int grid = a.ngroups < 148 * 16 ? a.ngroups : 148 * 16;
  k_lattice_bp<<<grid, kThreads, smem, st>>>(a, tile_bytes / 4, kap, e, p, w, init, AC);
}

}  // namespace pvr
