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
// order: each lattice point is interpolated / splatted once instead of once per pixel sharing
// it (c3: 2.9e9 lattice points instead of 6.5e9 samples per pass).
//
// Forward: one CTA per group (tiles of overlapping patches over the same stack pixels). The
// group's voxel footprint of X is staged once in shared memory, zero outside the grid, so the
// inner loop is 8 shared loads + 7 lerps with 32-bit addressing and no bounds logic (dropping
// out-of-grid corners == reading zeros there). Coverage is the same pass over the grid's
// indicator function, interpolated analytically (separable tents, no tile). The per-member
// constants of both (and of the backprojection) are built once per geometry by k_fwd_table /
// k_bp_table (one warp segment per group) and copied by each group's CTA.
//
// Backprojection: one CTA per group. Splats accumulate in a shared tile of the group's voxel
// bounding box as int32 fixed point on a per-group grid (one word per quantity on a 2^-21
// grid for interior groups; exact hi/lo word pairs, 2^-41, for groups that can reach the rim
// of the coverage or carry 1/kappa-amplified terms, and in the init / rigidity passes) with
// native ATOMS.ADD: fp32 shared atomics are CAS loops on sm_100a (5-10x slower under
// contention, profiles/r01_ubench_atomics2.txt). Precision and thresholds: DESIGN.md §7. Each
// thread walks a lattice line along its dominant axis with a two-plane register window. The
// tile is flushed with coalesced red.global.add.v4.f32 (voxel pairs), skipping cells outside
// the grid. Persistent CTAs claim groups dynamically (the next claim overlaps the splat).
#include <cfloat>
#include <cmath>
#include <mutex>
#include <type_traits>

#include "device_util.cuh"
#include "pvr_internal.h"

namespace pvr {

namespace {

constexpr int kMaxIp = 81;   // (2 ru + 1)(2 rv + 1) <= 81 (n <= 5)
constexpr int kMaxTp = 256;  // 2 cmax + 1
constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;
constexpr float kLoScale = 1048576.0f;  // 2^20: resolution of the lo word in hi units
constexpr float kTermMax = 1048576.0f;  // 2^20: largest splat term in hi units
constexpr float kWindowMax = 4194304.0f;  // 2^22: largest window plane sum (exact magic rounding)

// Member geometry shared by both kernels.
struct MemberGeom {
  float qa[3], qb[3], qc[3];
  int nu, nv, ru, rv, cmax, ntp, ip0, tp0;
};

__device__ __forceinline__ MemberGeom member_geom(const LatticeArgs& a, const PatchDev& pt) {
  MemberGeom g;
  const StackPsf ps = a.psf[pt.stack];
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

// Voxel index of lattice point (U0, V0, c0) of slice z, formed in fp64 and split into an
// integer part relative to `lo` and an fp32 fraction; kernels then add small fp32 offsets.
__device__ __forceinline__ void lattice_origin(const PatchDev& pt, int z, int U0, int V0, int c0,
                                               const int32_t* lo, int (&base)[3], float (&frac)[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x = pt.t0d[d] + z * pt.Mzd[d] + U0 * pt.Qad[d] + V0 * pt.Qbd[d] + c0 * pt.Qcd[d];
    const double f = floor(x);
    base[d] = (int)f - lo[d];
    frac[d] = (float)(x - f);
  }
}

// ------------------------------------------------------------------------------------------
// Forward (MODE 0) and coverage (MODE 1).
//   MODE 0: out = e (residual, 0 if unobserved); stats {sum p e^2, sum p, n_live | max e, -min e}
//   MODE 1: out = kappa;                         stats {n_obs, n_live, samples | max y, -min y}
// One CTA per group: stage the group's X tile, then one balanced pass over the lattice points
// of all members (T values into shared memory), then one pass over all their pixels.
// Dynamic shared memory: [t_floats] lattice values T of all members, then the X tile.
constexpr int kMaxMembers = 16;
#ifndef PVR_FWD_UNROLL
#define PVR_FWD_UNROLL 4
#endif
constexpr int kFwdUnroll = PVR_FWD_UNROLL;  // samples per iteration of the forward's c loop
constexpr int kFwdNtpFixed = 15;            // through-plane samples of the unrolled forward path

// Per-member constants of the forward / coverage, in global memory (k_fwd_table: once per
// geometry) and copied into shared memory by each group's CTA.
struct __align__(16) FwdMember {
  float of[3], qa[3], qb[3], qc[3];
  int ob[3];
  int LU, LV, t0, p0;  // lattice extent, offset into sT, first pixel index in the group order
  int patch, z, u0, v0, tu, tv;
  int sh;              // lattice point order (forward; coverage uses rows): strips of 2^sh U
                       // columns, V-major inside (sh = 2 axial-like, 3 x-normal), 0 = rows
  int skew;            // x-normal members (forward): the c loop of point (U, V) starts at phase V & 3
  float inv_LU, inv_s4;  // 1 / LU, 1 / (2^sh LV)
  float inv_tu;          // 1 / tu (pixel index decode)
  int pad[2];
};
static_assert(sizeof(FwdMember) % 16 == 0, "FwdMember is copied as int4");

struct __align__(16) FwdHdr {  // per-group totals and the group's stack PSF constants
  int nt, np;          // lattice points / pixels of all members
  int nu, nv, ru, rv, ip0, tp0, cmax;
  float tpsum;         // sum of tp over a line's samples (coverage: a line inside the grid)
  int pad[2];
};

#ifndef PVR_FWD_DYN
#define PVR_FWD_DYN 1
#endif

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_lattice_fwd(LatticeArgs a, int t_floats,
                                                          const char* __restrict__ tmaps,
                                                          const float* __restrict__ kap,
                                                          const float* __restrict__ pprev,
                                                          float* __restrict__ out,
                                                          double* __restrict__ partials,
                                                          int* __restrict__ next) {
  extern __shared__ __align__(128) float4 fsm4[];
  float* sT = reinterpret_cast<float*>(fsm4);
  float* sX = sT + t_floats;  // t_floats is a multiple of 32: 128-byte aligned TMA slabs
  __shared__ float s_ip[kMaxIp];
  __shared__ float2 s_tpc[2 * kMaxTp + 4];  // (tp(i mod ntp), i mod ntp): phase-shifted c loops
  __shared__ FwdMember sm[kMaxMembers];
  __shared__ __align__(8) uint64_t s_bar;  // TMA completion barrier (MODE 0)
  double acc_s[3] = {0.0, 0.0, 0.0};
  float acc_m[2] = {-FLT_MAX, -FLT_MAX};
  const int3 n = a.n;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar);
  const unsigned sX0 = (unsigned)__cvta_generic_to_shared(sX);
  if (MODE == 0 && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned phase = 0;
  // X footprint of group gg by TMA (thread 0): one 3D tensor copy (box dx x dy x 1) per z
  // slab, zero fill outside the grid, completion on the mbarrier. Issued for the CTA's first
  // group here and for each next group as soon as the current one's lattice pass is done (the
  // pixel pass does not read sX), so the copy overlaps the pixel pass.
  auto issue_tma = [&](int gg) {
    const GroupDev Gt = a.grp[gg];
    const int tdx = Gt.dim[0], tdy = Gt.dim[1], tdz = Gt.dim[2], tdxy = (tdx * tdy + 31) & ~31;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // sX reads -> async writes
    const char* tm = tmaps + 128 * Gt.tmap;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(tdz * tdx * tdy * 4)
                 : "memory");
    for (int z = 0; z < tdz; ++z)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sX0 + 4u * (unsigned)(z * tdxy)),
          "l"(tm), "r"(Gt.lo[0]), "r"(Gt.lo[1]), "r"(Gt.lo[2] + z), "r"(bar)
          : "memory");
  };
  // PVR_FWD_DYN: thread 0 claims each CTA's next group from a launch counter (reset before the
  // launch; MODE 0: when it issues that group's TMA copy); groups differ in cost (coverage:
  // interior groups skip the lattice pass), so a static stride leaves SMs idle at the end.
  // s_gn is published by the barrier at the loop top.
  constexpr bool kDyn = PVR_FWD_DYN;
  __shared__ int s_gn;
  if (threadIdx.x == 0) {
    s_gn = kDyn ? atomicAdd(next, 1) : (int)blockIdx.x;
    if (MODE == 0 && s_gn < a.ngroups) issue_tma(s_gn);
  }

  for (int g = blockIdx.x;; g += gridDim.x) {
    if (kDyn) {
      __syncthreads();
      g = s_gn;
    }
    if (g >= a.ngroups) break;
    const GroupDev G = a.grp[g];
    // tile: rows of pitch dx (the group's TMA box width), z slabs of dxy floats (128-byte
    // aligned); the box covers the group footprint (engine.cu: size_groups)
    const int dx = G.dim[0], dy = G.dim[1], dz = G.dim[2], dxy = (dx * dy + 31) & ~31;
    __syncthreads();  // the previous group's readers of sT / tables / sm are done
    // member rows and the stack's PSF tables (k_fwd_table)
    const FwdHdr H = reinterpret_cast<const FwdHdr*>(static_cast<const char*>(a.ftab) + a.fgoff)[g];
    {
      const int4* src = reinterpret_cast<const int4*>(static_cast<const FwdMember*>(a.ftab) + G.m0);
      int4* dst = reinterpret_cast<int4*>(sm);
      const int nq = G.nm * (int)(sizeof(FwdMember) / 16);
      for (int i = threadIdx.x; i < nq; i += kThreads) dst[i] = __ldg(src + i);
      const int nip = (2 * H.ru + 1) * (2 * H.rv + 1);
      for (int i = threadIdx.x; i < nip; i += kThreads) s_ip[i] = a.tab[H.ip0 + i];
      const int nt = 2 * H.cmax + 1;
      for (int i = threadIdx.x; i < 2 * nt + 4; i += kThreads) {
        const int c = i % nt;
        s_tpc[i] = make_float2(a.tab[H.tp0 + c], (float)c);
      }
    }
    if (MODE == 0) {  // the X tile has landed
      unsigned done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
      phase ^= 1u;
    }
    __syncthreads();
    const int ntp = 2 * H.cmax + 1;
    // lattice points of all members: T(U, V) = sum_c tp(c) trilerp(X, x(U, V, c))
    const bool skip = MODE == 1 && G.interior;
    float tpr[kFwdNtpFixed];  // the group's tp values when ntp == kFwdNtpFixed (forward)
#pragma unroll
    for (int c = 0; c < kFwdNtpFixed; ++c) tpr[c] = MODE == 0 ? s_tpc[c].x : 0.0f;
    int k = 0;  // the member of lattice point / pixel i (i only grows)
    for (int i = skip ? H.nt : threadIdx.x; i < H.nt; i += kThreads) {
      while (k + 1 < G.nm && i >= sm[k + 1].t0) ++k;
      const FwdMember& f = sm[k];
      const int li = i - f.t0;
      int iu, iv;
      if (MODE == 0 && f.sh) {  // strip sidx of 2^sh U columns (the last one narrower), V-major inside
        const int sw = 1 << f.sh;
        const int sidx = (int)(((float)li + 0.5f) * f.inv_s4);
        const int r = li - sidx * sw * f.LV;
        const int ws = min(sw, f.LU - sw * sidx);
        iv = ws == sw ? (r >> f.sh) : (int)(((float)r + 0.5f) / (float)ws);
        iu = sw * sidx + (r - iv * ws);
      } else {
        iv = (int)(((float)li + 0.5f) * f.inv_LU);
        iu = li - iv * f.LU;
      }
      const float U = (float)iu, V = (float)iv;
      float rx = f.of[0] + U * f.qa[0] + V * f.qb[0];
      float ry = f.of[1] + U * f.qa[1] + V * f.qb[1];
      float rz = f.of[2] + U * f.qa[2] + V * f.qb[2];
      // (x, y) travel as a packed pair; the lerps run on (z0, z1) pairs (FADD2 / FFMA2). The
      // samples are visited from phase ph (x-normal members: V & 3, else 0) with wrap-around:
      // s_tpc[ph + k] = (tp(c), c), c = (ph + k) mod ntp, and the position is r0 + c qc.
      const f2 rxy0 = pk(rx, ry);
      const f2 qcxy = pk(f.qc[0], f.qc[1]);
      const float qcz = f.qc[2];
      const f2 mag = pk(kMagic, kMagic);
      const float2* tpc = s_tpc + ((MODE == 0 && f.skew) ? (iv & 3) : 0);
      float acc = 0.0f;
      if (MODE == 1) {
        // coverage: the trilinear interpolant of the grid indicator is separable, per axis
        // (1 - f) [i in grid] + f [i + 1 in grid] at the floor i and fraction f of the forward's
        // own sample positions -- no tile, no shared loads
        const int gx = G.lo[0] + f.ob[0], gy = G.lo[1] + f.ob[1], gz = G.lo[2] + f.ob[2];
        // a line is straight and fma(c, q, r) is monotone in c: when the floors of both end
        // samples lie in [0, n - 2] on every axis, every sample's 8 corners are in the grid and
        // the line's sum is sum tp (most lines of a group that merely touches the border)
        {
          const float c1 = (float)(ntp - 1);
          const f2 e0 = add2_rd(rxy0, mag), e1 = add2_rd(fma2s(c1, qcxy, rxy0), mag);
          const float z0 = __fadd_rd(rz, kMagic), z1 = __fadd_rd(fmaf(c1, qcz, rz), kMagic);
          const int x0 = gx + __float_as_int(lo2(e0)) - kMagicBits, x1 = gx + __float_as_int(lo2(e1)) - kMagicBits;
          const int y0 = gy + __float_as_int(hi2(e0)) - kMagicBits, y1 = gy + __float_as_int(hi2(e1)) - kMagicBits;
          const int zz0 = gz + __float_as_int(z0) - kMagicBits, zz1 = gz + __float_as_int(z1) - kMagicBits;
          if (min(x0, x1) >= 0 && max(x0, x1) <= n.x - 2 && min(y0, y1) >= 0 && max(y0, y1) <= n.y - 2 &&
              min(zz0, zz1) >= 0 && max(zz0, zz1) <= n.z - 2) {
            sT[f.t0 + iv * f.LU + iu] = H.tpsum;
            continue;
          }
        }
#pragma unroll kFwdUnroll
        for (int k = 0; k < ntp; ++k) {
          const float2 q = tpc[k];
          const f2 rxy = fma2s(q.y, qcxy, rxy0);
          const float rzc = fmaf(q.y, qcz, rz);
          const f2 txy = add2_rd(rxy, mag);
          const float tz = __fadd_rd(rzc, kMagic);
          const int ix = gx + __float_as_int(lo2(txy)) - kMagicBits;
          const int iy = gy + __float_as_int(hi2(txy)) - kMagicBits;
          const int iz = gz + __float_as_int(tz) - kMagicBits;
          const f2 fxy = sub2(rxy, sub2(txy, mag));
          const float fz = rzc - __fsub_rn(tz, kMagic);
          const float fx = lo2(fxy), fy = hi2(fxy);
          const float wx = ((unsigned)ix < (unsigned)n.x ? 1.0f - fx : 0.0f) + ((unsigned)(ix + 1) < (unsigned)n.x ? fx : 0.0f);
          const float wy = ((unsigned)iy < (unsigned)n.y ? 1.0f - fy : 0.0f) + ((unsigned)(iy + 1) < (unsigned)n.y ? fy : 0.0f);
          const float wz = ((unsigned)iz < (unsigned)n.z ? 1.0f - fz : 0.0f) + ((unsigned)(iz + 1) < (unsigned)n.z ? fz : 0.0f);
          acc = fmaf(q.x, wx * wy * wz, acc);
        }
        sT[f.t0 + iv * f.LU + iu] = acc;
        continue;
      }
      const float* sXo = sX + f.ob[2] * dxy + f.ob[1] * dx + f.ob[0];
      // one sample at lattice step cq (tp value tpk) added to acc
      auto sample = [&](float tpk, float cq, float acc_in) -> float {
        const f2 rxy = fma2s(cq, qcxy, rxy0);
        const float rzc = fmaf(cq, qcz, rz);
        const f2 txy = add2_rd(rxy, mag);
        const float tz = __fadd_rd(rzc, kMagic);
        const int ix = __float_as_int(lo2(txy)) - kMagicBits;
        const int iy = __float_as_int(hi2(txy)) - kMagicBits;
        const int iz = __float_as_int(tz) - kMagicBits;
        const f2 fxy = sub2(rxy, sub2(txy, mag));
        const float fz = rzc - __fsub_rn(tz, kMagic);
        const float* p = sXo + iz * dxy + iy * dx + ix;
        PVR_CHECK(p >= sX && p + dxy + dx + 1 < sX + dz * dxy);
        const f2 x00 = pk(p[0], p[dxy]), x10 = pk(p[1], p[dxy + 1]);            // (z0, z1) at y0
        const f2 x01 = pk(p[dx], p[dxy + dx]), x11 = pk(p[dx + 1], p[dxy + dx + 1]);  // at y1
        const float fx = lo2(fxy), fy = hi2(fxy);
        const f2 cy0 = fma2s(fx, sub2(x10, x00), x00);   // x-lerp, (z0, z1) at y0
        const f2 cy1 = fma2s(fx, sub2(x11, x01), x01);   // at y1
        const f2 cz = fma2s(fy, sub2(cy1, cy0), cy0);    // y-lerp: (z0, z1)
        const float c0 = lo2(cz), c1 = hi2(cz);
        return fmaf(tpk, fmaf(fz, c1 - c0, c0), acc_in);
      };
      if (ntp == kFwdNtpFixed && !f.skew) {
        // the common slice profile (c1-c5 at q = 1: 15 samples): fully unrolled, tp from
        // registers instead of one shared load per sample
#pragma unroll
        for (int k = 0; k < kFwdNtpFixed; ++k) acc = sample(tpr[k], (float)k, acc);
      } else {
#pragma unroll kFwdUnroll
        for (int k = 0; k < ntp; ++k) {
          const float2 q = tpc[k];
          acc = sample(q.x, q.y, acc);
        }
      }
      sT[f.t0 + iv * f.LU + iu] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_gn = kDyn ? atomicAdd(next, 1) : g + (int)gridDim.x;
      if (MODE == 0 && s_gn < a.ngroups) issue_tma(s_gn);
    }
    // pixels of all members: yhat = sum_ab ip(a,b) T(nu u + a, nv v + b) / kappa
    const int w2 = 2 * H.ru + 1;
    k = 0;
    for (int i = threadIdx.x; i < H.np; i += kThreads) {
      while (k + 1 < G.nm && i >= sm[k + 1].p0) ++k;
      const FwdMember& f = sm[k];
      const int li = i - f.p0;
      const int dv = (int)(((float)li + 0.5f) * f.inv_tu), du = li - dv * f.tu;  // li < 2^16: exact
      const int u = f.u0 + du, v = f.v0 + dv;
      float s = 0.0f;
      if (skip) {
        s = 1.0f;  // every sample fully in the grid: kappa = sum psi = 1 (reading Q27)
      } else {
        if (H.ru == 1 && H.rv == 1) {  // n_u = n_v = 2 (every stack of c1-c5 at q = 1): 3 x 3 taps unrolled
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const float* row = sT + f.t0 + (H.nv * dv + b) * f.LU + H.nu * du;
#pragma unroll
            for (int aa = 0; aa < 3; ++aa) s += s_ip[b * 3 + aa] * row[aa];
          }
        } else {
          for (int b = 0; b <= 2 * H.rv; ++b) {
            const float* row = sT + f.t0 + (H.nv * dv + b) * f.LU + H.nu * du;
            for (int aa = 0; aa < w2; ++aa) s += s_ip[b * w2 + aa] * row[aa];
          }
        }
      }
      const PatchDev& pt = a.P[f.patch];
      const int64_t j = pt.pix0 + ((int64_t)f.z * pt.sy + v) * pt.sx + u;
      const float y = a.ys[pt.y0off + (int64_t)f.z * pt.HW + (int64_t)v * pt.W + u];
      if (MODE == 1) {
        if (a.mask && !a.mask[j]) s = 0.0f;  // f3: masked-out pixel is never observed (Q32)
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
        const float kk = kap[j];
        const float ppf = pprev[j];  // issued with kappa's load, not after its test
        float ev = 0.0f;
        if (kk >= a.prm.tau_obs) {
          ev = y - s / kk;
          if (kk >= a.prm.tau_live) {
            const double pp = ppf;
            if (a.prm.det) {
              // deterministic mode: every term on a fixed grid (2^-4, 2^-24): the fp64 sums of
              // these integers (< 2^53) are exact in any order, on any number of ranks
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
        out[j] = ev;
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
  // the last one up to nu (sx - 1) + ru inclusive (engine.cu: owned() matches)
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

struct Tile {  // planar int32 accumulators of the group bbox: A, C (+ lo words for HILO)
  int *ah, *ch, *al, *cl;
  int dx, dy;
};

// Per-member constants of the backprojection, in the member's window frame: axis 0 (m) is
// the dominant component of the sample step dir * Qc (so plane floors never decrease along a
// line), axes 1, 2 (p, q) the transverse ones. Geometry only: built once per geometry by
// k_bp_table (a warp per group, a lane per member) into global memory, indexed like the plan's
// members, and copied into shared memory by each group's CTA.
struct __align__(16) BpMember {
  float r[3];              // frame position of lattice point (Ulo, Vlo, first sample) - o
  float du[3], dv[3], dc[3];  // frame steps per U, per V, per sample (dc[0] >= 0)
  int o[3];                // integer origin in the tile (frame)
  int s[3];                // tile strides (frame)
  int ti0, dti, ns;        // tp index of the first sample, its step (+-1), samples per line
  int Ulo, Vlo, nU, nV;    // owned lattice range [Ulo, Ulo + nU) x [Vlo, Vlo + nV)
  int nU3, nUV3;           // line colouring: ceil(nU / 3), ceil(nU / 3) ceil(nV / 3)
  float inv_nU3, inv_nUV3, inv_rw, inv_nU;
  int lbeg, lend;          // flattened (padded, colour-ordered) line range of the member
  int pbeg, pend;          // flattened pixel range (== its R range)
  int plu, plv, phu, phv, rw;
  int64_t pixz, yz;        // first pixel of slice z in the local arrays / in the stacks
  int sx, W;
  int patch;               // local patch index (its weight w is read per iteration)
};
static_assert(sizeof(BpMember) % 16 == 0, "BpMember is copied as int4");

struct __align__(16) BpGroupHdr {  // per-group totals and the group's stack PSF constants
  int nl, np;              // lattice lines / pixels of all members
  int nu, nv, ru, rv, ip0, tp0, ntp;
  float tpmax;
  float tmax;              // largest splat term in fixed-point units (k_bp_table: window and
                           // per-cell total bounds)
  float lsc;               // lo-word scale (2^20, lower if a cell could take > 4096 flushes)
};

__device__ __forceinline__ float pick3(const float (&v)[3], int ax) {
  return ax == 0 ? v[0] : (ax == 1 ? v[1] : v[2]);
}
__device__ __forceinline__ int pick3i(const int (&v)[3], int ax) {
  return ax == 0 ? v[0] : (ax == 1 ? v[1] : v[2]);
}

#ifndef PVR_BP_COLOUR
#define PVR_BP_COLOUR 0  // 1: lines in colour classes (U mod 3, V mod 3): no same-cell lanes
#endif                    // (measured slower: the bank conflicts remain, plus padding)
#ifndef PVR_BP_PHASES
#define PVR_BP_PHASES 2   // lanes start their line at sample (lane mod P) ns / P (wrapping)
#endif
#ifndef PVR_BP_UNROLL
#define PVR_BP_UNROLL 4
#endif
constexpr int kBpUnroll = PVR_BP_UNROLL;  // steps per iteration of the splat window loop
constexpr int kCOff = kBpTileBytes / 2;  // single-word tile: byte offset of the C plane
// exact tile (HILO): A_hi, C_hi, A_lo, C_lo planes at fixed byte offsets kHQ apart
constexpr int kHQ = kBpTileBytes / 4;

// Flush one plane of the window: corner j's weight sum S_j times the line's (LA, LC) into the
// A and C words of the 4 transverse corners (a, +sp4, +sq4, +sp4+sq4). PREC: kPrecSingle one
// word per quantity (A at 0, C at kCOff), kPrecHiLo two (planes kHQ apart), kPrecDet three
// (planes kH6 apart: deterministic mode's global scale).
constexpr int kPrecSingle = 0, kPrecHiLo = 1, kPrecDet = 2;
__shared__ int s_cells;  // cells of the current group's tile (PVR_CHECK bounds)
// deterministic tile: A_hi, C_hi, A_lo, C_lo, A_lo2, C_lo2 planes of kBpDetPlane bytes
constexpr int kH6 = kBpDetPlane;
static_assert(kH6 % 16 == 0, "tile planes must stay 16-byte aligned");
template <int PREC>
__device__ __forceinline__ void flush4(unsigned a, int sp4, int sq4, float s0, float s1, float s2, float s3,
                                       f2 L, f2 mag, f2 lsc) {
  if (PREC == kPrecSingle) {
    // L S + magic: the fixed-point rounding of each window sum (one FFMA2 per corner)
    const f2 t0 = fma2s(s0, L, mag), t1 = fma2s(s1, L, mag), t2 = fma2s(s2, L, mag), t3 = fma2s(s3, L, mag);
    sred<0>(a, __float_as_int(lo2(t0)) - kMagicBits);
    sred<kCOff>(a, __float_as_int(hi2(t0)) - kMagicBits);
    sred<0>(a + sp4, __float_as_int(lo2(t1)) - kMagicBits);
    sred<kCOff>(a + sp4, __float_as_int(hi2(t1)) - kMagicBits);
    sred<0>(a + sq4, __float_as_int(lo2(t2)) - kMagicBits);
    sred<kCOff>(a + sq4, __float_as_int(hi2(t2)) - kMagicBits);
    sred<0>(a + sp4 + sq4, __float_as_int(lo2(t3)) - kMagicBits);
    sred<kCOff>(a + sp4 + sq4, __float_as_int(hi2(t3)) - kMagicBits);
  } else {
    // hi / lo words of S L (A and C as a packed pair): t = S L + magic rounds to the hi
    // integer h = t - magic (exact); the FMA S L - h is the remainder r, |r| <= 1/2, and
    // lo = round(r lsc), lsc = 2^20 (k_bp_table). hi + lo / lsc equals S L to 1 / (2 lsc) hi
    // units: the word pair resolves ~2^-41 of the group's largest splat term, whatever the
    // cell's own total. Deterministic mode adds lo2 = round((r lsc - lo) lsc): ~2^-61 of the
    // global scale's largest term, for one scale shared by every group (grouping-independent).
    const unsigned ac[4] = {a, a + sp4, a + sq4, a + sp4 + sq4};
    const float sj[4] = {s0, s1, s2, s3};
    constexpr int Q = PREC == kPrecDet ? kH6 : kHQ;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const f2 t = fma2s(sj[j], L, mag);
      const f2 r = fma2s(sj[j], L, sub2(mag, t));
      const f2 l = fma2(r, lsc, mag);
      sred<0>(ac[j], __float_as_int(lo2(t)) - kMagicBits);
      sred<Q>(ac[j], __float_as_int(hi2(t)) - kMagicBits);
      sred<2 * Q>(ac[j], __float_as_int(lo2(l)) - kMagicBits);
      sred<3 * Q>(ac[j], __float_as_int(hi2(l)) - kMagicBits);
      if (PREC == kPrecDet) {
        const f2 l2 = fma2(fma2(r, lsc, sub2(mag, l)), lsc, mag);
        sred<4 * Q>(ac[j], __float_as_int(lo2(l2)) - kMagicBits);
        sred<5 * Q>(ac[j], __float_as_int(hi2(l2)) - kMagicBits);
      }
    }
  }
}

// Splat one lattice line with a two-plane register window along the frame's axis 0. Every
// sample of the line carries the same (LA, LC) (the line's adjoint values), so the window
// holds unitless weight sums: per transverse corner j a packed pair (plane m, plane m + 1)
// accumulating tp(c) x bilinear corner weight x (1 - f_m, f_m) with one FFMA2, scaled by
// (LA, LC) only when a plane is flushed. Every step first flushes plane m to the tile (one
// int32 rounding per corner and quantity per step), then shifts: a lane whose floor advanced
// moves plane m + 1 into slot m; a lane whose floor stayed keeps slot m + 1 (slot m restarts
// empty); a lane whose transverse floors changed also flushes plane m + 1 and restarts. The
// flush is uniform across the warp (all lanes issue the same 8 shared reductions); only the
// rarer transverse restart branches. Window sums before rounding: < 4 terms of < 2^20 units
// each (group scale, k_lattice_bp). Tile: A words at shared address tA, C words at
// tA + kCOff; HILO (exact groups): every window sum split into exact hi / lo words
// (A_hi, C_hi, A_lo, C_lo planes, kHQ apart).
template <int PREC>
__device__ __forceinline__ void splat_line_win(unsigned tA, unsigned s_tp, const BpMember& M, float rm0,
                                               float rp, float rq, float LA, float LC, float lo_scale,
                                               int ph) {
  const f2 rpq0 = pk(rp, rq);
  const float qm = M.dc[0];
  const f2 qpq = pk(M.dc[1], M.dc[2]);
  const f2 mag = pk(kMagic, kMagic);
  const f2 L = pk(LA, LC);
  const f2 lsc = pk(lo_scale, lo_scale);
  const f2 one0 = pk(1.0f, 0.0f), m1p1 = pk(-1.0f, 1.0f);
  const int sm4 = 4 * M.s[0], sp4 = 4 * M.s[1], sq4 = 4 * M.s[2];
  const unsigned org = tA + (unsigned)(M.o[0] * sm4 + M.o[1] * sp4 + M.o[2] * sq4);
  const unsigned ta0 = s_tp + 4u * M.ti0;
  const int dta = 4 * M.dti;
  const int ns = M.ns;
  const float nsf = (float)ns;
  // samples are visited from index ph with wrap-around (ph = 0 for phase 0 lanes): lanes of a
  // warp that walk neighbouring lines then sit in different planes of the tile, so their
  // same-floor cells are different addresses and their banks are offset (the wrap costs one
  // restart flush)
  float kf = (float)ph;
  unsigned ta = ta0 + (unsigned)(dta * ph);
  int wm = 0, wp = 0, wq = 0;
  f2 P[4];  // corner j: (plane wm, plane wm + 1) weight sums
#pragma unroll
  for (int j = 0; j < 4; ++j) P[j] = pk(0.0f, 0.0f);
#pragma unroll kBpUnroll
  for (int k = 0; k < ns; ++k) {
    const float rm = fmaf(kf, qm, rm0);
    const f2 rpq = fma2s(kf, qpq, rpq0);
    const float tm = __fadd_rd(rm, kMagic);
    const f2 tpq = add2_rd(rpq, mag);
    const int im = __float_as_int(tm) - kMagicBits;
    const int ip = __float_as_int(lo2(tpq)) - kMagicBits;
    const int iq = __float_as_int(hi2(tpq)) - kMagicBits;
    if (k > 0) {  // (uniform) the first sample only opens the window
      const bool same = (ip == wp) & (iq == wq);
      const bool keep = same & (im == wm);
      const bool adv = same & (im == wm + 1);
      const unsigned a0 = org + wm * sm4 + wp * sp4 + wq * sq4;
      PVR_CHECK(a0 >= tA && a0 + sm4 + sp4 + sq4 < tA + 4u * (unsigned)s_cells);
      flush4<PREC>(a0, sp4, sq4, lo2(P[0]), lo2(P[1]), lo2(P[2]), lo2(P[3]), L, mag, lsc);  // plane wm
      if (!keep && !adv)  // restart (transverse change, the wrap, a jump): plane wm + 1 too
        flush4<PREC>(a0 + sm4, sp4, sq4, hi2(P[0]), hi2(P[1]), hi2(P[2]), hi2(P[3]), L, mag, lsc);
      // shift: keep -> (0, m+1); advance -> (m+1, 0); restart -> (0, 0)
      const f2 sh = pk(adv ? 1.0f : 0.0f, keep ? 1.0f : 0.0f);
#pragma unroll
      for (int j = 0; j < 4; ++j) P[j] = mul2s(hi2(P[j]), sh);
    }
    wm = im;
    wp = ip;
    wq = iq;
    // this sample's weights
    float t;
    asm("ld.shared.f32 %0, [%1];" : "=f"(t) : "r"(ta));
    const float flm = __fsub_rn(tm, kMagic);
    const f2 fpq = sub2(rpq, sub2(tpq, mag));
    const float fm = rm - flm, fp = lo2(fpq), fq = hi2(fpq);
    const f2 TM = mul2s(t, fma2s(fm, m1p1, one0));  // t (1 - fm, fm)
    const f2 WP = fma2s(fp, m1p1, one0);            // (1 - fp, fp)
    const f2 w01 = mul2s(1.0f - fq, WP), w23 = mul2s(fq, WP);
    P[0] = fma2s(lo2(w01), TM, P[0]);
    P[1] = fma2s(hi2(w01), TM, P[1]);
    P[2] = fma2s(lo2(w23), TM, P[2]);
    P[3] = fma2s(hi2(w23), TM, P[3]);
    kf += 1.0f;
    ta += dta;
    if (kf == nsf) {  // wrap to the line's first sample
      kf = 0.0f;
      ta = ta0;
    }
  }
  const unsigned a0 = org + wm * sm4 + wp * sp4 + wq * sq4;
  PVR_CHECK(a0 >= tA && a0 + sm4 + sp4 + sq4 < tA + 4u * (unsigned)s_cells);
  flush4<PREC>(a0, sp4, sq4, lo2(P[0]), lo2(P[1]), lo2(P[2]), lo2(P[3]), L, mag, lsc);
  flush4<PREC>(a0 + sm4, sp4, sq4, hi2(P[0]), hi2(P[1]), hi2(P[2]), hi2(P[3]), L, mag, lsc);
}

// Member tables of all groups of a backprojection plan (geometry only: rebuilt after every
// set_transforms / re-plan, reused by every iteration). One W-lane segment of a warp per group
// (W >= the plan's largest member count: c3 groups have ~3 members, so W = 4 puts 8 groups in
// a warp), one lane per member; the flattened line / pixel ranges by segment scans.
template <int W>
__global__ void __launch_bounds__(kThreads) k_bp_table(LatticeArgs a, BpMember* __restrict__ tm,
                                                      BpGroupHdr* __restrict__ th) {
  static_assert(W >= 1 && W <= 32 && (W & (W - 1)) == 0, "segment width: a power of two <= 32");
  const int lane = threadIdx.x & (W - 1);
  const unsigned seg = W == 32 ? 0xffffffffu : (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)));
  const int g = (int)((blockIdx.x * blockDim.x + threadIdx.x) / W);
  if (g >= a.ngroups) return;  // uniform per segment
  const GroupDev G = a.grp[g];
  if (G.nm == 0) {  // emptied by a device re-plan split (engine.cu: replan_on_device)
    if (lane == 0) {
      BpGroupHdr h = {};
      th[g] = h;
    }
    return;
  }
  const int dx = G.dim[0], dy = G.dim[1];
  int nl = 0, np = 0;
  BpMember M;
  MemberGeom mg;
  if (lane < G.nm) {
    const MemberDev m = a.mem[G.m0 + lane];
    const PatchDev& pt = a.P[m.patch];
    mg = member_geom(a, pt);
    const Owned o = owned_range(m, pt, mg);
    const float aq0 = fabsf(mg.qc[0]), aq1 = fabsf(mg.qc[1]), aq2 = fabsf(mg.qc[2]);
    const int am = (aq0 >= aq1 && aq0 >= aq2) ? 0 : (aq1 >= aq2 ? 1 : 2);
    const int ap = am == 0 ? 1 : 0, aq = am == 2 ? 1 : 2;
    const int dir = pick3(mg.qc, am) >= 0.0f ? 1 : -1;
    const int cs = dir > 0 ? m.c0 : m.c1;
    int ob[3];
    float of[3];
    lattice_origin(pt, m.z, o.Ulo, o.Vlo, cs, G.lo, ob, of);
    const int st[3] = {1, dx, dx * dy};
    const int ax[3] = {am, ap, aq};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      M.r[d] = pick3(of, ax[d]);
      M.o[d] = pick3i(ob, ax[d]);
      M.s[d] = pick3i(st, ax[d]);
      M.du[d] = pick3(mg.qa, ax[d]);
      M.dv[d] = pick3(mg.qb, ax[d]);
      M.dc[d] = (float)dir * pick3(mg.qc, ax[d]);
    }
    M.ti0 = cs + mg.cmax;
    M.dti = dir;
    M.ns = m.c1 - m.c0 + 1;
    M.Ulo = o.Ulo;
    M.Vlo = o.Vlo;
    M.nU = o.Uhi - o.Ulo;
    M.nV = o.Vhi - o.Vlo;
    M.nU3 = (M.nU + 2) / 3;
    M.nUV3 = M.nU3 * ((M.nV + 2) / 3);
    M.inv_nU3 = 1.0f / (float)M.nU3;
    M.inv_nUV3 = 1.0f / (float)M.nUV3;
    M.inv_nU = 1.0f / (float)M.nU;
    M.plu = o.plu; M.phu = o.phu; M.plv = o.plv; M.phv = o.phv;
    // R block of the member: its feeding pixels [plu, phu] x [plv, phv] with a zero border of
    // one pixel, so the line gather reads its up to 4 taps without bounds tests
    M.rw = o.phu - o.plu + 3;
    M.inv_rw = 1.0f / (float)M.rw;
    M.pixz = pt.pix0 + (int64_t)m.z * pt.sy * pt.sx;
    M.yz = pt.y0off + (int64_t)m.z * pt.HW;
    M.sx = pt.sx;
    M.W = pt.W;
    M.patch = m.patch;
#if PVR_BP_COLOUR
    nl = 9 * M.nUV3;  // 9 colour classes (U mod 3, V mod 3), padded to whole classes
#else
    nl = M.nU * M.nV;
#endif
    np = M.rw * (o.phv - o.plv + 3);
  }
  // window bound: a flushed plane sums the terms of all samples whose floor along m is
  // m - 1 (<= ceil(1 / qm) of them, qm = the step along m >= |qc| / sqrt 3) and of one at
  // floor m; nterm tmax <= 2^22 keeps the magic rounding exact (c3: qm ~ 0.89, nterm = 3,
  // tmax = 2^20; ns bounds nterm for a degenerate step)
  float nterm = 1.0f;
  // Per-cell totals (int32 words): a cell k takes, from one member, the lines whose transverse
  // position lies within 1 voxel of it -- lattice points of the (du, dv) transverse lattice in
  // a 2 x 2 square: <= (2 + |du_t| + |dv_t|)^2 / |du_t x dv_t| -- each flushing the plane of k
  // at most ceil(2 / qm) + 2 times, with weights along m summing to <= 1 / qm + 1. So the hi
  // total is <= sum_members (1 / qm + 1) nlines tmax and the lo total (|lo| <= lsc / 2 per
  // flush) <= sum_members (ceil(2 / qm) + 2) nlines lsc / 2; both are kept below 2^30.
  float hib = 0.0f, flb = 0.0f;
  if (lane < G.nm) {
    const float qm = fmaxf(M.dc[0], 1e-6f);
    nterm = fminf(ceilf(1.0f / qm), (float)M.ns) + 1.0f;
    const float at = fabsf(M.du[1] * M.dv[2] - M.du[2] * M.dv[1]);
    const float lu = sqrtf(M.du[1] * M.du[1] + M.du[2] * M.du[2]);
    const float lv = sqrtf(M.dv[1] * M.dv[1] + M.dv[2] * M.dv[2]);
    const float nlines = fminf((2.0f + lu + lv) * (2.0f + lu + lv) / fmaxf(at, 1e-12f),
                               (float)(M.nU * M.nV));
    const float steps = fminf(1.0f / qm + 1.0f, (float)M.ns);
    hib = steps * nlines;
    flb = fminf(ceilf(2.0f / qm) + 2.0f, (float)M.ns + 1.0f) * nlines;
  }
#pragma unroll
  for (int d = W / 2; d > 0; d >>= 1) {
    nterm = fmaxf(nterm, __shfl_xor_sync(seg, nterm, d, W));
    hib += __shfl_xor_sync(seg, hib, d, W);
    flb += __shfl_xor_sync(seg, flb, d, W);
  }
  int sl = nl, sp = np;  // inclusive scans over the members
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    const int tl = __shfl_up_sync(seg, sl, d, W), tp = __shfl_up_sync(seg, sp, d, W);
    if (lane >= d) { sl += tl; sp += tp; }
  }
  const int tl = __shfl_sync(seg, sl, G.nm - 1, W), tpx = __shfl_sync(seg, sp, G.nm - 1, W);
  if (lane < G.nm) {
    M.lbeg = sl - nl; M.lend = sl;
    M.pbeg = sp - np; M.pend = sp;
    tm[G.m0 + lane] = M;
  }
  if (lane == 0) {  // all members of a group share the stack (and its PSF)
    BpGroupHdr h;
    h.nl = tl; h.np = tpx;
    h.nu = mg.nu; h.nv = mg.nv; h.ru = mg.ru; h.rv = mg.rv;
    h.ip0 = mg.ip0; h.tp0 = mg.tp0; h.ntp = mg.ntp;
    h.tpmax = a.psf[a.P[a.mem[G.m0].patch].stack].tpmax;
    h.tmax = fminf(fminf(kTermMax, kWindowMax / nterm), 1073741824.0f / fmaxf(hib, 1.0f));
    h.lsc = fminf(kLoScale, 2147483648.0f / fmaxf(flb, 1.0f));
    th[g] = h;
  }
}

#ifndef PVR_BP_DYN
#define PVR_BP_DYN 1
#endif

// Dynamic shared memory: the tile (exact group: planes A_hi, C_hi, A_lo, C_lo at byte offsets
// kHQ apart; single-word group: A at 0, C at kCOff; offsets are immediates of the splat's
// shared reductions), then R after kBpTileBytes. kBpCtasPerSm CTAs per SM.
// DET: the deterministic mode's instance (three-word tiles, int64 accumulators); the default
// instance carries only the single-word and hi/lo paths (fewer registers).
template <bool DET>
__global__ void __launch_bounds__(kBpThreads, kBpCtasPerSm) k_lattice_bp(LatticeArgs a, int tile_words,
                                                         const BpMember* __restrict__ tm,
                                                         const BpGroupHdr* __restrict__ th,
                                                         const float* __restrict__ kap,
                                                         const float* __restrict__ e,
                                                         const float* __restrict__ p,
                                                         const float* __restrict__ w, int init,
                                                         float2* __restrict__ AC,
                                                         int* __restrict__ next) {
  extern __shared__ int4 bsm4[];
  int* base = reinterpret_cast<int*>(bsm4);

  float2* R = reinterpret_cast<float2*>(base + kBpTileBytes / 4);
  __shared__ float s_ip[kMaxIp], s_tp[kMaxTp];
  __shared__ float s_red[2][kBpThreads >> 5];
  __shared__ BpMember sbm[kMaxMembers];
  const int3 n = a.n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned tA = (unsigned)__cvta_generic_to_shared(base);
  const unsigned tpA = (unsigned)__cvta_generic_to_shared(s_tp);

#if PVR_BP_DYN
  // persistent CTAs (resident count per SM x SMs) take the next group from the plan's launch
  // counter (after the group headers, reset before every launch): groups differ in cost, and a
  // static stride left SMs idle at the end (bp 14.59 -> 14.22 ms at c3)
  // The next group is claimed (and its header fetched into shared memory) by thread 0 as soon
  // as the current group's phase A is done, so the claim's and the header loads' round trips
  // overlap the splat instead of opening the next group.
  __shared__ int s_next;
  __shared__ GroupDev s_G;
  __shared__ BpGroupHdr s_H;
  auto claim = [&]() {
    const int gn = atomicAdd(next, 1);
    if (gn < a.ngroups) {
      s_G = a.grp[gn];
      s_H = th[gn];
    }
    s_next = gn;
  };
  if (threadIdx.x == 0) claim();
  for (;;) {
    __syncthreads();  // s_next / s_G / s_H of this group are published; the previous group is done
    const int g = s_next;
    if (g >= a.ngroups) break;
    const GroupDev G = s_G;
    const BpGroupHdr H = s_H;
#else
  for (int g = blockIdx.x; g < a.ngroups; g += gridDim.x) {
    const GroupDev G = a.grp[g];
    const BpGroupHdr H = th[g];
#endif
    // CTA-uniform: this group's tile precision (deterministic mode: three words everywhere)
    const int prec = DET ? kPrecDet : (init || G.exact) ? kPrecHiLo : kPrecSingle;
    const bool ex = prec != kPrecSingle;
    const int NW = prec == kPrecDet ? 6 : ex ? 4 : 2;
    const int QW = prec == kPrecDet ? kH6 / 4 : kHQ / 4;  // words between the exact planes
    int* cbase = ex ? base + QW : base + kCOff / 4;
    const int dx = G.dim[0], dy = G.dim[1], dz = G.dim[2];
    const int nvox = dx * dy * dz;
#if !PVR_BP_DYN
    __syncthreads();  // previous group's flush is done with the tile / R / tables / sbm
#endif                // (PVR_BP_DYN: the barrier at the loop top)
    if (threadIdx.x == 0) s_cells = nvox;
    {  // member table, the stack's PSF factors, the tile reset
      const int4* src = reinterpret_cast<const int4*>(tm + G.m0);
      int4* dst = reinterpret_cast<int4*>(sbm);
      const int nq = G.nm * (int)(sizeof(BpMember) / 16);
      for (int i = threadIdx.x; i < nq; i += kBpThreads) dst[i] = __ldg(src + i);
      const int nip = (2 * H.ru + 1) * (2 * H.rv + 1);
      for (int i = threadIdx.x; i < nip; i += kBpThreads) s_ip[i] = a.tab[H.ip0 + i];
      for (int i = threadIdx.x; i < H.ntp; i += kBpThreads) s_tp[i] = a.tab[H.tp0 + i];
      const int4 z4 = make_int4(0, 0, 0, 0);
      const int nv4 = (nvox + 3) >> 2;  // tile_words is a multiple of 4
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        if (q >= NW) break;
        int4* t4 = reinterpret_cast<int4*>(ex ? base + q * QW : (q == 1 ? cbase : base));
        for (int i = threadIdx.x; i < nv4; i += kBpThreads) t4[i] = z4;
      }
    }
    __syncthreads();
    // ---- phase A: per-pixel (rA, rC) of every member into R; group maxima for the scale
    float mA = 0.0f, mC = 0.0f;
    {
      const int np = H.np;
      int mi = 0;
      for (int i = threadIdx.x; i < np; i += kBpThreads) {
        while (i >= sbm[mi].pend) ++mi;
        const BpMember& M = sbm[mi];
        const int li = i - M.pbeg;
        const int vv = (int)(((float)li + 0.5f) * M.inv_rw);
        const int uu = li - vv * M.rw;
        const int u = M.plu - 1 + uu, v = M.plv - 1 + vv;
        float rA = 0.0f, rC = 0.0f;
        if (u < M.plu || u > M.phu || v < M.plv || v > M.phv) {  // the zero border
          R[i] = make_float2(0.0f, 0.0f);
          continue;
        }
        const int64_t j = M.pixz + (int64_t)v * M.sx + u;
        // every load is issued before the observed test (one round trip, not two): the
        // patch weight w (1 in the init / rigidity passes; rigidity: vs = the patch score pbar)
        const float wm = init == 1 ? 1.0f : w[M.patch];
        const float ws = init ? 1.0f : wm, vs = init == 2 ? wm : 1.0f;
        const float k = kap[j];
        const float pj = init == 1 ? 1.0f : p[j];
        const float val = init == 1 ? a.ys[M.yz + (int64_t)v * M.W + u] : init == 2 ? pj * vs : e[j];
        if (ws != 0.0f && k >= a.prm.tau_obs) {
          const float pv = init ? 1.0f : pj;
          rC = ws * pv / k;
          rA = rC * val;
        }
        R[i] = make_float2(rA, rC);
        mA = fmaxf(mA, fabsf(rA));
        mC = fmaxf(mC, rC);
      }
    }
    mA = warp_max(mA);
    mC = warp_max(mC);
    if (lane == 0) {
      s_red[0][wid] = mA;
      s_red[1][wid] = mC;
    }
    __syncthreads();
#if PVR_BP_DYN
    // every thread holds G and H in registers by now: thread 0 may claim the next group
    if (threadIdx.x == 0) claim();
#endif
    float xA = 0.0f, xC = 0.0f;  // every thread forms the same group maxima and scales
#pragma unroll
    for (int i = 0; i < (kBpThreads >> 5); ++i) {
      xA = fmaxf(xA, s_red[0][i]);
      xC = fmaxf(xC, s_red[1][i]);
    }
    // every splat term |L tp w| <= max|r| tpmax  ->  <= H.tmax units; a register window
    // plane sums at most nterm such terms before rounding (<= 2^22; k_bp_table)
    float scA = xA > 0.0f ? H.tmax / (xA * H.tpmax) : 0.0f;
    float scC = xC > 0.0f ? H.tmax / (xC * H.tpmax) : 0.0f;
    if (scA == 0.0f && scC == 0.0f) continue;  // nothing to splat (excluded patches)
    if (DET) {  // one scale for every group (k_det_scales), grouping-independent
      scA = xA > 0.0f ? (float)a.det_scale[0] : 0.0f;
      scC = xC > 0.0f ? (float)a.det_scale[1] : 0.0f;
    }
    const Tile T{base, cbase, base + 2 * QW, base + 3 * QW, dx, dy};

    // ---- phase B: splat every owned lattice line of every member, one flattened range
    // (one tail per group); consecutive lanes take consecutive U lines of a member
    {
      const int nl = H.nl;
      const int w2 = 2 * H.ru + 1;
      const float inv_nu = 1.0f / (float)H.nu, inv_nv = 1.0f / (float)H.nv;
      int mi = 0;
      for (int i = threadIdx.x; i < nl; i += kBpThreads) {
        while (i >= sbm[mi].lend) ++mi;
        const BpMember& M = sbm[mi];
        // colour-ordered lines: class (U mod 3, V mod 3), then rows of the class. The lanes of
        // a warp take lines >= 3 lattice steps (~2.5 voxels) apart, so no two lanes flush the
        // same tile cell in one shared reduction (adjacent lines 0.83 voxel apart did: 2.4
        // wavefronts per ATOMS, 58% of them conflicts; ncu v14)
        const int li = i - M.lbeg;
#if PVR_BP_COLOUR
        const int cls = (int)(((float)li + 0.5f) * M.inv_nUV3);
        const int r = li - cls * M.nUV3;
        const int b3 = (int)(((float)r + 0.5f) * M.inv_nU3);
        const int cv = (int)(((float)cls + 0.5f) * (1.0f / 3.0f));
        const int iu = (cls - 3 * cv) + 3 * (r - b3 * M.nU3);
        const int iv = cv + 3 * b3;
        if (iu >= M.nU || iv >= M.nV) continue;  // padding of the class grid
#else
        const int iv = (int)(((float)li + 0.5f) * M.inv_nU);
        const int iu = li - iv * M.nU;
#endif
        const int U = M.Ulo + iu, V = M.Vlo + iv;
        // pixels feeding lattice point U: u = (U - a) / nu with a = U mod nu (and a - nu when
        // that is within [-ru, ru]); same along V. U >= -ru > -nu: the float floor is exact.
        const int ub = __float2int_rd(((float)U + 0.5f) * inv_nu), ra = U - ub * H.nu;
        const int vb = __float2int_rd(((float)V + 0.5f) * inv_nv), rb = V - vb * H.nv;
        // taps (ja, jb): a = ra - ja nu, b = rb - jb nv at pixel (ub + ja, vb + jb); with
        // ru = nu - 1 (engine.cu build_psf) a = ra is always in [-ru, ru] and a = ra - nu is
        // iff ra > 0; pixels outside [plu, phu] x [plv, phv] read the R block's zero border.
        // Summed in the order of the tap loop (jb, then ja).
        const bool a1 = ra > 0, b1 = rb > 0;
        const float* ipr = s_ip + (rb + H.rv) * w2 + (ra + H.ru);
        const float w00 = ipr[0];
        const float w10 = a1 ? ipr[-H.nu] : 0.0f;
        const float w01 = b1 ? ipr[-H.nv * w2] : 0.0f;
        const float w11 = (a1 && b1) ? ipr[-H.nv * w2 - H.nu] : 0.0f;
        const float2* rp0 = R + M.pbeg + (vb - M.plv + 1) * M.rw + (ub - M.plu + 1);
        const float2 r00 = rp0[0], r10 = rp0[1], r01 = rp0[M.rw], r11 = rp0[M.rw + 1];
        float LA = w00 * r00.x, LC = w00 * r00.y;
        LA += w10 * r10.x;
        LC += w10 * r10.y;
        LA += w01 * r01.x;
        LC += w01 * r01.y;
        LA += w11 * r11.x;
        LC += w11 * r11.y;
        if (LA == 0.0f && LC == 0.0f) continue;
        LA *= scA;
        LC *= scC;
        const float fU = (float)iu, fV = (float)iv;
        const float rm = M.r[0] + fU * M.du[0] + fV * M.dv[0];
        const float rp = M.r[1] + fU * M.du[1] + fV * M.dv[1];
        const float rq = M.r[2] + fU * M.du[2] + fV * M.dv[2];
        const int ph = PVR_BP_PHASES > 1 ? ((lane & (PVR_BP_PHASES - 1)) * M.ns) / PVR_BP_PHASES : 0;
        if (DET)
          splat_line_win<kPrecDet>(tA, tpA, M, rm, rp, rq, LA, LC, kLoScale, ph);
        else if (prec == kPrecHiLo)
          splat_line_win<kPrecHiLo>(tA, tpA, M, rm, rp, rq, LA, LC, H.lsc, ph);
        else
          splat_line_win<kPrecSingle>(tA, tpA, M, rm, rp, rq, LA, LC, H.lsc, ph);
      }
    }
    __syncthreads();
    // ---- phase C: flush the tile, one red.v4 per in-grid (even, odd) voxel pair along x
    const double iA = scA > 0.0f ? 1.0 / scA : 0.0, iC = scC > 0.0f ? 1.0 / scC : 0.0;
    const double ilo = 1.0 / (double)H.lsc;
    const float fA = (float)iA, fC = (float)iC;
    const int hx = (dx + 1) >> 1, npair = hx * dy * dz;
    const float inv_hx = 1.0f / (float)hx, inv_dy = 1.0f / (float)dy;
    // flat pair index i = (zl * dy + yl) * hx + pl, decoded by float reciprocals (exact for
    // these small integers); 32-bit voxel offsets (the volume has < 2^31 voxels)
    const int gbase = (G.lo[2] * n.y + G.lo[1]) * a.nxp + G.lo[0];
    if (DET) {
      for (int i = threadIdx.x; i < npair; i += kBpThreads) {
        const int row = (int)(((float)i + 0.5f) * inv_hx);
        const int pl = i - row * hx;
        const int zl = (int)(((float)row + 0.5f) * inv_dy);
        const int yl = row - zl * dy;
        const int gy = G.lo[1] + yl, gz = G.lo[2] + zl, gx = G.lo[0] + 2 * pl;
        if ((unsigned)gy >= (unsigned)n.y || (unsigned)gz >= (unsigned)n.z || (unsigned)gx >= (unsigned)a.nxp)
          continue;
        const int k = row * dx + 2 * pl;
        const bool two = 2 * pl + 1 < dx;  // odd pitch: the last pair has one tile cell
        // deterministic mode: exact int64 totals per voxel and quantity, hi and (lo 2^20 + lo2)
        // parts at the global scale, accumulated by integer reductions (order-independent)
        for (int h = 0; h < (two ? 2 : 1); ++h) {
          const int kk = k + h;
          long long v[4];
          for (int qn = 0; qn < 2; ++qn) {
            v[2 * qn] = base[qn * QW + kk];
            v[2 * qn + 1] = (long long)base[(2 + qn) * QW + kk] * 1048576LL + base[(4 + qn) * QW + kk];
          }
          if ((v[0] | v[1] | v[2] | v[3]) == 0) continue;
          unsigned long long* d = a.ACd + 4 * (size_t)(gbase + (zl * n.y + yl) * a.nxp + 2 * pl + h);
          for (int qn = 0; qn < 4; ++qn)
            if (v[qn]) atomicAdd(d + qn, (unsigned long long)v[qn]);
        }
      }
      continue;
    }
    // (row, pl) of a thread's successive pairs advance by (kBpThreads / hx, kBpThreads % hx)
    // with one carry; one loop per tile precision (CTA-uniform), the single-word one free of
    // the lo words
    const int dq = kBpThreads / hx, dr = kBpThreads - dq * hx;
    const int row0 = (int)(((float)threadIdx.x + 0.5f) * inv_hx), pl0 = (int)threadIdx.x - row0 * hx;
    auto flush_tile = [&](auto exact_words) {
      constexpr bool EXW = decltype(exact_words)::value;
      int row = row0, pl = pl0;
      for (int i = threadIdx.x; i < npair; i += kBpThreads) {
        const int r = row, q = pl;
        pl += dr;
        row += dq;
        if (pl >= hx) {
          pl -= hx;
          ++row;
        }
        const int zl = (int)(((float)r + 0.5f) * inv_dy);
        const int yl = r - zl * dy;
        const int gy = G.lo[1] + yl, gz = G.lo[2] + zl, gx = G.lo[0] + 2 * q;
        if ((unsigned)gy >= (unsigned)n.y || (unsigned)gz >= (unsigned)n.z || (unsigned)gx >= (unsigned)a.nxp)
          continue;
        const int k = r * dx + 2 * q;
        const bool two = 2 * q + 1 < dx;  // odd pitch: the last pair has one tile cell
        const int ah0 = T.ah[k], ah1 = two ? T.ah[k + 1] : 0, ch0 = T.ch[k], ch1 = two ? T.ch[k + 1] : 0;
        float A0, A1, C0, C1;
        if (EXW) {
          const int al0 = T.al[k], al1 = two ? T.al[k + 1] : 0;
          const int cl0 = T.cl[k], cl1 = two ? T.cl[k + 1] : 0;
          if ((ah0 | ah1 | ch0 | ch1 | al0 | al1 | cl0 | cl1) == 0) continue;
          A0 = (float)(((double)ah0 + (double)al0 * ilo) * iA);
          A1 = (float)(((double)ah1 + (double)al1 * ilo) * iA);
          C0 = (float)(((double)ch0 + (double)cl0 * ilo) * iC);
          C1 = (float)(((double)ch1 + (double)cl1 * ilo) * iC);
        } else {
          if ((ah0 | ah1 | ch0 | ch1) == 0) continue;
          A0 = (float)ah0 * fA; A1 = (float)ah1 * fA;
          C0 = (float)ch0 * fC; C1 = (float)ch1 * fC;
        }
        PVR_CHECK(gbase + (zl * n.y + yl) * a.nxp + 2 * q + 1 < n.z * n.y * a.nxp + 2);
        red_v4(AC + (gbase + (zl * n.y + yl) * a.nxp + 2 * q), A0, C0, A1, C1);
      }
    };
    if (ex)
      flush_tile(std::true_type{});
    else
      flush_tile(std::false_type{});
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------
// Per-device kernel attributes and occupancy (cudaFuncSetAttribute applies to the current
// device only; contexts on several GPUs of one process each configure theirs once).
struct DevConfig {
  int nsm = 0, resident = 0;
};
constexpr int kMaxDevices = 64;
static DevConfig g_dev[kMaxDevices];
static std::once_flag g_dev_once[kMaxDevices];

static const DevConfig& configure() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  std::call_once(g_dev_once[dev], [dev] {
    DevConfig& c = g_dev[dev];
    cudaFuncSetAttribute(k_lattice_bp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_lattice_bp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_lattice_fwd<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_lattice_fwd<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.resident, k_lattice_bp<false>, kBpThreads, kBpTileBytes + kRBytes);
  });
  return g_dev[dev];
}

// Forward member rows of all groups of a plan (geometry only: rebuilt after every
// set_transforms / re-plan, reused by every forward and coverage pass). One W-lane warp
// segment per group, one lane per member; the lattice-point and pixel offsets by segment scans.
template <int W>
__global__ void __launch_bounds__(kThreads) k_fwd_table(LatticeArgs a, FwdMember* __restrict__ fm,
                                                       FwdHdr* __restrict__ fh) {
  const int lane = threadIdx.x & (W - 1);
  const unsigned seg = W == 32 ? 0xffffffffu : (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)));
  const int g = (int)((blockIdx.x * blockDim.x + threadIdx.x) / W);
  if (g >= a.ngroups) return;  // uniform per segment
  const GroupDev G = a.grp[g];
  if (G.nm == 0) {  // emptied by a device re-plan split
    if (lane == 0) {
      FwdHdr h = {};
      fh[g] = h;
    }
    return;
  }
  FwdMember f = {};
  StackPsf ps = {};
  int nt = 0, np = 0;
  if (lane < G.nm) {
    const MemberDev m = a.mem[G.m0 + lane];
    const PatchDev& pt = a.P[m.patch];
    ps = a.psf[pt.stack];
    f.LU = ps.nu * (m.tu - 1) + 2 * ps.ru + 1;
    f.LV = ps.nv * (m.tv - 1) + 2 * ps.rv + 1;
    lattice_origin(pt, m.z, ps.nu * m.u0 - ps.ru, ps.nv * m.v0 - ps.rv, -ps.cmax, G.lo, f.ob, f.of);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      f.qa[d] = pt.Qa[d];
      f.qb[d] = pt.Qb[d];
      f.qc[d] = pt.Qc[d];
    }
    f.patch = m.patch; f.z = m.z; f.u0 = m.u0; f.v0 = m.v0; f.tu = m.tu; f.tv = m.tv;
    // V along the tile's y axis (axial-like stacks): a warp of row-ordered points straddles
    // two lattice rows one tile row (dx floats) apart -> bank conflicts; blocks of 4 U x 8 V
    // points hit 32 distinct banks (rows 4 (mod 8) banks apart). x-normal stacks (c along
    // x): lanes differ only in y and z, whose tile offsets are multiples of 4 floats (TMA row
    // pitch), so a warp reaches 8 banks (4 wavefronts per load); blocks of 8 U x 4 V with the
    // c loop of row V started at phase V & 3 spread the lanes over 4 x offsets
    // (tools/banksim_forward.py: 4.0 -> 1.5 wavefronts). Other stacks keep rows. (Coverage
    // reads no X tile and walks rows: k_lattice_fwd<1> ignores sh and skew.)
    const float ab0 = fabsf(pt.Qb[0]), ab1 = fabsf(pt.Qb[1]), ab2 = fabsf(pt.Qb[2]);
    const float ac0 = fabsf(pt.Qc[0]), ac1 = fabsf(pt.Qc[1]), ac2 = fabsf(pt.Qc[2]);
    const bool xn = ac0 >= ac1 && ac0 >= ac2;
    f.sh = (ab1 >= ab0 && ab1 >= ab2 && f.LU >= 4) ? 2 : (xn && f.LU >= 8 ? 3 : 0);
    f.skew = xn ? 1 : 0;
    f.inv_LU = 1.0f / (float)f.LU;
    f.inv_s4 = 1.0f / (float)((1 << f.sh) * f.LV);
    f.inv_tu = 1.0f / (float)f.tu;
    nt = f.LU * f.LV;
    np = f.tu * f.tv;
  }
  int st = nt, sp = np;  // inclusive scans over the members
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    const int tt = __shfl_up_sync(seg, st, d, W), tp = __shfl_up_sync(seg, sp, d, W);
    if (lane >= d) { st += tt; sp += tp; }
  }
  const int tot_t = __shfl_sync(seg, st, G.nm - 1, W), tot_p = __shfl_sync(seg, sp, G.nm - 1, W);
  if (lane < G.nm) {
    f.t0 = st - nt;
    f.p0 = sp - np;
    fm[G.m0 + lane] = f;
  }
  if (lane == 0) {  // all members of a group share the stack (and its PSF)
    FwdHdr h = {};
    h.nt = tot_t; h.np = tot_p;
    h.nu = ps.nu; h.nv = ps.nv; h.ru = ps.ru; h.rv = ps.rv;
    h.ip0 = ps.ip0; h.tp0 = ps.tp0; h.cmax = ps.cmax;
    float ts = 0.0f;  // in the order of the coverage's c loop
    for (int c = 0; c < 2 * ps.cmax + 1; ++c) ts += a.tab[ps.tp0 + c];
    h.tpsum = ts;
    fh[g] = h;
  }
}

size_t fwd_table_bytes(int64_t nmembers, int64_t ngroups, size_t* group_off) {
  const size_t m = (size_t)nmembers * sizeof(FwdMember);
  if (group_off) *group_off = m;
  return m + (size_t)ngroups * sizeof(FwdHdr);
}

void launch_fwd_table(cudaStream_t st, const LatticeArgs& a, void* table, size_t group_off, int max_members) {
  if (a.ngroups <= 0) return;
  FwdMember* fm = static_cast<FwdMember*>(table);
  FwdHdr* fh = reinterpret_cast<FwdHdr*>(static_cast<char*>(table) + group_off);
  const int W = max_members <= 4 ? 4 : max_members <= 8 ? 8 : max_members <= 16 ? 16 : 32;
  const int grid = (int)(((int64_t)a.ngroups * W + kThreads - 1) / kThreads);
  if (W == 4)
    k_fwd_table<4><<<grid, kThreads, 0, st>>>(a, fm, fh);
  else if (W == 8)
    k_fwd_table<8><<<grid, kThreads, 0, st>>>(a, fm, fh);
  else if (W == 16)
    k_fwd_table<16><<<grid, kThreads, 0, st>>>(a, fm, fh);
  else
    k_fwd_table<32><<<grid, kThreads, 0, st>>>(a, fm, fh);
}

int launch_coverage(cudaStream_t st, const LatticeArgs& a, int t_floats, int x_floats, float* kap,
                    double* partials) {
  (void)configure();
  (void)x_floats;  // coverage interpolates the grid indicator analytically: no X tile
  const int smem = t_floats * 4;
  int* next = reinterpret_cast<int*>(partials + kStatBlocks * 5);  // the launch's group counter
  const int grid = kStatBlocks;
  if (PVR_FWD_DYN) cudaMemsetAsync(next, 0, sizeof(int), st);
  k_lattice_fwd<1><<<grid, kThreads, smem, st>>>(a, t_floats, nullptr, nullptr, nullptr, kap, partials, next);
  return grid;
}

void launch_forward(cudaStream_t st, const LatticeArgs& a, int t_floats, int x_floats, const void* tmaps,
                    const float* kap, const float* p, float* e, double* partials) {
  (void)configure();
  const int smem = (t_floats + x_floats) * 4;
  int* next = reinterpret_cast<int*>(partials + kStatBlocks * 5);  // the launch's group counter
  if (PVR_FWD_DYN) cudaMemsetAsync(next, 0, sizeof(int), st);
  k_lattice_fwd<0><<<kStatBlocks, kThreads, smem, st>>>(a, t_floats, (const char*)tmaps, kap, p, e,
                                                        partials, next);
}

size_t bp_table_bytes(int64_t nmembers, int64_t ngroups, size_t* group_off) {
  const size_t m = (size_t)nmembers * sizeof(BpMember);
  if (group_off) *group_off = m;
  return m + (size_t)ngroups * sizeof(BpGroupHdr) + 16;  // + the launch's group counter
}

void launch_bp_table(cudaStream_t st, const LatticeArgs& a, void* table, size_t group_off, int max_members) {
  if (a.ngroups <= 0) return;
  BpMember* tm = static_cast<BpMember*>(table);
  BpGroupHdr* th = reinterpret_cast<BpGroupHdr*>(static_cast<char*>(table) + group_off);
  const int64_t threads = (int64_t)a.ngroups * (max_members <= 4 ? 4 : max_members <= 8 ? 8 : max_members <= 16 ? 16 : 32);
  const int grid = (int)((threads + kThreads - 1) / kThreads);
  if (max_members <= 4)
    k_bp_table<4><<<grid, kThreads, 0, st>>>(a, tm, th);
  else if (max_members <= 8)
    k_bp_table<8><<<grid, kThreads, 0, st>>>(a, tm, th);
  else if (max_members <= 16)
    k_bp_table<16><<<grid, kThreads, 0, st>>>(a, tm, th);
  else
    k_bp_table<32><<<grid, kThreads, 0, st>>>(a, tm, th);
}

void launch_backproject(cudaStream_t st, const LatticeArgs& a, int tile_words, int r_bytes,
                        void* table, size_t group_off, bool build_table, int max_members, const float* kap,
                        const float* e, const float* p, const float* w, int init, float2* AC) {
  if (a.ngroups <= 0) return;
  const DevConfig& dc = configure();
  BpMember* tm = static_cast<BpMember*>(table);
  BpGroupHdr* th = reinterpret_cast<BpGroupHdr*>(static_cast<char*>(table) + group_off);
  int* next = reinterpret_cast<int*>(th + a.ngroups);
  if (build_table) launch_bp_table(st, a, table, group_off, max_members);
#if PVR_BP_DYN
  const int per = dc.nsm * (dc.resident > 0 ? dc.resident : 1);
  const int grid = a.ngroups < per ? a.ngroups : per;
  cudaMemsetAsync(next, 0, sizeof(int), st);
#else
  (void)dc;
  const int grid = a.ngroups < 148 * 16 ? a.ngroups : 148 * 16;
#endif
  if (a.prm.det)
    k_lattice_bp<true><<<grid, kBpThreads, kBpTileBytes + r_bytes, st>>>(a, tile_words, tm, th, kap, e, p, w, init, AC,
                                                                       next);
  else
    k_lattice_bp<false><<<grid, kBpThreads, kBpTileBytes + r_bytes, st>>>(a, tile_words, tm, th, kap, e, p, w, init, AC,
                                                                        next);
}

}  // namespace pvr
