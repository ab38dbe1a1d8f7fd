// pvr_internal.h — device-side data layout and kernel launchers of libpvr.so.
// Private to the product (engine.cu, kernels.cu, lattice.cu); see DESIGN.md §Data layout.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pvr {

// One patch of the local shard, composed on the host in fp64 (engine.cu) and uploaded as
// fp32. Continuous voxel index of PSF lattice point (a, b, c) of pixel (u, v, z):
//   x = base + frac + u*Mu + v*Mv + z*Mz + a*Qa + b*Qb + c*Qc,
// with Mu = n_u*Qa and Mv = n_v*Qb (the in-plane PSF lattice is commensurate with the pixel
// pitch, reading Q5), so the fine in-plane lattice index U = n_u*u + a addresses it as
//   x = base + frac + z*Mz + U*Qa + V*Qb + c*Qc.
// `base` is an integer voxel so the fp32 part stays small (|frac + ...| <~ patch extent).
struct PatchDev {
  float Mu[3], Mv[3], Mz[3];  // voxel-index step per pixel column / row / slice
  float Qa[3], Qb[3], Qc[3];  // voxel-index step per PSF lattice step a / b / c
  float frac[3];              // position of pixel (0,0,0), lattice (0,0,0), minus base
  int32_t base[3];
  int32_t stack;
  int32_t x0, y0, z0, sx, sy, sz;
  int64_t pix0;               // first pixel of the patch in the local pixel arrays
  int64_t y0off;              // offset of pixel (x0, y0, z0) in the concatenated stacks
  int32_t W, HW;              // row / slice pitch of the patch's stack (elements)
  int32_t S, pad0;            // PSF samples per pixel (direct count)
  // fp64 copies: each CTA forms its tile origin in fp64, then steps in small fp32 offsets
  double t0d[3], Mzd[3], Qad[3], Qbd[3], Qcd[3];
};

// Separable PSF of one stack (in-plane sinc x through-plane slice profile):
// psi(a, b, c) = ip[(b + rv) * (2 ru + 1) + (a + ru)] * tp[c + cmax],
// a in [-ru, ru] (ru = n_u - 1), b in [-rv, rv], c in [-cmax, cmax]; ip is zero outside
// the main-lobe disk R < 1 (reading Q2). Both factors sum to 1.
struct StackPsf {
  int32_t nu, nv, ru, rv, cmax;
  int32_t ip0, tp0;  // offsets into the float table
  float tpmax;       // max over c of tp
};

// Work decomposition of the lattice kernels (engine.cu: build_plan). A member is a tile of
// tu x tv pixels of one slice z of one patch. Members whose pixels cover the same stack
// pixels (overlapping patches of one stack) form a group: one CTA per group, sharing one
// shared-memory accumulation tile of the group's voxel bounding box (backprojection) and the
// same volume footprint in L1 (forward).
struct MemberDev {
  int32_t patch;            // local patch index
  int32_t z, u0, v0, tu, tv;
  int32_t c0, c1;           // through-plane lattice range [c0, c1] (backprojection segments)
  int32_t flags;            // kMemberRim: the member may touch cells at the rim of the
                            // coverage (engine.cu: build_natural) -> exact tile words
};
constexpr int32_t kMemberRim = 1;
struct GroupDev {
  int32_t m0, nm;           // members [m0, m0 + nm)
  int32_t lo[3];            // voxel bbox origin (not clipped to the grid; lo[0] even, forward:
                            // a multiple of 4)
  int32_t dim[3];           // voxel bbox size (row / plane pitches of the shared tile: odd;
                            // forward: dim[0] = 4 x odd, the TMA box width)
  int32_t tmap;             // forward: index of the group's TMA box tensor map
  int32_t interior;         // 1 if every PSF sample's 8 trilinear corners are in the grid
                            // (forward: kappa = sum psi = 1 exactly; coverage skips the lattice)
  int32_t exact;            // backprojection: hi/lo tile words (a rim member, a footprint that
                            // leaves the grid, or PVR_PARAM_BP_EXACT = 2), 16 B per cell; else
                            // one word per quantity, 8 B per cell
};

// EM state on the device (written by k_em_params / k_range_finish, read by later kernels).
struct EmDev {
  double sigma2, c, m;
  double s2min, lo, hi;        // from the live-y range at set_transforms
  double ymin, ymax;
  float logk, inv2s2;          // p = 1 / (1 + exp(logk + e^2 * inv2s2))
  int32_t mode;                // 0 normal, 1 p = 1 (degenerate / c >= 1), 2 p = 0 (c <= 0)
  int32_t pad;
  int64_t t;                   // iterations since set_transforms
  double stats[5];             // reduced {sum p e^2, sum p, n_live, max e, -min e}
                               // (after coverage: {n_obs, n_live, samples_obs, max y, -min y})
  // f4 multi-round EM (reading Q30)
  double stats2[3];            // reduced E-step partials {sum p e^2, sum p, LL} over live pixels
  double ll_prev;              // LL of the round before the last
  float lnbm;                  // ln((1 - c) m): the uniform term of the log-likelihood
  int32_t done;                // rounds converged (or degenerate): later rounds are no-ops
  int32_t degenerate;          // round 1 took the degenerate path
  int32_t rounds;              // E-step rounds run in the last iteration
  // f4 two-Gaussian patch classification (reading Q31)
  double mix_mu[2], mix_v[2], mix_pi, mix_ll_prev;  // [0] inliers, [1] outliers
  double mix_stats[7];         // reduced round sums (see kernels.cu k_mix_round)
  int32_t mix_done, mix_degenerate;
  // deterministic mode: global maxima of the backprojection inputs |rA|, rC (float bits,
  // atomicMax over the ranks' patches) and the global tile scales formed from them
  float det_max[2];
  double det_scale[2];
};

struct Params {
  float tau_live, tau_obs, tau_C, tau_patch;
  float c0, delta;
  int clamp;
  int det;  // PVR_PARAM_DETERMINISTIC: order-independent (integer) reductions everywhere
};

// Everything a lattice kernel needs about the problem (passed by value).
struct LatticeArgs {
  const PatchDev* P;
  const StackPsf* psf;
  const float* tab;        // PSF factor tables
  const MemberDev* mem;
  const GroupDev* grp;
  int32_t ngroups;
  int3 n;                  // volume dims
  int32_t nxp;             // row pitch of X and (A, C) (nx rounded up to a multiple of 4)
  const float* ys;         // concatenated stacks
  const uint8_t* mask;     // f3: per-pixel patch mask (local shard; NULL = all pixels)
  Params prm;
  // deterministic mode: the global tile scales (A, C) and the int64 accumulators, per voxel
  // {A hi, A lo 2^20 + lo2, C hi, C lo 2^20 + lo2} (k_det_to_float forms A, C)
  const double* det_scale;
  unsigned long long* ACd;
  // forward / coverage: the plan's member rows and group headers (k_fwd_table, geometry only;
  // the header array starts fgoff bytes into ftab)
  const void* ftab;
  size_t fgoff;
};

constexpr int kThreads = 256;      // CTA size of the lattice kernels
constexpr int kStatBlocks = 1184;  // 148 SMs x 8: fixed grid of the statistics kernels
#ifndef PVR_BP_TILE_KB
#define PVR_BP_TILE_KB 56
#endif
// Backprojection tile budget (shared memory). An exact group (GroupDev::exact) uses four int32
// planes A_hi, C_hi, A_lo, C_lo of kBpTileBytes / 4 bytes each (16 B per voxel); a
// single-word group two planes A, C of kBpTileBytes / 2 bytes (8 B per voxel).
constexpr int kBpTileBytes = PVR_BP_TILE_KB * 1024;
// Backprojection tile precision (PVR_PARAM_BP_EXACT): 0 one word everywhere (a timing
// reference), 1 exact hi/lo words for rim groups only (default), 2 exact everywhere.
enum { kBpSingle = 0, kBpRim = 1, kBpAll = 2, kBpDet = 3 /* deterministic mode: three words, 24 B */ };
#ifndef PVR_BP_THREADS
#define PVR_BP_THREADS 256
#endif
constexpr int kBpThreads = PVR_BP_THREADS;  // CTA size of the backprojection
#ifndef PVR_BP_CTAS
#define PVR_BP_CTAS (kBpThreads > 256 ? 2 : PVR_BP_TILE_KB <= 56 ? 3 : 2)
#endif
constexpr int kBpCtasPerSm = PVR_BP_CTAS;  // __launch_bounds__ minimum CTAs per SM
constexpr int kBpDetPlane = (kBpTileBytes / 6) & ~15;  // deterministic mode: 6 planes
#ifndef PVR_R_KB
#define PVR_R_KB 12
#endif
constexpr int kRBytes = PVR_R_KB * 1024;   // backprojection: per-pixel (rA, rC) buffer budget
#ifndef PVR_FWD_TILE_KB
#define PVR_FWD_TILE_KB 48
#endif
constexpr int kFwdTileBytes = PVR_FWD_TILE_KB * 1024;  // forward: 4 B/voxel X tile budget
constexpr int kFwdTBytes = 12 * 1024;     // forward: lattice values of a group's members
constexpr int kMaxGroupMembers = 16;      // members per group (lattice.cu kMaxMembers)

// f1 registration (registration.cu): per local patch, pixel (u, v, z) sits at world position
// m0 + u mu + v mv + z mz under its current transform T_s; c = the transformed patch centre.
struct RegPatch {
  double m0[3], mu[3], mv[3], mz[3], c[3];
  int64_t y0off;             // offset of pixel (0, 0, 0) in the concatenated stacks
  int32_t W, HW, sx, sy, sz, pad;
};
struct RegArgs {
  const RegPatch* P;
  const float* X;            // current reconstruction, row pitch nxp
  const float* ys;
  int3 n;
  int32_t nxp;
  double o[3], s;            // voxel (0,0,0) world position and spacing
  int32_t levels, iters, min_valid, pad;
};

// Volume-space PSF mode (volpsf.cu; PVR_PARAM_PSF_MODE = 2, reading Q34): per local patch, the
// voxel index of pixel (u, v, z)'s centre is base + xc + u Mu + v Mv + z Mz; Minv maps an index
// offset to the slice-frame offset (a, b, c) in mm (s [u; v; w] A^-1); h is the half-extent of
// the support's index box.
struct VolPatch {
  float xc[3], Mu[3], Mv[3], Mz[3];
  float Minv[9];
  float h[3];
  float idx, idy, i2s2, cmax;  // 1 / dx, 1 / dy, 1 / (2 sw^2), nsigma sw (mm)
  int32_t base[3];
  int32_t sx, sy, sz, W, HW;
  int64_t pix0, y0off;
  // fp64 copies for the support decisions of voxels within 1e-3 of its edge (R = 1, |c| = cmax)
  double xcd[3], Mud[3], Mvd[3], Mzd[3], Minvd[9];
  double dxd, dyd, cmaxd;
};

// ---- launchers; all asynchronous on `st` ----
// volpsf.cu: mode 0 forward (e, EM partials), 1 coverage (kappa, row normaliser vin, stats),
// 2 adjoint into (A, C) (init as launch_backproject; w per patch, p per pixel)
void launch_volpsf(cudaStream_t st, int mode, const struct VolPatch* VP, int64_t npatch, const LatticeArgs& a,
                   const float* X, float* kap, float* vin, const float* pprev, float* e, double* partials,
                   const float* w, const float* p, int init, float2* AC);
// lattice.cu
// returns the grid it launched: the number of per-block partials to reduce
int launch_coverage(cudaStream_t st, const LatticeArgs& a, int t_floats, int x_floats,
                    float* kap, double* partials);
// tmaps: device array of CUtensorMap (128 B each), one per box shape (GroupDev::tmap), over
// the X buffer to read
void launch_forward(cudaStream_t st, const LatticeArgs& a, int t_floats, int x_floats,
                    const void* tmaps, const float* kap, const float* p, float* e,
                    double* partials);
// init: 0 iteration (w p e / kappa, w p / kappa), 1 init pass (y / kappa, 1 / kappa),
// 2 rigidity pass (p pbar / kappa, 1 / kappa; w carries pbar)
// `table`: the plan's per-member / per-group constants (bp_table_bytes; members first, the
// group headers at byte `group_off`, then the launch's int group counter), geometry only:
// rebuilt by this launch when `build_table` (after a set_transforms / re-plan), else reused.
size_t bp_table_bytes(int64_t nmembers, int64_t ngroups, size_t* group_off);
// Member tables of a backprojection plan alone (geometry only): set_transforms builds them on an
// auxiliary stream, overlapped with the coverage pass.
void launch_bp_table(cudaStream_t st, const LatticeArgs& a, void* table, size_t group_off, int max_members);
// Member rows and group headers of a forward plan (geometry only): built by set_transforms
// before the coverage pass, read by every forward.
size_t fwd_table_bytes(int64_t nmembers, int64_t ngroups, size_t* group_off);
void launch_fwd_table(cudaStream_t st, const LatticeArgs& a, void* table, size_t group_off, int max_members);
// Each group's tile precision is GroupDev::exact (init / rigidity passes: always exact).
void launch_backproject(cudaStream_t st, const LatticeArgs& a, int tile_words, int r_bytes,
                        void* table, size_t group_off, bool build_table, int max_members, const float* kap,
                        const float* e, const float* p, const float* w, int init, float2* AC);
// superpixels.cu (f3): SLIC labels [K][H][W] (device) of one stack (device), synchronous
cudaError_t slic_stack(cudaStream_t st, const float* y, int W, int H, int K, int S, int m, int iters,
                       int32_t* lab);
// registration.cu (f1)
void launch_register(cudaStream_t st, const RegArgs& a, int nloc, int max_pix, float* pose, int32_t* status);
void launch_patch_cc(cudaStream_t st, const RegArgs& a, int n, int max_pix, const int32_t* which,
                     const float* poses, double* out);
// kernels.cu
void launch_range_finish(cudaStream_t st, double s2floor, EmDev* em);
void launch_fill(cudaStream_t st, float* x, int64_t n, float v);
void launch_em_reduce(cudaStream_t st, const double* partials, int nblk, EmDev* em);
void launch_em_params(cudaStream_t st, Params prm, EmDev* em);
// round 1: always runs; round >= 2: a no-op once em->done. rpart [npatch][3] (may be NULL):
// per-patch {sum p e^2, sum p, LL} over live pixels for the next M-step.
void launch_estep(cudaStream_t st, const PatchDev* P, int64_t npatch, Params prm, EmDev* em,
                  const float* kap, const float* e, float* p, float* pbar, float* w, int round,
                  double* rpart, int32_t* nlive);
void launch_em_reduce3(cudaStream_t st, const double* rpart, int64_t npatch, EmDev* em);
// f4 patch mixture: nlive [npatch] from the last E-step (launch_estep's nlive output)
void launch_mix_init(cudaStream_t st, const float* pbar, const int32_t* nlive, int64_t npatch, EmDev* em);
void launch_mix_params_init(cudaStream_t st, EmDev* em);
void launch_mix_round(cudaStream_t st, const float* pbar, const int32_t* nlive, int64_t npatch, EmDev* em, float* r);
void launch_mix_update(cudaStream_t st, EmDev* em, int round, double tol);
void launch_mix_weights(cudaStream_t st, const int32_t* nlive, int64_t npatch, const EmDev* em, float* w);
void launch_em_round(cudaStream_t st, Params prm, EmDev* em, int round, double tol);
// planes [zlo, zhi) only (a rank's slab; the stencil reads the planes on either side)
void launch_update(cudaStream_t st, const float* X0, const float2* AC, const int3 dims, int nxp,
                   Params prm, const EmDev* em, float alpha, float lambda, float* X2, int zlo, int zhi);
void launch_unpack_ac(cudaStream_t st, const float2* AC, int3 dims, int nxp, int which, float* out);
void launch_scale(cudaStream_t st, float* x, int64_t n, float f);
// deterministic mode: per-patch maxima of the backprojection inputs into em->det_max (init:
// 0 iteration, 1 init, 2 rigidity, as launch_backproject), the global scales from them, and the
// int64 accumulators into the float (A, C) volume
void launch_bp_maxima(cudaStream_t st, const PatchDev* P, int64_t npatch, Params prm, const float* kap,
                      const float* e, const float* p, const float* w, const float* ys, int init, EmDev* em);
void launch_det_scales(cudaStream_t st, EmDev* em);
void launch_det_to_float(cudaStream_t st, const unsigned long long* ACd, int64_t Vp, const EmDev* em, float2* AC);
constexpr float kDetTermMax = 16384.0f;  // 2^14: deterministic mode's largest splat term (window
                                         // sums < 2^22 for lines of up to 255 samples)
void launch_ratio(cudaStream_t st, const float2* AC, const int3 dims, int nxp, float tau_C, float* out);
constexpr int kMaxBoxShapes = 4096;  // forward TMA box shapes the device re-plan may pick from
// nappend (backprojection): counter of single-member groups appended after ngroups (< cap)
// bp_mode (backprojection): PVR_PARAM_BP_EXACT; vox_budget: forward voxels, backprojection
// tile bytes (a group needs 16 B per cell if exact, else 8)
void launch_replan(cudaStream_t st, const MemberDev* mem, GroupDev* grp, int ngroups, int cap, const PatchDev* P,
                   const StackPsf* psf, int fwd, int3 n, int64_t vox_budget, const int* shapes, int nshape,
                   int* maxvox, int* fail, int* nappend, int bp_mode);
void launch_init_fill(cudaStream_t st, const float2* AC, const int3 dims, int nxp, Params prm,
                      float* X);

}  // namespace pvr
