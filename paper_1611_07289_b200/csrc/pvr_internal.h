// pvr_internal.h — device-side data layout and kernel launchers of libpvr.so.
// Private to the product (engine.cu + kernels.cu); see DESIGN.md §Data layout.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pvr {

// One patch of the local shard, composed on the host in fp64 (engine.cu) and uploaded
// as fp32. Continuous voxel index of PSF lattice point (a, b, c) of pixel (u, v, z):
//   x = base + frac + u*Mu + v*Mv + z*Mz + a*Qa + b*Qb + c*Qc
// with Mu = n_u*Qa and Mv = n_v*Qb (the in-plane PSF lattice is commensurate with the
// pixel pitch, reading Q5). `base` is an integer voxel so the fp32 part stays small.
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
  int32_t psf0, S;            // this stack's PSF samples: psf[psf0 .. psf0+S)
  int32_t pad[2];
};

// EM state on the device (written by k_em_params / k_range, read by later kernels).
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
};

struct Params {
  float tau_live, tau_obs, tau_C, tau_patch;
  float c0, delta;
  int clamp;
};

constexpr int kTile = 256;        // pixels per forward / backprojection tile
constexpr int kStatBlocks = 1184; // 148 SMs x 8: fixed grid of the statistics kernels

// ---- launchers (kernels.cu); all asynchronous on `st` ----
void launch_coverage(cudaStream_t st, const PatchDev* P, const float4* psf, const int2* tiles,
                     int64_t ntiles, const float* ystack, const int3 dims, Params prm, float* kap,
                     double* partials);
void launch_range_finish(cudaStream_t st, double s2floor, EmDev* em);
void launch_fill(cudaStream_t st, float* x, int64_t n, float v);
void launch_forward(cudaStream_t st, const PatchDev* P, const float4* psf, const int2* tiles,
                    int64_t ntiles, const float* ystack, const float* X, const int3 dims,
                    Params prm, const float* kap, const float* p, float* e, double* partials);
void launch_em_reduce(cudaStream_t st, const double* partials, int nblk, EmDev* em);
void launch_em_params(cudaStream_t st, Params prm, EmDev* em);
void launch_estep(cudaStream_t st, const PatchDev* P, int64_t npatch, Params prm, const EmDev* em,
                  const float* kap, const float* e, float* p, float* pbar, float* w);
void launch_backproject(cudaStream_t st, const PatchDev* P, const float4* psf, const int2* tiles,
                        int64_t ntiles, const float* ystack, const int3 dims, Params prm,
                        const float* kap, const float* e, const float* p, const float* w, int init,
                        float2* AC);
void launch_update(cudaStream_t st, const float* X0, const float2* AC, const int3 dims, Params prm,
                   const EmDev* em, float alpha, float lambda, float* X2);
void launch_init_fill(cudaStream_t st, const float2* AC, const int3 dims, Params prm, float* X);

}  // namespace pvr
