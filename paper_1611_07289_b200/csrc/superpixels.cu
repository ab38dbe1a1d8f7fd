// superpixels.cu — f3 (Eq. 3 P:140-145 "superpixels ... SLIC"; P:154 dilation;
// DESIGN.md readings Q32, Q33): integer SLIC on every slice of a stack, on the device.
//
// The algorithm is oracle/pvro.c pvro_slic exactly, in integer arithmetic so that every
// label decision is bit-exact on both sides: intensities quantised to 10 bits over the stack's
// range in fp64 (I = floor(1023 (y - ymin) / (ymax - ymin) + 0.5), IEEE-rounded operations in
// the same order), cluster centres in 1/16 units on the S-grid, each pixel picks the smallest
// D = S^2 (16 I - cI)^2 + m^2 ((16 x - cx)^2 + (16 y - cy)^2) among the 3 x 3 neighbouring grid
// cells' centres (ties to the lowest cluster index), centres move to the rounded means.
// All K slices of a stack run together: one thread per pixel (assignment, accumulation) or per
// centre (update); the accumulation aggregates equal labels within a warp (__match_any_sync)
// before its 64-bit global atomics.
#include <cstdint>

#include "device_util.cuh"
#include "pvr_internal.h"

namespace pvr {

namespace {

__device__ __forceinline__ int quant(float y, float ymin, float ymax) {
  if (!(ymax > ymin)) return 0;
  const double t = __ddiv_rn(__dmul_rn(__dsub_rn((double)y, (double)ymin), 1023.0),
                             __dsub_rn((double)ymax, (double)ymin));
  return (int)floor(__dadd_rn(t, 0.5));
}

struct SlicArgs {
  const float* y;      // stack [K][H][W]
  int W, H, K, S, m, nxc, nyc;
  float ymin, ymax;
  int64_t* c;          // centres [K][nc][3] (cx, cy, cI) in 1/16 units
  unsigned long long* acc;  // [K][nc][4] (n, sum x, sum y, sum I)
  int32_t* lab;        // [K][H][W]
};

__global__ void k_slic_init(SlicArgs a) {
  const int nc = a.nxc * a.nyc;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * a.K) return;
  const int z = (int)(t / nc), k = (int)(t % nc), i = k % a.nxc, j = k / a.nxc;
  const int px = min(i * a.S + a.S / 2, a.W - 1), py = min(j * a.S + a.S / 2, a.H - 1);
  int64_t* c = a.c + 3 * t;
  c[0] = 16 * (int64_t)px;
  c[1] = 16 * (int64_t)py;
  c[2] = 16 * (int64_t)quant(a.y[((int64_t)z * a.H + py) * a.W + px], a.ymin, a.ymax);
}

__global__ void k_slic_assign(SlicArgs a, int accumulate) {
  const int64_t HW = (int64_t)a.H * a.W;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < HW * a.K;
  int z = 0, x = 0, y = 0, bk = 0, I = 0;
  if (live) {
    z = (int)(t / HW);
    const int r = (int)(t - z * HW);
    y = r / a.W;
    x = r - y * a.W;
    I = quant(a.y[t], a.ymin, a.ymax);
    const int64_t I16 = 16 * (int64_t)I, S2 = (int64_t)a.S * a.S, m2 = (int64_t)a.m * a.m;
    const int ci = x / a.S, cj = y / a.S, nc = a.nxc * a.nyc;
    const int64_t* cz = a.c + 3 * (int64_t)z * nc;
    int64_t best = INT64_MAX;
    bk = -1;
    for (int dj = -1; dj <= 1; ++dj)
      for (int di = -1; di <= 1; ++di) {
        const int i = ci + di, j = cj + dj;
        if (i < 0 || i >= a.nxc || j < 0 || j >= a.nyc) continue;
        const int k = j * a.nxc + i;
        const int64_t dI = I16 - cz[3 * k + 2], dx = 16 * (int64_t)x - cz[3 * k], dy = 16 * (int64_t)y - cz[3 * k + 1];
        const int64_t D = S2 * dI * dI + m2 * (dx * dx + dy * dy);
        if (D < best) { best = D; bk = k; }
      }
    a.lab[t] = bk;
  }
  if (!accumulate) return;
  // per-cluster sums; lanes with equal (slice, label) combine before the atomics
  const unsigned active = __ballot_sync(0xffffffffu, live);
  if (!live) return;
  const int key = z * (a.nxc * a.nyc) + bk;
  const unsigned peers = __match_any_sync(active, key);
  const int leader = __ffs(peers) - 1;
  unsigned long long s[4] = {1ull, (unsigned long long)x, (unsigned long long)y, (unsigned long long)I};
  for (int q = 0; q < 4; ++q) {
    unsigned long long v = s[q], tot = 0;
    // sum over the peer lanes (a reduction by key without a fixed tree: peers are few)
    unsigned rem = peers;
    while (rem) {
      const int l = __ffs(rem) - 1;
      tot += __shfl_sync(peers, v, l);
      rem &= rem - 1;
    }
    s[q] = tot;
  }
  if ((int)(threadIdx.x & 31) == leader) {
    unsigned long long* acc = a.acc + 4 * (int64_t)key;
    for (int q = 0; q < 4; ++q) atomicAdd(acc + q, s[q]);
  }
}

__global__ void k_slic_update(SlicArgs a) {
  const int nc = a.nxc * a.nyc;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * a.K) return;
  const unsigned long long* s = a.acc + 4 * t;
  const int64_t n = (int64_t)s[0];
  if (n == 0) return;
  int64_t* c = a.c + 3 * t;
  c[0] = (16 * (int64_t)s[1] + n / 2) / n;
  c[1] = (16 * (int64_t)s[2] + n / 2) / n;
  c[2] = (16 * (int64_t)s[3] + n / 2) / n;
}

// stack range (min, max) of a float array: per-block partials, then one block
__global__ void k_minmax(const float* __restrict__ y, int64_t n, float* __restrict__ part) {
  float lo = 3.4e38f, hi = -3.4e38f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    lo = fminf(lo, y[i]);
    hi = fmaxf(hi, y[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ float sl[32], sh[32];
  if ((threadIdx.x & 31) == 0) { sl[threadIdx.x >> 5] = lo; sh[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fminf(lo, sl[w]); hi = fmaxf(hi, sh[w]); }
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
  }
}

}  // namespace

// SLIC labels [K][H][W] (device) of one stack y [K][H][W] (device). Scratch is allocated here.
cudaError_t slic_stack(cudaStream_t st, const float* y, int W, int H, int K, int S, int m, int iters,
                       int32_t* lab) {
  const int nxc = (W + S - 1) / S, nyc = (H + S - 1) / S, nc = nxc * nyc;
  const int64_t npx = (int64_t)W * H * K, ncl = (int64_t)nc * K;
  float* part = nullptr;
  int64_t* c = nullptr;
  unsigned long long* acc = nullptr;
  cudaError_t e = cudaMalloc(&part, 2 * 148 * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&c, 3 * ncl * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc(&acc, 4 * ncl * sizeof(unsigned long long));
  float rng[2 * 148];
  if (e == cudaSuccess) {
    k_minmax<<<148, 1024, 0, st>>>(y, npx, part);
    e = cudaMemcpyAsync(rng, part, sizeof(rng), cudaMemcpyDeviceToHost, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    float lo = rng[0], hi = rng[1];
    for (int b = 1; b < 148; ++b) { lo = fminf(lo, rng[2 * b]); hi = fmaxf(hi, rng[2 * b + 1]); }
    SlicArgs a{y, W, H, K, S, m, nxc, nyc, lo, hi, c, acc, lab};
    const unsigned gc = (unsigned)((ncl + 255) / 256), gp = (unsigned)((npx + 255) / 256);
    k_slic_init<<<gc, 256, 0, st>>>(a);
    for (int it = 0; it < iters; ++it) {
      cudaMemsetAsync(acc, 0, 4 * ncl * sizeof(unsigned long long), st);
      k_slic_assign<<<gp, 256, 0, st>>>(a, 1);
      k_slic_update<<<gc, 256, 0, st>>>(a);
    }
    k_slic_assign<<<gp, 256, 0, st>>>(a, 0);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  cudaFree(part);
  cudaFree(c);
  cudaFree(acc);
  return e;
}

}  // namespace pvr
