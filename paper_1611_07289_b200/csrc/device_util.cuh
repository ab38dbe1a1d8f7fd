// device_util.cuh — small device helpers shared by kernels.cu and lattice.cu (product only).
#pragma once
#include <cfloat>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pvr {

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

// Block-reduce NS sums (double) and NM maxima (float) of the CTA into out[] (thread 0 writes
// out[0..NS+NM)). Deterministic: fixed warp and tree order. Ends with a barrier.
template <int NS, int NM>
__device__ __forceinline__ void block_reduce_store(double (&s)[NS], float (&mx)[NM], double* out) {
  __shared__ double sh_s[32][NS > 0 ? NS : 1];
  __shared__ float sh_m[32][NM > 0 ? NM : 1];
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
  __syncthreads();
}

__device__ __forceinline__ void red_v2(float2* addr, float a, float c) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(c) : "memory");
}
__device__ __forceinline__ void red_v4(float2* addr, float a0, float c0, float a1, float c1) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a0), "f"(c0),
               "f"(a1), "f"(c1)
               : "memory");
}

// floor(x) for |x| < 2^22 without the conversion pipe: x + 1.5 * 2^23 rounded toward -inf
// (FADD.RM) holds floor(x) in its low mantissa bits; fl = float(floor(x)) exactly.
__device__ __forceinline__ int mfloor(float x, float& fl) {
  const float t = __fadd_rd(x, 12582912.0f);
  fl = __fsub_rn(t, 12582912.0f);
  return __float_as_int(t) - 0x4B400000;
}

__device__ __forceinline__ int floor_div(int a, int b) {  // b > 0
  int q = a / b;
  return (a % b != 0 && a < 0) ? q - 1 : q;
}

}  // namespace pvr
