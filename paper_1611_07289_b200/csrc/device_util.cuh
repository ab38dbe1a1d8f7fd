// device_util.cuh — small device helpers shared by kernels.cu and lattice.cu (product only).
#pragma once
#include <cfloat>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pvr {

// Debug builds (-DPVR_CHECKS=1, tools/ab_build.py): device-side bounds checks of the shared
// tiles and the global reductions; a violation traps (the launch fails with an error). The
// compute-sanitizer is closed on this GPU pool, so these stand in for memcheck.
#ifdef PVR_CHECKS
#define PVR_CHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define PVR_CHECK(cond) \
  do {                  \
  } while (0)
#endif

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

// Packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2: two lanes of fp32 math per issue slot).
// A scalar operand is broadcast by the hardware (R.F32 operand), so pk(s, s) costs nothing.
struct f2 {
  unsigned long long v;
};
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo2(f2 a) {
  float l;
  asm("{.reg .f32 t; mov.b64 {%0, t}, %1;}" : "=f"(l) : "l"(a.v));
  return l;
}
__device__ __forceinline__ float hi2(f2 a) {
  float h;
  asm("{.reg .f32 t; mov.b64 {t, %0}, %1;}" : "=f"(h) : "l"(a.v));
  return h;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 add2_rd(f2 a, f2 b) {
  f2 r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
__device__ __forceinline__ f2 mul2s(float s, f2 b) { return mul2(pk(s, s), b); }
__device__ __forceinline__ f2 fma2s(float s, f2 b, f2 c) { return fma2(pk(s, s), b, c); }

// Shared-memory integer reduction at a 32-bit shared address (+ immediate byte offset).
template <int OFF>
__device__ __forceinline__ void sred(unsigned addr, int v) {
  asm volatile("red.shared.add.s32 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(OFF) : "memory");
}

__device__ __forceinline__ int floor_div(int a, int b) {  // b > 0
  int q = a / b;
  return (a % b != 0 && a < 0) ? q - 1 : q;
}

}  // namespace pvr
