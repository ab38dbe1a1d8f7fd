// Microbenchmark 2 for the backprojection design (a5): accumulate-
// primitive throughput with cheap (register) address generation so the primitive, not the
// address arithmetic, is the bottleneck. Patterns:
//   spread : lanes of a warp hit distinct addresses (stride 37 words)
//   lattice: lane i hits base + floor(i * 5 / 6)  (lattice pitch 0.83 voxel: neighbours collide)
// Primitives: LDS gather, ATOMS.ADD int32, ATOMS.CAS f32 (atomicAdd float), red.global.add.v2.f32
// (L2-resident), red.global.add.v4.f32 coalesced (a warp flushes 32 consecutive float4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_atomics2 tools/ubench_atomics2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int WORDS = 8192;  // 32 KB tile
constexpr int ITERS = 512;

template <int MODE>  // 0 LDS, 1 ATOMS int, 2 f32 atomicAdd (CAS), 3 ATOMS u64 (packed A|C pair)
__global__ void k_smem(float* out, int pattern) {
  __shared__ float s[WORDS];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) s[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int off = pattern == 0 ? lane * 37 : (lane * 5) / 6;
  int b = (blockIdx.x * 977 + (threadIdx.x >> 5) * 131) & (WORDS - 1);
  float acc = 0.f;
  for (int it = 0; it < ITERS; ++it) {
    b = (b + 1031) & (WORDS / 2 - 1);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      int a = b + off + (c & 1) + ((c >> 1) & 1) * 32 + (c >> 2) * 1024;
      if (MODE == 0) acc += s[a];
      else if (MODE == 1) atomicAdd(reinterpret_cast<int*>(&s[a]), it);
      else if (MODE == 3) atomicAdd(reinterpret_cast<unsigned long long*>(&s[2 * (a & (WORDS / 2 - 1))]), (unsigned long long)it);
      else atomicAdd(&s[a], 1.0f);
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + s[threadIdx.x];
}

__global__ void k_gred_v2(float2* g, int region_mask, int pattern) {
  const int lane = threadIdx.x & 31;
  int off = pattern == 0 ? lane * 37 : (lane * 5) / 6;
  int b = (blockIdx.x * 7919 + (threadIdx.x >> 5) * 131) & region_mask;
  for (int it = 0; it < ITERS / 4; ++it) {
    b = (b + 104729) & region_mask;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float2* p = g + b + off + (c & 1) + ((c >> 1) & 1) * 427 + (c >> 2) * 427 * 427;
      asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(2.f) : "memory");
    }
  }
}

__global__ void k_flush_v4(float4* g, int region_mask) {
  // each warp flushes 32 consecutive float4 (= 64 voxels of interleaved (A, C))
  int b = ((blockIdx.x * 8 + (threadIdx.x >> 5)) * 32 * 7) & region_mask;
  for (int it = 0; it < ITERS / 4; ++it) {
    b = (b + 32 * 1031) & region_mask;
    float4* p = g + b + (threadIdx.x & 31);
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f) : "memory");
  }
}

__global__ void k_flush_v2(float2* g, int region_mask) {
  int b = ((blockIdx.x * 8 + (threadIdx.x >> 5)) * 32 * 7) & region_mask;
  for (int it = 0; it < ITERS / 4; ++it) {
    b = (b + 32 * 1031) & region_mask;
    float2* p = g + b + (threadIdx.x & 31);
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(2.f) : "memory");
  }
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  const double clk = p.clockRate * 1e3;
  const int threads = 256, blocks = sms * 6 * 8;
  float* out;
  float2* g2;
  float4* g4;
  const int region = 1 << 26;  // 64M float2 = 512 MB (beyond L2)
  CK(cudaMalloc(&out, (size_t)blocks * threads * 4));
  CK(cudaMalloc(&g2, (size_t)region * 8 + (1 << 24)));
  CK(cudaMalloc(&g4, (size_t)region * 16 / 2 + (1 << 24)));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto rep = [&](const char* name, float ms, double lane_ops) {
    printf("%-40s %8.3f ms %9.1f Glane-op/s %6.2f lane-op/SM/clk\n", name, ms, lane_ops / ms * 1e-6,
           lane_ops / (ms * 1e-3) / sms / clk);
  };
  const double smem_ops = (double)blocks * threads * ITERS * 8;
  for (int r = 0; r < 2; ++r) {
    for (int pat = 0; pat < 2; ++pat) {
      const char* pn = pat ? "lattice" : "spread";
      char nm[64];
      float ms;
      cudaEventRecord(a); k_smem<0><<<blocks, threads>>>(out, pat); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); snprintf(nm, 64, "LDS gather (%s)", pn); rep(nm, ms, smem_ops);
      cudaEventRecord(a); k_smem<1><<<blocks, threads>>>(out, pat); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); snprintf(nm, 64, "ATOMS.ADD int32 (%s)", pn); rep(nm, ms, smem_ops);
      cudaEventRecord(a); k_smem<3><<<blocks, threads>>>(out, pat); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); snprintf(nm, 64, "ATOMS.ADD u64 (%s)", pn); rep(nm, ms, smem_ops);
      cudaEventRecord(a); k_smem<2><<<blocks, threads>>>(out, pat); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); snprintf(nm, 64, "atomicAdd f32 smem CAS (%s)", pn); rep(nm, ms, smem_ops);
      cudaEventRecord(a); k_gred_v2<<<blocks, threads>>>(g2, (1 << 24) - 1, pat); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); snprintf(nm, 64, "red.global.v2 16M-entry region (%s)", pn); rep(nm, ms, smem_ops / 4);
    }
    float ms;
    const double fl = (double)blocks * threads * (ITERS / 4);
    cudaEventRecord(a); k_flush_v4<<<blocks, threads>>>(g4, (region / 2 - 1) & ~31); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); rep("flush red.global.v4 coalesced (float4 ops)", ms, fl);
    printf("    = %.1f GB/s of (A,C) payload\n", fl * 16 / (ms * 1e-3) * 1e-9);
    cudaEventRecord(a); k_flush_v2<<<blocks, threads>>>(g2, (region - 1) & ~31); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); rep("flush red.global.v2 coalesced (float2 ops)", ms, fl);
    printf("    = %.1f GB/s of (A,C) payload\n", fl * 8 / (ms * 1e-3) * 1e-9);
  }
  CK(cudaGetLastError());
  return 0;
}
