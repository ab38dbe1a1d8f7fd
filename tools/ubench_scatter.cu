// Microbenchmark for the backprojection design choice:
// throughput of the accumulate primitives a trilinear splat can use on sm_100a.
//   1. shared-memory fp32 atomicAdd   (compiles to an ATOMS.CAST.SPIN CAS loop)
//   2. shared-memory int32 atomicAdd  (native ATOMS.ADD; fixed-point splat)
//   3. global red.add.v2.f32 into an L2-resident buffer (REDG.F32x2)
//   4. global red.add.f32 into an L2-resident buffer
//   5. shared-memory random gather (LDS)
//   6. global random gather through L1 (LDG, L1/L2 resident)
// Addresses follow a "lattice splat" pattern: each lane walks a pseudo-random
// base inside a 16K-entry tile and touches 8 trilinear corners around it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench_scatter.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int NX = 32, NY = 32, NZ = 8;             // 8192-entry tile (32 KB)
constexpr int TILE = NX * NY * NZ;
constexpr int ITERS = 256;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ int base_of(uint32_t h) {
  int i = h % (NX - 1), j = (h >> 8) % (NY - 1), l = (h >> 16) % (NZ - 1);
  return (l * NY + j) * NX + i;
}

__global__ void k_smem_f32(float* out) {
  __shared__ float s[TILE];
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) s[i] = 0.f;
  __syncthreads();
  uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
    // lanes of a warp splat neighbouring lattice points (coherent, like a real tile)
    int b = base_of(hash(seed / 32 * 977 + it)) + (threadIdx.x & 7) + ((threadIdx.x >> 3) & 3) * NX;
    b = b % (TILE - NX * NY - NX - 1);
    float v = 1.0f + it;
#pragma unroll
    for (int c = 0; c < 8; ++c) atomicAdd(&s[b + (c & 1) + ((c >> 1) & 1) * NX + (c >> 2) * NX * NY], v);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) out[blockIdx.x * TILE + i] = s[i];
}

__global__ void k_smem_i32(int* out) {
  __shared__ int s[TILE];
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
    int b = base_of(hash(seed / 32 * 977 + it)) + (threadIdx.x & 7) + ((threadIdx.x >> 3) & 3) * NX;
    b = b % (TILE - NX * NY - NX - 1);
    int v = 1 + it;
#pragma unroll
    for (int c = 0; c < 8; ++c) atomicAdd(&s[b + (c & 1) + ((c >> 1) & 1) * NX + (c >> 2) * NX * NY], v);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) out[blockIdx.x * TILE + i] = s[i];
}

__global__ void k_gred_v2(float2* g, int region) {
  uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
  int off = (hash(blockIdx.x) % (region / TILE)) * TILE;
  for (int it = 0; it < ITERS; ++it) {
    int b = base_of(hash(seed / 32 * 977 + it)) + (threadIdx.x & 7) + ((threadIdx.x >> 3) & 3) * NX;
    b = b % (TILE - NX * NY - NX - 1);
    float v = 1.0f + it;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float2* p = g + off + b + (c & 1) + ((c >> 1) & 1) * NX + (c >> 2) * NX * NY;
      asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v), "f"(v) : "memory");
    }
  }
}

__global__ void k_gred_f32(float* g, int region) {
  uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
  int off = (hash(blockIdx.x) % (region / TILE)) * TILE;
  for (int it = 0; it < ITERS; ++it) {
    int b = base_of(hash(seed / 32 * 977 + it)) + (threadIdx.x & 7) + ((threadIdx.x >> 3) & 3) * NX;
    b = b % (TILE - NX * NY - NX - 1);
    float v = 1.0f + it;
#pragma unroll
    for (int c = 0; c < 8; ++c) atomicAdd(g + off + b + (c & 1) + ((c >> 1) & 1) * NX + (c >> 2) * NX * NY, v);
  }
}

__global__ void k_lds(float* out) {
  __shared__ float s[TILE];
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) s[i] = i * 0.5f;
  __syncthreads();
  uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int it = 0; it < ITERS; ++it) {
    int b = base_of(hash(seed / 32 * 977 + it)) + (threadIdx.x & 7) + ((threadIdx.x >> 3) & 3) * NX;
    b = b % (TILE - NX * NY - NX - 1);
#pragma unroll
    for (int c = 0; c < 8; ++c) acc += s[b + (c & 1) + ((c >> 1) & 1) * NX + (c >> 2) * NX * NY];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_ldg(const float* __restrict__ g, float* out, int region) {
  uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
  int off = (hash(blockIdx.x) % (region / TILE)) * TILE;
  float acc = 0.f;
  for (int it = 0; it < ITERS; ++it) {
    int b = base_of(hash(seed / 32 * 977 + it)) + (threadIdx.x & 7) + ((threadIdx.x >> 3) & 3) * NX;
    b = b % (TILE - NX * NY - NX - 1);
#pragma unroll
    for (int c = 0; c < 8; ++c) acc += __ldg(g + off + b + (c & 1) + ((c >> 1) & 1) * NX + (c >> 2) * NX * NY);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("device %s, %d SMs, clock %d kHz\n", p.name, sms, p.clockRate);
  const int threads = 256;
  const int blocks = sms * 4 * 4;                    // 4+ CTAs/SM resident (32 KB smem each) x 4 waves
  const int region = 16 * 1024 * 1024;               // 16M entries: 128 MB of float2 (L2-ish), 64 MB of f32
  float* fout; int* iout; float2* g2; float* g1; float* gsrc;
  CK(cudaMalloc(&fout, (size_t)blocks * TILE * 4));
  CK(cudaMalloc(&iout, (size_t)blocks * TILE * 4));
  CK(cudaMalloc(&g2, (size_t)region * 8));
  CK(cudaMalloc(&g1, (size_t)region * 4));
  CK(cudaMalloc(&gsrc, (size_t)region * 4));
  CK(cudaMemset(g2, 0, (size_t)region * 8)); CK(cudaMemset(g1, 0, (size_t)region * 4));
  CK(cudaMemset(gsrc, 0, (size_t)region * 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  double ops = (double)blocks * threads * ITERS * 8;  // lane-ops
  auto report = [&](const char* name, float ms) {
    double per_s = ops / (ms * 1e-3);
    double per_sm_clk = per_s / sms / (p.clockRate * 1e3);
    printf("%-28s %8.3f ms  %8.2f Glane-op/s  %6.2f lane-op/SM/clk(at max clk)\n", name, ms, per_s * 1e-9, per_sm_clk);
  };
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); k_smem_f32<<<blocks, threads>>>(fout); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); report("smem f32 atomicAdd (CAS)", ms);
    cudaEventRecord(a); k_smem_i32<<<blocks, threads>>>(iout); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); report("smem i32 atomicAdd", ms);
    cudaEventRecord(a); k_gred_v2<<<blocks, threads>>>(g2, region); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); report("global red.v2.f32", ms);
    cudaEventRecord(a); k_gred_f32<<<blocks, threads>>>(g1, region); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); report("global red.f32", ms);
    cudaEventRecord(a); k_lds<<<blocks, threads>>>(fout); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); report("smem gather (LDS)", ms);
    cudaEventRecord(a); k_ldg<<<blocks, threads>>>(gsrc, fout, region); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); report("global gather (LDG)", ms);
  }
  CK(cudaGetLastError());
  return 0;
}
