// tma_check.cu -- standalone check of the forward's TMA staging pattern (3D tiled copy of a
// pitched fp32 volume into a dense shared box, zero fill out of bounds, mbarrier completion),
// with the tensor map in global memory (mode 0) or as a __grid_constant__ parameter (mode 1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_check tools/tma_check.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

__device__ int g_variant;
__device__ void load_box(const void* tm, int x0, int y0, int z0, int bx, int by, int bz, float* out) {
  extern __shared__ __align__(128) float sbuf[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned sraw = (unsigned)__cvta_generic_to_shared(sbuf);
  const unsigned s0 = (g_variant & 1) ? ((sraw + 127u) & ~127u) : sraw;
  float* sb = sbuf + (s0 - sraw) / 4;
  const int slab = (bx * by + 31) & ~31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    if (g_variant & 2) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (g_variant & 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bz * bx * by * 4) : "memory");
    for (int z = 0; z < bz; ++z)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(s0 + 4u * (unsigned)(z * slab)),
          "l"(tm), "r"(x0), "r"(y0), "r"(z0 + z), "r"(b)
          : "memory");
  }
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b), "r"(0u) : "memory");
  __syncthreads();
  for (int i = threadIdx.x; i < bx * by * bz; i += blockDim.x) {
    const int x = i % bx, y = (i / bx) % by, z = i / (bx * by);
    out[i] = sb[z * slab + y * bx + x];
  }
}

__global__ void k_global(const void* tm, int x0, int y0, int z0, int bx, int by, int bz, float* out) {
  load_box(tm, x0, y0, z0, bx, by, bz, out);
}
__global__ void k_param(const __grid_constant__ CUtensorMap tm, int x0, int y0, int z0, int bx, int by, int bz,
                        float* out) {
  load_box(&tm, x0, y0, z0, bx, by, bz, out);
}

int main(int argc, char** argv) {
  const int m0 = argc > 1 ? atoi(argv[1]) : 0;
  const int var = argc > 2 ? atoi(argv[2]) : 0;
  cudaMemcpyToSymbol(g_variant, &var, 4);
  const int nx = 37, ny = 29, nz = 11, nxp = 40;
  const int bx = argc > 3 ? atoi(argv[3]) : 20, by = argc > 4 ? atoi(argv[4]) : 13, bz = 5;
  const int x0 = argc > 5 ? atoi(argv[5]) : -3, y0 = argc > 6 ? atoi(argv[6]) : 20, z0 = argc > 7 ? atoi(argv[7]) : 8;
  const int promo = argc > 8 ? atoi(argv[8]) : 1;
  std::vector<float> h((size_t)nxp * ny * nz);
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nxp; ++x) h[((size_t)z * ny + y) * nxp + x] = x < nx ? 1 + x + 100 * y + 10000 * z : -1;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&o, bx * by * bz * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  const cuuint64_t dim[3] = {nx, ny, nz}, str[2] = {nxp * 4, (cuuint64_t)nxp * ny * 4};
  const cuuint32_t box[3] = {bx, by, 1}, es[3] = {1, 1, 1};
  CUresult r = ((EncodeTiledFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_NONE, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  void* dtm;
  cudaMalloc(&dtm, 128);
  cudaMemcpy(dtm, &tm, 128, cudaMemcpyHostToDevice);
  for (int mode = m0; mode < 2; ++mode) {
    cudaMemset(o, 0, bx * by * bz * 4);
    const int smem = ((bx * by + 31) & ~31) * bz * 4 + 128;
    if (mode == 0) k_global<<<1, 128, smem>>>(dtm, x0, y0, z0, bx, by, bz, o);
    else k_param<<<1, 128, smem>>>(tm, x0, y0, z0, bx, by, bz, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> out(bx * by * bz);
    cudaMemcpy(out.data(), o, out.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int z = 0; z < bz; ++z)
      for (int y = 0; y < by; ++y)
        for (int x = 0; x < bx; ++x) {
          const int gx = x0 + x, gy = y0 + y, gz = z0 + z;
          const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz;
          const float want = in ? h[((size_t)gz * ny + gy) * nxp + gx] : 0.0f;
          if (out[(z * by + y) * bx + x] != want) ++bad;
        }
    printf("mode %d: %d mismatches of %d\n", mode, bad, bx * by * bz);
  }
  return 0;
}
