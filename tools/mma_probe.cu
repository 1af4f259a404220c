// Microbenchmark: cycles for a chain of 32 tcgen05.mma kind::tf32 (M=128, K=8)
// with A from TMEM (TS) or smem (SS), B in the no-swizzle "plane" layout or
// SW128, for several N.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1912_12055_b200/csrc/sm100.cuh"

using namespace nnab;

__global__ void probe(int variant, int N, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 13);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  uint32_t ph = 0;
  long long best = 1ll << 60;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    long long t0 = clock64();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t idesc = idesc_tf32(128, N);
      const uint32_t b0 = smem_u32(base + 64 * 1024);
      const uint32_t a0 = smem_u32(base);
      for (int k = 0; k < 32; ++k) {
        uint64_t bd;
        if (variant & 1) {  // B SW128 K-major
          bd = (uint64_t)(((b0 + (k & 3) * 32 + (k >> 2) * N * 128) >> 4) & 0x3FFF) | (1ull << 16) |
               ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
        } else {  // plane layout: LBO = 272, SBO = 128
          const uint32_t addr = b0 + ((8 * k & 127) >> 2) * 272 + ((8 * k) >> 7) * 16;
          bd = (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(272 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) |
               (1ull << 46);
        }
        if (variant & 2) {  // A from smem SW128 (16 KB tile reused)
          const uint64_t ad = (uint64_t)(((a0 + (k & 3) * 32) >> 4) & 0x3FFF) | (1ull << 16) |
                              ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
          mma_tf32(t + 256, ad, bd, idesc, k > 0);
        } else {
          mma_tf32_ts(t + 256, t + 8 * k, bd, idesc, k > 0);
        }
      }
      mma_commit(&bar);
    }
    mbar_wait(&bar, ph);
    ph ^= 1;
    long long dt = clock64() - t0;
    if (dt < best) best = dt;
  }
  if (tid == 0) out[blockIdx.x] = best;
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<512>(t);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[4] = {"TS A, plane B", "TS A, SW128 B", "SS A, plane B", "SS A, SW128 B"};
  for (int v = 0; v < 4; ++v)
    for (int N : {16, 32, 64, 128, 256}) {
      probe<<<1, 128, 100 * 1024>>>(v, N, 20, d);
      long long h = 0;
      cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%-16s N=%3d : %6lld cycles for 32 MMAs (%5.1f / MMA, floor %d)  %s\n", names[v], N, h, h / 32.0,
             128 * N / 256, cudaGetErrorString(e));
    }
  return 0;
}
