// Microbenchmark: cycles per tcgen05.mma for kind::f16 (K=16) vs kind::tf32
// (K=8), M = 64 / 128, several N, A and B from smem (no-swizzle K-major core
// matrices, the layouts the CQT2010v2 chain uses), with 1 or 4 independent
// accumulators, and with 1 or 2 CTAs per SM issuing at once.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe2 mma_probe2.cu
#include <cstdint>
#include <cstdio>

#include "../paper_1912_12055_b200/csrc/sm100.cuh"

using namespace nnab;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int NACC>
__global__ void probe(int f16, int M, int N, int iters, long long* out) {
  constexpr int nacc = NACC;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 80 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.f;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc<256>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  uint32_t ph = 0;
  long long best = 1ll << 60;
  const int n_mma = 64;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    long long t0 = clock64();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t idesc = f16 ? idesc_f16(M, N) : idesc_tf32(M, N);
      const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 32 * 1024);
#pragma unroll 16
      for (int k = 0; k < n_mma; ++k) {
        // no-swizzle K-major: core matrix 8 rows x 16 B; LBO = 128 B (next K core), SBO = 256 B (next 8 rows)
        const uint64_t ad = sdesc_kmajor_noswz(a0 + (k & 7) * 16, 128 * 2, 256 * 2);
        const uint64_t bd = sdesc_kmajor_noswz(b0 + (k & 7) * 16, 128 * 2, 256 * 2);
        const uint32_t dd = t + (uint32_t)(k % nacc) * (uint32_t)(N > 64 ? 0 : 64);
        if (f16) mma_f16(dd, ad, bd, idesc, k >= nacc);
        else mma_tf32(dd, ad, bd, idesc, k >= nacc);
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
  if (tid < 32) tmem_dealloc<256>(t);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 512);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int f16 = 0; f16 < 2; ++f16)
    for (int M : {128})
      for (int N : {32, 64, 128, 256})
        for (int ctas : {1, 2}) for (int nacc : {1, 2, 4}) {
          // 2 CTAs on one SM: grid = 2 * 148 with 100 KB smem each forces co-residency
          const int grid = ctas == 1 ? 148 : 296;
          if (nacc == 1) probe<1><<<grid, 128, 100 * 1024>>>(f16, M, N, 20, d);
          if (nacc == 2) probe<2><<<grid, 128, 100 * 1024>>>(f16, M, N, 20, d);
          if (nacc == 4) probe<4><<<grid, 128, 100 * 1024>>>(f16, M, N, 20, d);
          long long h[296] = {};
          cudaError_t e = cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
          long long mx = 0;
          for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
          const double macs = (double)M * N * (f16 ? 16 : 8);
          printf("acc=%d %s M=%3d N=%3d ctas/SM=%d : %7.1f cycles/MMA  %6.0f MAC/clk/CTA  %s\n", nacc, f16 ? "f16 " : "tf32", M, N,
                 ctas, h[0] / 64.0, macs * 64 / h[0], cudaGetErrorString(e));
        }
  return 0;
}
