// Probe: TMA tile load with elementStrides = 2 along the inner dimension.
// Checks which global elements land where in shared memory (no swizzle and
// 128-byte swizzle), for odd and even start coordinates.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stride_probe tma_stride_probe.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>

#include "../paper_1912_12055_b200/csrc/sm100.cuh"

using namespace nnab;

__global__ void k(const __grid_constant__ CUtensorMap tm, int c0, int c1, int bytes, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_expect_tx(&bar, bytes);
    tma_load_2d(sm, &tm, &bar, c0, c1);
  }
  __syncthreads();
  const long long t0 = clock64();
  while (!mbar_try_wait(&bar, 0)) {
    if (clock64() - t0 > 200000000ll) {  // ~0.1 s: report a timeout instead of hanging
      if (threadIdx.x == 0) out[0] = -1.f;
      return;
    }
  }
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main() {
  const int W = 256, R = 16;
  std::vector<float> h(W * R);
  for (int i = 0; i < W * R; ++i) h[i] = (float)i;  // value = linear index
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 65536);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  for (int sw : {0, 128})
    for (int c0 : {0, 2, 1}) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)R};
      cuuint64_t strides[1] = {(cuuint64_t)W * 4};
      cuuint32_t box[2] = {64, 8};
      cuuint32_t estr[2] = {2, 1};
      CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d (sw %d)\n", (int)r, sw);
        continue;
      }
      const int bytes = 32 * 8 * 4;
      for (int tx : {bytes, bytes / 2, 2 * bytes}) {
        cudaMemset(o, 0, 65536);
        k<<<1, 128, 4096>>>(tm, c0, 2, tx, o);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("sw %d c0 %d tx %d: %s\n", sw, c0, tx, cudaGetErrorString(e));
          return 1;
        }
        std::vector<float> g(tx / 4);
        cudaMemcpy(g.data(), o, tx, cudaMemcpyDeviceToHost);
        printf("sw %3d c0 %3d expect_tx %4d:", sw, c0, tx);
        if (g[0] != -1.f)
          for (int i = 0; i < tx / 4; ++i) printf("%s%g", i % 32 ? " " : "\n   ", g[i]);
        printf("\n");
        if (g[0] != -1.f) break;
      }
    }
  return 0;
}
