// The reference's signal primitives as standalone device ops (signal.py), for
// the `spectro` shim's pad_signal / downsample2: the transforms fuse both into
// their own kernels (stage_rows_kernel, cqt2010_tc_kernel); these serve callers
// of the primitives themselves and their known-answer tests.
#include <algorithm>

#include "internal.h"

namespace nnab {
namespace {

// np.pad(x, (left, right), "reflect" | "constant") (signal.py:138-156): bit-exact copy
__global__ void pad_kernel(const float* __restrict__ x, int64_t B, int64_t L, int64_t left, int64_t right, int mode,
                           float* __restrict__ y) {
  const int64_t n = L + left + right, total = B * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / n, i = e - b * n;
    int64_t j = i - left;
    float v = 0.f;
    if (mode == NNAB_PAD_REFLECT) {
      if (j < 0) j = -j;
      if (j >= L) j = 2 * (L - 1) - j;
      v = x[b * L + j];
    } else if (j >= 0 && j < L) {
      v = x[b * L + j];
    }
    y[e] = v;
  }
}

constexpr int kDsOut = 1024;  // outputs per CTA

// downsample2 (signal.py:232-247): y[i] = sum_m taps[m] * xpad[2i + n - 1 - m]
// (np.convolve flips the taps), xpad = reflect-pad(x, (n-1)/2).  The CTA's input
// span and the taps sit in shared memory; FP32 accumulation in tap order.
__global__ void __launch_bounds__(256) downsample2_kernel(const float* __restrict__ x, int64_t L,
                                                          const float* __restrict__ taps, int n_taps,
                                                          float* __restrict__ y, int64_t Lout) {
  extern __shared__ float sm[];
  float* tp = sm;               // [n_taps], flipped: tp[k] = taps[n - 1 - k]
  float* span = sm + n_taps;    // input span
  const int64_t b = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * kDsOut;
  const int n_out = (int)std::min<int64_t>(kDsOut, Lout - i0);
  if (n_out <= 0) return;
  const int half = (n_taps - 1) / 2;
  const int64_t p0 = 2 * i0 - half;  // unpadded coordinate of span[0]
  const int n_in = 2 * (n_out - 1) + n_taps;
  const float* xb = x + b * L;
  for (int k = threadIdx.x; k < n_taps; k += blockDim.x) tp[k] = taps[n_taps - 1 - k];
  for (int u = threadIdx.x; u < n_in; u += blockDim.x) {
    int64_t j = p0 + u;
    if (j < 0) j = -j;
    if (j >= L) j = 2 * (L - 1) - j;
    span[u] = __ldg(xb + j);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < n_out; o += blockDim.x) {
    const float* s = span + 2 * o;
    float acc = 0.f;
    for (int k = 0; k < n_taps; ++k) acc = fmaf(tp[k], s[k], acc);
    y[b * Lout + i0 + o] = acc;
  }
}

}  // namespace
}  // namespace nnab

using namespace nnab;

// x (B, L) -> y (B, L + left + right); mode NNAB_PAD_REFLECT or NNAB_PAD_ZERO.
// EINVAL mirrors pad_signal's ValueErrors: negative pads, reflect pad >= L.
extern "C" int nnab_pad_signal(const float* x, int64_t B, int64_t L, int64_t left, int64_t right, int32_t mode,
                               float* y, void* stream) {
  if (!x || !y || B < 0 || L < 1 || left < 0 || right < 0) return NNAB_EINVAL;
  if (mode != NNAB_PAD_REFLECT && mode != NNAB_PAD_ZERO) return NNAB_EINVAL;
  if (mode == NNAB_PAD_REFLECT && (left >= L || right >= L)) return NNAB_EINVAL;
  const int64_t total = B * (L + left + right);
  if (total == 0) return NNAB_OK;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
  pad_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, B, L, left, right, mode, y);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

// x (B, L) -> y (B, ceil(L / 2)) with the odd-length FIR taps (device, n_taps
// floats).  EINVAL mirrors downsample2's ValueErrors: even length, L < n_taps.
extern "C" int nnab_downsample2(const float* x, int64_t B, int64_t L, const float* taps, int32_t n_taps, float* y,
                                void* stream) {
  if (!x || !y || !taps || B < 0 || n_taps < 1 || n_taps % 2 == 0 || L < n_taps) return NNAB_EINVAL;
  if (n_taps > 4095) return NNAB_ENOTSUP;
  const int64_t Lout = (L + 1) / 2;
  if (B == 0) return NNAB_OK;
  const dim3 grid((unsigned)((Lout + kDsOut - 1) / kDsOut), (unsigned)B);
  const size_t smem = (size_t)(n_taps + 2 * (kDsOut - 1) + n_taps) * sizeof(float);
  NNAB_CUDA_TRY(cudaFuncSetAttribute(downsample2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  downsample2_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(x, L, taps, n_taps, y, Lout);
  NNAB_LAUNCHED();
  return NNAB_OK;
}
