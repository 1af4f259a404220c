// CQT2010v2: octave recursion with time-domain kernels (transforms.py:241-323).
//
//   early_stages x downsample2                      (transforms.py:295-296)
//   for alpha in 0..n_octaves-1:
//       downsample2 if alpha > 0                    (transforms.py:300-301)
//       centred complex conv, top-octave bank, hop kernel_hop >> alpha
//   trim to the shortest octave, scatter rows to first_bin + skip + j - alpha*b
//
// downsample2 (signal.py:232-247) = reflect pad (taps-1)/2, full-rate FIR,
// keep every second sample.  Only the kept samples are computed, and the
// 255-tap cutoff-0.5 windowed sinc is applied in symmetric-pair form over its
// non-zero taps (a half-band filter: 64 pairs + centre; the even-offset taps are
// <= 6.6e-17 and dropped by the host when it builds the pair list).
//
// Stage kernel: one CTA per (clip, 2048-output segment); the input span with
// its reflected halo is staged once in shared memory, then each thread
// produces consecutive outputs from registers.  The per-octave conv writes its
// 12 complex rows straight into the final (B, n_bins, T) output.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {

namespace {

constexpr int kSegOut = 2048;  // outputs per CTA
constexpr int kMaxPairs = 256;

struct FirPairs {
  float centre;
  int32_t n_pairs;
  int32_t half;               // (taps-1)/2: reflect pad of downsample2
  int32_t d[kMaxPairs];       // offsets from the centre (> 0)
  float h[kMaxPairs];         // tap value at +-d
};

__device__ __forceinline__ int64_t reflect_idx(int64_t j, int64_t n) {
  if (j < 0) j = -j;
  if (j >= n) j = 2 * (n - 1) - j;
  return j;
}

// y[i] = sum_m taps[m] * xpad[2i + m],  xpad = reflect-pad(x, half)
__global__ void __launch_bounds__(256) halve_kernel(const float* __restrict__ x, int64_t L, float* __restrict__ y,
                                                    int64_t Lout, const __grid_constant__ FirPairs fir) {
  extern __shared__ float span[];
  const int64_t b = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * kSegOut;
  const int64_t rem = Lout - i0;
  const int n_out = rem < kSegOut ? (int)rem : kSegOut;
  if (n_out <= 0) return;
  const int half = fir.half;
  // input positions (unpadded coordinates) 2*i0 - half .. 2*(i0+n_out-1) + half
  const int64_t p0 = 2 * i0 - half;
  const int n_in = 2 * (n_out - 1) + 2 * half + 1;
  const float* xb = x + b * L;
  for (int u = threadIdx.x; u < n_in; u += blockDim.x) span[u] = __ldg(xb + reflect_idx(p0 + u, L));
  __syncthreads();
  const int np = fir.n_pairs;
  for (int o = threadIdx.x; o < n_out; o += blockDim.x) {
    const int c = 2 * o + half;  // centre in span
    float acc = fir.centre * span[c];
    for (int k = 0; k < np; ++k) acc = fmaf(fir.h[k], span[c - fir.d[k]] + span[c + fir.d[k]], acc);
    y[b * Lout + i0 + o] = acc;
  }
}

// downsample2 for a half-band filter (pairs at every odd offset 1, 3, ..,
// 2P-1, as the reference's 255-tap design): y[i] = c x[2i] + sum_k g_k
// (x[2i - 2k - 1] + x[2i + 2k + 1]) only touches the even sample of the centre
// and odd samples otherwise, so the CTA stages the odd phase xo and the even
// phase xe of its span contiguously (reflect-padded) and each thread keeps 4
// consecutive outputs: per 4 taps one aligned 16-byte load per side feeds 16
// FMAs, conflict-free (lanes 16 bytes apart).  Same FMA order as halve_kernel.
constexpr int kHbOut = 1024;  // outputs per CTA (256 threads x 4)

__global__ void __launch_bounds__(256) halfband_kernel(const float* __restrict__ x, int64_t L, float* __restrict__ y,
                                                       int64_t Lout, const __grid_constant__ FirPairs fir) {
  extern __shared__ __align__(16) float hb[];
  const int P = fir.n_pairs;
  float* xo = hb;                // [kHbOut + 2P]: xo[u] = x[2 (i0 + u) - 2P + 1]
  float* xe = hb + kHbOut + 2 * P + 4;  // [kHbOut]:   xe[u] = x[2 (i0 + u)]
  const int64_t b = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * kHbOut;
  const int n_out = (int)min((int64_t)kHbOut, Lout - i0);
  if (n_out <= 0) return;
  const float* xb = x + b * L;
  for (int u = threadIdx.x; u < n_out + 2 * P; u += blockDim.x) xo[u] = __ldg(xb + reflect_idx(2 * (i0 + u) - 2 * P + 1, L));
  for (int u = threadIdx.x; u < n_out; u += blockDim.x) xe[u] = __ldg(xb + reflect_idx(2 * (i0 + u), L));
  __syncthreads();
  const int ii = 4 * threadIdx.x;
  if (ii >= n_out) return;
  float acc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = fir.centre * xe[ii + j];
  // right taps: xo[ii + P + k + j]; left taps: xo[ii + P - 1 - k + j]  (P % 4 == 0)
  const float4* r4 = reinterpret_cast<const float4*>(xo + ii + P);
  const float4* l4 = reinterpret_cast<const float4*>(xo + ii + P - 4);
  float4 ra = r4[0], lhi = l4[1];
#pragma unroll 1
  for (int k0 = 0; k0 < P; k0 += 4) {
    const float4 rb = r4[k0 / 4 + 1], llo = l4[-(k0 / 4)];
    const float r[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};          // xo[ii + P + k0 + 0..7]
    const float l[8] = {llo.x, llo.y, llo.z, llo.w, lhi.x, lhi.y, lhi.z, lhi.w};  // xo[ii + P - 4 - k0 + 0..7]
#pragma unroll
    for (int dk = 0; dk < 4; ++dk) {
      const float g = fir.h[k0 + dk];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fmaf(g, l[3 - dk + j] + r[dk + j], acc[j]);
    }
    ra = rb;
    lhi = llo;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (ii + j < n_out) y[b * Lout + i0 + ii + j] = acc[j];
}

// One octave: frames t < T_out of the centred complex conv at `hop`, written
// to rows row0 + j (j >= skip) of out (B, n_bins, T_out).
__global__ void octave_conv_kernel(const float* __restrict__ x, int64_t L, const float* __restrict__ k_re,
                                   const float* __restrict__ k_im, int32_t n_filt, int32_t width, int32_t hop,
                                   int32_t pad_mode, int32_t skip, int32_t row0, int32_t n_bins, int32_t T_out,
                                   int32_t out_kind, float* __restrict__ out, int64_t B) {
  const int64_t total = B * (int64_t)(n_filt - skip) * T_out;
  const int pad = width / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e % T_out);
    const int64_t r = e / T_out;
    const int j = skip + (int)(r % (n_filt - skip));
    const int64_t b = r / (n_filt - skip);
    const float* xb = x + b * L;
    const float* kr = k_re + (int64_t)j * width;
    const float* ki = k_im + (int64_t)j * width;
    float re = 0.f, im = 0.f;
    const int64_t s0 = (int64_t)t * hop - pad;
    for (int m = 0; m < width; ++m) {
      int64_t q = s0 + m;
      float v;
      if (pad_mode == NNAB_PAD_REFLECT) {
        v = __ldg(xb + reflect_idx(q, L));
      } else {
        v = (q >= 0 && q < L) ? __ldg(xb + q) : 0.f;
      }
      re = fmaf(v, __ldg(kr + m), re);
      im = fmaf(v, __ldg(ki + m), im);
    }
    const int row = row0 + j;
    float* o = out + ((b * n_bins + row) * (int64_t)T_out + t) * (out_kind == NNAB_OUT_COMPLEX ? 2 : 1);
    if (out_kind == NNAB_OUT_COMPLEX) {
      o[0] = re;
      o[1] = im;
    } else if (out_kind == NNAB_OUT_POWER) {
      o[0] = fmaf(re, re, im * im);
    } else {
      o[0] = sqrtf(fmaf(re, re, im * im));
    }
  }
}

// The same octave conv, one CTA per (128 frames, clip): the frames' signal span
// (reflect / zero padded) and the bank sit in shared memory, thread = frame with
// all 2 x n_filt accumulators in registers.  The span is stored skewed -- one pad
// word per hop-length row -- so the lanes (frames hop samples apart) hit
// distinct banks for every hop.  Same per-output FMA order as octave_conv_kernel.
constexpr int kConvFrames = 128;

template <int kMaxFilt>  // filters per octave, rounded up to 4 (12 for 12 bins per octave)
__global__ void __launch_bounds__(kConvFrames) octave_conv_smem_kernel(
    const float* __restrict__ x, int64_t L, const float* __restrict__ k_re, const float* __restrict__ k_im,
    int32_t n_filt, int32_t width, int32_t hop, int32_t pad_mode, int32_t skip, int32_t row0, int32_t n_bins,
    int32_t T_out, int32_t out_kind, float* __restrict__ out) {
  extern __shared__ float sm[];
  float* kr = sm;                          // [width][kMaxFilt]: tap-major, one row per tap
  float* ki = kr + width * kMaxFilt;
  float* sx = ki + width * kMaxFilt;       // skewed span
  const int64_t b = blockIdx.y;
  const int t0 = blockIdx.x * kConvFrames;
  const int nf = min(kConvFrames, T_out - t0);
  const int pad = width / 2;
  const int span = (nf - 1) * hop + width;
  const float* xb = x + b * L;
  for (int e = threadIdx.x; e < width * kMaxFilt; e += blockDim.x) {
    const int m = e / kMaxFilt, j = e - m * kMaxFilt;
    kr[e] = j < n_filt ? __ldg(k_re + (int64_t)j * width + m) : 0.f;
    ki[e] = j < n_filt ? __ldg(k_im + (int64_t)j * width + m) : 0.f;
  }
  const int64_t q0 = (int64_t)t0 * hop - pad;
  for (int i = threadIdx.x; i < span; i += blockDim.x) {
    const int64_t q = q0 + i;
    float v;
    if (pad_mode == NNAB_PAD_REFLECT) {
      v = __ldg(xb + reflect_idx(q, L));
    } else {
      v = (q >= 0 && q < L) ? __ldg(xb + q) : 0.f;
    }
    sx[i + i / hop] = v;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= nf) return;
  float re[kMaxFilt], im[kMaxFilt];
#pragma unroll
  for (int j = 0; j < kMaxFilt; ++j) re[j] = im[j] = 0.f;
  for (int m = 0; m < width; ++m) {
    const int r = t + m / hop, c = m - (m / hop) * hop;
    const float v = sx[r * (hop + 1) + c];
    const float4* kr4 = reinterpret_cast<const float4*>(kr + m * kMaxFilt);
    const float4* ki4 = reinterpret_cast<const float4*>(ki + m * kMaxFilt);
#pragma unroll
    for (int j4 = 0; j4 < kMaxFilt / 4; ++j4) {
      const float4 a = kr4[j4], bq = ki4[j4];
      re[4 * j4] = fmaf(v, a.x, re[4 * j4]);
      re[4 * j4 + 1] = fmaf(v, a.y, re[4 * j4 + 1]);
      re[4 * j4 + 2] = fmaf(v, a.z, re[4 * j4 + 2]);
      re[4 * j4 + 3] = fmaf(v, a.w, re[4 * j4 + 3]);
      im[4 * j4] = fmaf(v, bq.x, im[4 * j4]);
      im[4 * j4 + 1] = fmaf(v, bq.y, im[4 * j4 + 1]);
      im[4 * j4 + 2] = fmaf(v, bq.z, im[4 * j4 + 2]);
      im[4 * j4 + 3] = fmaf(v, bq.w, im[4 * j4 + 3]);
    }
  }
  const int tt = t0 + t;
#pragma unroll
  for (int j = 0; j < kMaxFilt; ++j) {
    if (j < skip || j >= n_filt) continue;
    float* o = out + ((b * n_bins + row0 + j) * (int64_t)T_out + tt) * (out_kind == NNAB_OUT_COMPLEX ? 2 : 1);
    if (out_kind == NNAB_OUT_COMPLEX) {
      o[0] = re[j];
      o[1] = im[j];
    } else if (out_kind == NNAB_OUT_POWER) {
      o[0] = fmaf(re[j], re[j], im[j] * im[j]);
    } else {
      o[0] = sqrtf(fmaf(re[j], re[j], im[j] * im[j]));
    }
  }
}

}  // namespace

}  // namespace nnab

using namespace nnab;

static int64_t halved(int64_t n) { return (n + 1) / 2; }

extern "C" size_t nnab_cqt2010v2_workspace_bytes(int64_t B, int64_t L, int32_t early_stages) {
  int64_t n = L;
  for (int i = 0; i < early_stages; ++i) n = halved(n);
  const int64_t a = halved(L);  // largest intermediate
  return (size_t)(2 * B * std::max<int64_t>(a, n) + 64) * sizeof(float);
}

extern "C" int nnab_cqt2010v2_forward(const float* x, int64_t B, int64_t L, const float* taps, int32_t n_taps,
                                      const float* k_re, const float* k_im, int32_t n_filters, int32_t width,
                                      int32_t early_stages, int32_t n_octaves, int32_t kernel_hop, int32_t first_bin,
                                      int32_t bins_per_octave, int32_t n_bins, int32_t pad_mode, int32_t out_kind,
                                      int32_t precision, float* out, int32_t* n_frames_out, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  if (!x || !taps || !k_re || !k_im || !out || n_taps < 3 || n_taps % 2 == 0) return NNAB_EINVAL;
  if (n_octaves < 1 || kernel_hop < 1 || width < 1 || n_filters < 1 || early_stages < 0) return NNAB_EINVAL;
  if ((kernel_hop >> (n_octaves - 1)) < 1) return NNAB_EINVAL;  // transforms.py:253-257
  if (pad_mode != NNAB_PAD_REFLECT && pad_mode != NNAB_PAD_ZERO) return NNAB_EINVAL;
  if (out_kind != NNAB_OUT_MAGNITUDE && out_kind != NNAB_OUT_POWER && out_kind != NNAB_OUT_COMPLEX)
    return NNAB_EINVAL;
  // signal lengths through the recursion, and every check the reference makes
  int64_t n = L;
  for (int i = 0; i < early_stages; ++i) {
    if (n < n_taps) return NNAB_EINVAL;  // signal.py:242-243
    n = halved(n);
  }
  int32_t T = INT32_MAX;
  for (int a = 0; a < n_octaves; ++a) {
    if (a > 0) {
      if (n < n_taps) return NNAB_EINVAL;
      n = halved(n);
    }
    if (pad_mode == NNAB_PAD_REFLECT && width / 2 >= n) return NNAB_EINVAL;  // signal.py:147-150
    const int64_t padded = n + 2 * (width / 2);
    if (width > padded) return NNAB_EINVAL;
    T = (int32_t)std::min<int64_t>(T, (padded - width) / (kernel_hop >> a) + 1);
  }
  if (n_frames_out) *n_frames_out = T;
  if (B == 0) return NNAB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == NNAB_PREC_TF32) {  // tensor-core chain (FP16 operands) when the clip fits in shared memory
    // default (NNAB_CQT2010_LEVELS unset or 3): the warp-specialised front kernel runs stages
    // 1-2 of every clip (cqt2010_front.cu), one chain launch the octave halvings of clip
    // groups (cqt2010_chain.cu), one batched launch the 12-bin convs of all octaves and clips.
    // 2: the fused kernel runs stages 1-2 and the halvings per clip, then the batched convs.
    // 1: fused front for stages 1-2 only, level-synchronous HALVE launches, batched convs.
    // 0: the single fused kernel with its convs (also the path without a workspace).
    static const int levels = [] {
      const char* e = getenv("NNAB_CQT2010_LEVELS");
      return e && e[0] >= '0' && e[0] <= '3' ? e[0] - '0' : 3;
    }();
    int rc = NNAB_ENOTSUP;
    if (levels && workspace)
      rc = launch_cqt2010_levels(x, B, L, taps, n_taps, k_re, k_im, n_filters, width, early_stages, n_octaves,
                                 kernel_hop, first_bin, bins_per_octave, n_bins, pad_mode, out_kind, T, out, workspace,
                                 workspace_bytes, s, levels);
    if (rc == NNAB_ENOTSUP)
      rc = launch_cqt2010_tc(x, B, L, taps, n_taps, k_re, k_im, n_filters, width, early_stages, n_octaves,
                             kernel_hop, first_bin, bins_per_octave, n_bins, pad_mode, out_kind, T, out, s);
    if (rc != NNAB_ENOTSUP) return rc;
  }
  if (!workspace || workspace_bytes < nnab_cqt2010v2_workspace_bytes(B, L, early_stages)) return NNAB_EINVAL;

  // symmetric pair list of the non-negligible taps (taps are a HOST array)
  const float* h = taps;
  FirPairs fp{};
  fp.half = (n_taps - 1) / 2;
  fp.centre = h[fp.half];
  float hmax = 0.f;
  for (int i = 0; i < n_taps; ++i) hmax = std::max(hmax, std::fabs(h[i]));
  for (int d = 1; d <= fp.half; ++d)
    if (h[fp.half + d] != h[fp.half - d]) return NNAB_EINVAL;  // FirFilter symmetry, signal.py:86-87
  for (int d = 1; d <= fp.half; ++d) {
    const float v = h[fp.half + d];
    if (std::fabs(v) <= 1e-12f * hmax) continue;  // exact-zero / half-band even taps
    if (fp.n_pairs == kMaxPairs) return NNAB_ENOTSUP;
    fp.d[fp.n_pairs] = d;
    fp.h[fp.n_pairs] = v;
    ++fp.n_pairs;
  }

  float* buf[2] = {reinterpret_cast<float*>(workspace),
                   reinterpret_cast<float*>(workspace) + B * std::max<int64_t>(halved(L), 1) + 32};
  const float* cur = x;
  int64_t cur_len = L;
  int pp = 0;
  // half-band (pairs exactly at offsets 1, 3, .., 2P-1 with P % 4 == 0): the polyphase kernel
  bool halfband = fp.n_pairs > 0 && fp.n_pairs % 4 == 0;
  for (int k = 0; halfband && k < fp.n_pairs; ++k) halfband = fp.d[k] == 2 * k + 1;
  auto halve = [&]() -> int {
    const int64_t lo = halved(cur_len);
    if (halfband && cur_len > 2 * fp.n_pairs) {
      const dim3 grid((unsigned)((lo + kHbOut - 1) / kHbOut), (unsigned)B);
      const size_t smem = (size_t)(2 * kHbOut + 2 * fp.n_pairs + 4) * sizeof(float);
      halfband_kernel<<<grid, 256, smem, s>>>(cur, cur_len, buf[pp], lo, fp);
    } else {
      dim3 grid((unsigned)((lo + kSegOut - 1) / kSegOut), (unsigned)B);
      const size_t smem = (size_t)(2 * (kSegOut - 1) + 2 * fp.half + 1) * sizeof(float);
      halve_kernel<<<grid, 256, smem, s>>>(cur, cur_len, buf[pp], lo, fp);
    }
    NNAB_LAUNCHED();
    cur = buf[pp];
    cur_len = lo;
    pp ^= 1;
    return NNAB_OK;
  };
  int rc;
  for (int i = 0; i < early_stages; ++i)
    if ((rc = halve())) return rc;
  for (int a = 0; a < n_octaves; ++a) {
    if (a > 0 && (rc = halve())) return rc;
    const int skip = std::max(0, a * bins_per_octave - first_bin);
    if (skip >= n_filters) continue;
    const int row0 = first_bin - a * bins_per_octave;
    const int hop = kernel_hop >> a;
    const int mf = n_filters <= 12 ? 12 : 16;
    const size_t smem = (size_t)(2 * width * mf + ((kConvFrames - 1) * (int64_t)hop + width) * (hop + 1) / hop + 8) *
                        sizeof(float);
    if (n_filters <= 16 && smem <= 200 * 1024) {
      auto kern = mf == 12 ? octave_conv_smem_kernel<12> : octave_conv_smem_kernel<16>;
      NNAB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const dim3 grid((unsigned)((T + kConvFrames - 1) / kConvFrames), (unsigned)B);
      kern<<<grid, kConvFrames, smem, s>>>(cur, cur_len, k_re, k_im, n_filters, width, hop, pad_mode, skip, row0,
                                           n_bins, T, out_kind, out);
    } else {
      const int64_t total = B * (int64_t)(n_filters - skip) * T;
      const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 32);
      octave_conv_kernel<<<blocks, 256, 0, s>>>(cur, cur_len, k_re, k_im, n_filters, width, hop, pad_mode, skip,
                                               row0, n_bins, T, out_kind, out, B);
    }
    NNAB_LAUNCHED();
  }
  return NNAB_OK;
}
