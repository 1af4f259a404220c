// Trainable layers (gradients.py:28-149) on the device.
//
// Forward (training): the STFT GEMM epilogue additionally stores re, im and
// the smoothed magnitude S = sqrt(re^2 + im^2 + eps) per (bin, frame slot) in
// slot-major layout [bin][ld], the K-major operand layout the backward GEMMs
// read.  Backward:
//   conv layer  (gradients.py:125-129):  coef = g*re/S, g*im/S  ->  dK = coef @ frames
//   mel layer   (gradients.py:118-121):  dW = g @ S^T
//   joint mel+STFT (nnAudio trainable_mel + trainable_STFT): dS = W^T g, then as conv
//   input grad  (gradients.py:133-149):  frame grads = coef^T @ h, overlap-add, fold pad
// All products run on the tcgen05 reduction GEMM (rgemm.cu); the glue here is
// elementwise and HBM-bound.
#include <cuda_fp16.h>

#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

// out[r][b*R + t] = g[b][r][t] for t < T, 0 for the staging-only slots and the
// tail up to ld.  Block b < B: clip b, one warp per row at a time, lanes over its R
// slots (coalesced on both sides, no per-element index division); block B: the tail.
__global__ void to_slots_kernel(const float* __restrict__ g, int64_t B, int32_t rows, int32_t T, int32_t R,
                                int64_t ld, float* __restrict__ out, int round, float* __restrict__ lo) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int64_t b = blockIdx.x; b <= B; b += gridDim.x) {
    const int64_t s0 = b * R, n = b < B ? R : ld - B * R;
    for (int r = w; r < rows; r += nw) {
      const float* src = g + (b * rows + r) * (int64_t)T;
      float* dst = out + (int64_t)r * ld + s0;
      float* dlo = lo ? lo + (int64_t)r * ld + s0 : nullptr;
      for (int64_t t = lane; t < n; t += 32) {
        const float v = (b < B && t < T) ? src[t] : 0.f;
        if (round) {
          const float h = tf32_rne(v);
          dst[t] = h;
          if (dlo) dlo[t] = tf32_rne(v - h);
        } else {
          dst[t] = v;
        }
      }
    }
  }
}

// out[b][r][t] = src[r][b*R + t]   (slot-major GEMM output -> (B, rows, T))
__global__ void from_slots_kernel(const float* __restrict__ src, int64_t B, int32_t rows, int32_t T, int32_t R,
                                  int64_t ld, float* __restrict__ out) {
  const int64_t total = B * rows * (int64_t)T;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e % T);
    const int64_t br = e / T;
    const int r = (int)(br % rows);
    const int64_t b = br / rows;
    out[e] = src[(int64_t)r * ld + b * R + t];
  }
}

// coef rows [0, F): dS*re/S, rows [F, 2F): dS*im/S  (gradients.py:127-128)
__global__ void coef_kernel(const float* __restrict__ ds_slots, const float* __restrict__ g_bft,
                            const float* __restrict__ re, const float* __restrict__ im, int32_t F, int64_t B,
                            int32_t T, int32_t R, int64_t ld, float eps, int split, float* __restrict__ hi,
                            float* __restrict__ lo) {
  const int64_t total = (int64_t)F * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = e / ld, slot = e - f * ld;
    const int64_t b = slot / R;
    const int t = (int)(slot - b * R);
    float d = 0.f;
    if (b < B && t < T) d = ds_slots ? ds_slots[e] : g_bft[(b * F + f) * (int64_t)T + t];
    float cr, ci;
    if (im) {
      const float r = re[e], i = im[e];
      const float di = d * rsqrtf(fmaf(r, r, i * i) + eps);  // as rgemm.cu coef_store
      cr = di * r;
      ci = di * i;
    } else {  // re holds the unit phasor (re/S, im/S) as FP16 pairs (TF32 training forward)
      const float2 ph = __half22float2(reinterpret_cast<const __half2*>(re)[e]);
      cr = d * ph.x;
      ci = d * ph.y;
    }
    const float hr = tf32_rne(cr), hi_ = tf32_rne(ci);
    hi[e] = hr;
    hi[e + (int64_t)F * ld] = hi_;
    if (split) {
      lo[e] = tf32_rne(cr - hr);
      lo[e + (int64_t)F * ld] = tf32_rne(ci - hi_);
    }
  }
}

// dst[c][r] = src[r][c] (c < cols, r < rows), zero for r in [rows, ld); tf32 hi/lo
__global__ void transpose_kernel(const float* __restrict__ src, int32_t rows, int32_t cols, int32_t ld, int split,
                                 float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = (int64_t)cols * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / ld;
    const int r = (int)(e - c * ld);
    const float v = r < rows ? src[(int64_t)r * cols + c] : 0.f;
    const float h = tf32_rne(v);
    hi[e] = h;
    if (split) lo[e] = tf32_rne(v - h);
  }
}

// tf32 hi/lo split of a dense matrix, in place layout (rows x cols, ld)
__global__ void split_kernel(const float* __restrict__ src, int64_t n, int split, float* __restrict__ hi,
                             float* __restrict__ lo) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = src[e];
    const float h = tf32_rne(v);
    hi[e] = h;
    if (split) lo[e] = tf32_rne(v - h);
  }
}

// Input gradient: padded-domain overlap-add of frame grads fg[m][slot]
// (fg^T = h^T @ coef, gradients.py:135), then fold through the pad index map
// (gradients.py:140-148).  One thread per output sample gathers its frames:
// deterministic, no atomics.
__global__ void input_grad_kernel(const float* __restrict__ fg, int64_t ld_fg, int64_t B, int64_t L, int32_t width,
                                  int32_t hop, int32_t pad, int32_t mode, int32_t T, int32_t R,
                                  float* __restrict__ gx) {
  const int64_t total = B * L;
  const int64_t Lp = L + 2ll * pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / L, j = e - b * L;
    // padded positions mapping to sample j: j+pad, and for reflect the mirrors
    int64_t pos[3];
    int np = 0;
    pos[np++] = j + pad;
    if (mode == NNAB_PAD_REFLECT && pad > 0) {
      if (j >= 1 && j <= pad) pos[np++] = pad - j;                      // left mirror
      if (j >= L - 1 - pad && j <= L - 2) pos[np++] = pad + 2 * (L - 1) - j;  // right mirror
    }
    float acc = 0.f;
    for (int u = 0; u < np; ++u) {
      const int64_t p = pos[u];
      if (p < 0 || p >= Lp) continue;
      // frames t with t*hop <= p < t*hop + width
      int64_t t_hi = p / hop;
      int64_t t_lo = (p - width) / hop + 1;
      if (p - width < 0) t_lo = 0;
      if (t_hi > T - 1) t_hi = T - 1;
      for (int64_t t = t_lo; t <= t_hi; ++t) {
        const int64_t m = p - t * hop;
        acc += fg[m * ld_fg + b * R + t];  // frame grads stored transposed: [tap][slot]
      }
    }
    gx[e] = acc;
  }
}

int grid_for(int64_t total) { return (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 32); }

// ---- 3xF16 kernel gradient operands -------------------------------------------------
// The staged frames of clip b are x * 2^e_b (FP16 hi/lo, stage_rows_f16*).  The coef row
// m enters the dK GEMM as FP16 hi/lo of coef * 2^(r_m - e_b): 2^-e_b makes the product
// with the staged frames exact, 2^r_m keeps the row's largest magnitude below 2^14
// (FP16 holds 2^16; no overflow is possible) and the epilogue multiplies by 2^-r_m.
// r_m comes from a bound, not a max pass over coef: |coef| <= |dS| (|re|, |im| <= S)
// and |dS[f]| <= sum_m |W[m][f]| * G with G = max |g * 2^-e_b|.  A loose bound only
// moves small values toward FP16's subnormal range, whose spacing (2^-24 against the
// row's 2^14 ceiling) is far below the 2^-22 split error.

// gmax = max over clips b of 2^-e_b * max |v| over clip b's elements (+ |lo|), as float
// bits (non-negative floats order as unsigned): element (r, t) of clip b at
// v[b * clip_stride + r * row_stride + t], r < rows, t < T.  One block per clip, one
// warp per row at a time (no per-element index division).
__global__ void clip_absmax_kernel(const float* __restrict__ v, const float* __restrict__ lo, int64_t B, int32_t rows,
                                   int64_t row_stride, int64_t clip_stride, int32_t T,
                                   const int32_t* __restrict__ exps, unsigned* __restrict__ gmax) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const float* vb = v + b * clip_stride;
    const float* lb = lo ? lo + b * clip_stride : nullptr;
    float mx = 0.f;
    for (int r = w; r < rows; r += nw) {
      for (int t = lane; t < T; t += 32) {
        const int64_t o = r * row_stride + t;
        mx = fmaxf(mx, fabsf(vb[o]) + (lb ? fabsf(lb[o]) : 0.f));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mx *= __int_as_float((127 - exps[b]) << 23);
    if (lane == 0 && mx > 0.f) atomicMax(gmax, __float_as_uint(mx));
  }
}

// row_exp[f] = row_exp[F + f] = 14 - ceil(log2(bound_f)), bound_f = colsum_f * G with
// colsum_f = sum_m |wt[f][m]| (wt null: 1); 0 where the bound is 0 or not finite
__global__ void row_exp_kernel(const float* __restrict__ wt_hi, const float* __restrict__ wt_lo, int32_t F,
                               int32_t kp, int32_t n_mels, const unsigned* __restrict__ gmax,
                               int32_t* __restrict__ row_exp) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  float c = 1.f;
  if (wt_hi) {
    c = 0.f;
    for (int m = 0; m < n_mels; ++m) c += fabsf(wt_hi[(int64_t)f * kp + m]) + (wt_lo ? fabsf(wt_lo[(int64_t)f * kp + m]) : 0.f);
  }
  const float b = c * __uint_as_float(*gmax) * 1.001f;  // margin for the rounding of the sums
  int e = 0;
  if (b > 0.f && b < INFINITY) {
    int ex;
    frexpf(b, &ex);  // b < 2^ex
    e = max(-125, min(125, 14 - ex));
  }
  row_exp[f] = e;
  row_exp[F + f] = e;
}

// coef_kernel's conv-layer form (g straight from (B, F, T)) writing the 3xF16 dK operand
__global__ void coef_f16_kernel(const float* __restrict__ g_bft, const float* __restrict__ re,
                                const float* __restrict__ im, int32_t F, int64_t B, int32_t T, int32_t R, int64_t ld,
                                float eps, const int32_t* __restrict__ exps, const int32_t* __restrict__ row_exp,
                                __half* __restrict__ hi, __half* __restrict__ lo) {
  const int64_t total = (int64_t)F * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = e / ld, slot = e - f * ld;
    const int64_t b = slot / R;
    const int t = (int)(slot - b * R);
    float cr = 0.f, ci = 0.f;
    if (b < B && t < T) {
      const float d = g_bft[(b * F + f) * (int64_t)T + t];
      const float sc = __int_as_float((127 - exps[b]) << 23) * __int_as_float((127 + row_exp[f]) << 23);
      if (im) {
        const float r = re[e], i = im[e];
        const float di = d * rsqrtf(fmaf(r, r, i * i) + eps);
        cr = di * r * sc;
        ci = di * i * sc;
      } else {  // the FP16 unit phasor (re/S, im/S) of a TF32-backward forward
        const float2 ph = __half22float2(reinterpret_cast<const __half2*>(re)[e]);
        cr = d * ph.x * sc;
        ci = d * ph.y * sc;
      }
    }
    const __half hr = __float2half_rn(cr), hi_ = __float2half_rn(ci);
    hi[e] = hr;
    hi[e + (int64_t)F * ld] = hi_;
    if (lo) {
      lo[e] = __float2half_rn(cr - __half2float(hr));
      lo[e + (int64_t)F * ld] = __float2half_rn(ci - __half2float(hi_));
    }
  }
}

}  // namespace
}  // namespace nnab

using namespace nnab;

extern "C" int64_t nnab_slots_ld(const nnab_frames* f) {
  FrameGeom g;
  if (frame_geometry(f, &g)) return -1;
  return (g.B * g.R + 31) / 32 * 32;
}

extern "C" int nnab_stft_forward_train_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo,
                                              int32_t n_bins, int32_t fold_nyquist, int32_t precision,
                                              int32_t out_kind, float power, float eps, const float* mel_w,
                                              int32_t n_mels, int32_t mel_ld, const int32_t* mel_band, float* out,
                                              float* save_re, float* save_im, float* save_mag, int64_t ld,
                                              const void* workspace, size_t workspace_bytes, void* stream) {
  const int phasor = (out_kind & NNAB_SAVE_PHASOR) != 0;
  const int mag_split = (out_kind & NNAB_SAVE_MAG_SPLIT) != 0;
  out_kind &= ~(NNAB_SAVE_PHASOR | NNAB_SAVE_MAG_SPLIT);
  if (!prec_valid(precision)) return NNAB_EINVAL;
  const int split = prec_is_split(precision);
  // saves: TF32 / F16 forward -> FP16 phasor (+ TF32 |X|); split modes -> fp32 re, im
  // (the 3xTF32 backward's operands) unless NNAB_SAVE_PHASOR asks for the TF32-backward format
  const bool want_im = split && !phasor;
  if (!packed_hi || (split && !packed_lo) || !save_re || (want_im && !save_im)) return NNAB_EINVAL;
  if (out_kind != NNAB_OUT_SMOOTH_MAG && out_kind != NNAB_OUT_MEL) return NNAB_EINVAL;
  if (!out && out_kind != NNAB_OUT_SMOOTH_MAG) return NNAB_EINVAL;  // out may be null: save slots only
  if (out_kind == NNAB_OUT_MEL && (!mel_w || n_mels < 1)) return NNAB_EINVAL;
  FrameGeom g;
  const void *hi, *lo;
  const int32_t* exps;
  int rc = staged_views(f, precision, workspace, workspace_bytes, &g, &hi, &lo, &exps);
  if (rc) return rc;
  if (ld < g.B * g.R || ld % 32) return NNAB_EINVAL;
  FrameGeom gb;  // the slot layout is the TF32 backward's: the forward must stage the same rows per clip
  if ((rc = frame_geometry(f, &gb)) || gb.R != g.R) return rc ? rc : NNAB_ENOTSUP;
  if (g.B == 0) return NNAB_OK;
  StftGemmArgs a{};
  a.a_hi = reinterpret_cast<const float*>(hi);
  a.a_lo = reinterpret_cast<const float*>(lo);
  a.a_exp = exps;
  if (exps)
    a.b_exp = reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(packed_hi) +
                                               nnab_dft_bank_bytes_prec(n_bins, g.width, fold_nyquist, precision) -
                                               256) + 1;
  a.b_hi = packed_hi;
  a.b_lo = packed_lo;
  a.n_tiles = nnab_dft_bank_tiles(n_bins, fold_nyquist);
  a.n_bins = n_bins;
  a.fold = fold_nyquist ? 1 : 0;
  a.out_kind = out_kind;
  a.power = power;
  a.eps = eps;
  a.mel_w = mel_w;
  a.n_mels = n_mels;
  a.mel_ld = mel_ld;
  a.mel_band = mel_band;
  a.out = out;
  a.save_re = save_re;
  a.save_im = want_im ? save_im : nullptr;
  a.save_mag = save_mag;
  if (mag_split) {  // [2][n_bins][ld]: the 3xTF32 pair of |X| (split modes' fp32 saves only)
    if (!split || phasor || !save_mag) return NNAB_EINVAL;
    a.save_mag_lo = save_mag + (int64_t)n_bins * ld;
  }
  a.ld_slots = ld;
  a.save_phasor = phasor;
  return launch_stft_gemm(g, a, precision, (cudaStream_t)stream);
}

// as nnab_grad_to_slots, fused with the GEMM-operand split: hi = TF32(v) and, in
// 3xTF32, lo = TF32(v - hi) -- the layout nnab_rgemm / nnab_mel_dft_coef read
extern "C" int nnab_grad_to_slots_split(const float* g_brt, int64_t B, int32_t rows, int32_t T, int32_t R, int64_t ld,
                                        int32_t precision, float* hi, float* lo, void* stream) {
  if (!g_brt || !hi || rows < 1 || T < 1 || R < T || ld < B * R) return NNAB_EINVAL;
  if (precision == NNAB_PREC_3XTF32 && !lo) return NNAB_EINVAL;
  const int64_t total = (int64_t)rows * ld;
  if (total == 0) return NNAB_OK;
  to_slots_kernel<<<(int)std::min<int64_t>(B + 1, 65535), 256, 0, (cudaStream_t)stream>>>(
      g_brt, B, rows, T, R, ld, hi, 1, precision == NNAB_PREC_3XTF32 ? lo : nullptr);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_grad_to_slots(const float* g_brt, int64_t B, int32_t rows, int32_t T, int32_t R, int64_t ld,
                                  float* out, void* stream) {
  if (!g_brt || !out || rows < 1 || T < 1 || R < T || ld < B * R) return NNAB_EINVAL;
  const int64_t total = (int64_t)rows * ld;
  if (total == 0) return NNAB_OK;
  to_slots_kernel<<<(int)std::min<int64_t>(B + 1, 65535), 256, 0, (cudaStream_t)stream>>>(g_brt, B, rows, T, R, ld,
                                                                                           out, 0, nullptr);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_from_slots(const float* src, int64_t B, int32_t rows, int32_t T, int32_t R, int64_t ld,
                               float* out_brt, void* stream) {
  if (!src || !out_brt || rows < 1 || T < 1 || R < T || ld < B * R) return NNAB_EINVAL;
  const int64_t total = B * rows * (int64_t)T;
  if (total == 0) return NNAB_OK;
  from_slots_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(src, B, rows, T, R, ld, out_brt);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_dft_coef(const float* ds_slots, const float* g_bft, const float* re_s, const float* im_s,
                             int32_t F, int64_t B, int32_t T, int32_t R, int64_t ld, float eps, int32_t precision,
                             float* coef_hi, float* coef_lo, void* stream) {
  if ((!ds_slots && !g_bft) || !re_s || !coef_hi || F < 1 || ld < B * R) return NNAB_EINVAL;
  const int split = precision == NNAB_PREC_3XTF32;
  if (!im_s && split) return NNAB_EINVAL;  // phasor input: TF32 only
  if (split && !coef_lo) return NNAB_EINVAL;
  const int64_t total = (int64_t)F * ld;
  coef_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(ds_slots, g_bft, re_s, im_s, F, B, T, R, ld, eps,
                                                                 split, coef_hi, coef_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_transpose_pad(const float* src, int32_t rows, int32_t cols, int32_t ld, int32_t precision,
                                  float* hi, float* lo, void* stream) {
  if (!src || !hi || rows < 1 || cols < 1 || ld < rows) return NNAB_EINVAL;
  const int split = precision == NNAB_PREC_3XTF32;
  if (split && !lo) return NNAB_EINVAL;
  const int64_t total = (int64_t)cols * ld;
  transpose_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(src, rows, cols, ld, split, hi, lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_tf32_split(const float* src, int64_t n, int32_t precision, float* hi, float* lo, void* stream) {
  if (!src || !hi || n < 0) return NNAB_EINVAL;
  const int split = precision == NNAB_PREC_3XTF32;
  if (split && !lo) return NNAB_EINVAL;
  if (n == 0) return NNAB_OK;
  split_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(src, n, split, hi, lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" size_t nnab_rgemm_partial_bytes(int32_t M, int32_t N, int64_t K, int32_t splits) {
  return rgemm_partial_bytes(M, N, K, splits);
}

extern "C" int nnab_rgemm(int32_t M, int32_t N, int64_t K, const float* a_hi, const float* a_lo, int64_t lda,
                          const float* b_hi, const float* b_lo, int64_t ldb, int32_t b_mn, int32_t b_row_len,
                          int64_t b_rows, float* c, int64_t ldc, int32_t splits, float* partial, int32_t precision,
                          void* stream) {
  if (M < 1 || N < 1 || K < 1 || !a_hi || !b_hi || !c) return NNAB_EINVAL;
  if (precision == NNAB_PREC_3XTF32 && (!a_lo || !b_lo)) return NNAB_EINVAL;
  RGemmArgs g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.a_hi = a_hi;
  g.a_lo = a_lo;
  g.lda = lda;
  g.b_hi = b_hi;
  g.b_lo = b_lo;
  g.ldb = ldb;
  g.b_mn = b_mn;
  g.b_row_len = b_row_len;
  g.b_rows = b_rows;
  g.c = c;
  g.ldc = ldc;
  g.splits = splits;
  g.partial = partial;
  return launch_rgemm(g, precision, (cudaStream_t)stream);
}

// Joint mel + trainable STFT backward, dS = W^T g fused with the coef step:
// coef rows [0, F) = dS*re/S, [F, 2F) = dS*im/S (gradients.py:125-128,
// nnAudio trainable_mel over trainable_STFT).  wt: W^T zero-padded to
// [F][kp] (kp = n_mels rounded up to 32); gs: the upstream grad in slot
// layout [n_mels][ld] (nnab_grad_to_slots); re/im: [F][ld] from the training
// forward.  dS never reaches HBM: the GEMM epilogue reads re/im and writes coef.
extern "C" int nnab_mel_dft_coef(int32_t F, int64_t ld, int32_t kp, const float* wt_hi, const float* wt_lo,
                                 const float* gs_hi, const float* gs_lo, int32_t n_mels, const float* re_s,
                                 const float* im_s, float eps, int32_t precision, float* coef_hi, float* coef_lo,
                                 void* stream) {
  if (F < 1 || ld < 1 || kp < n_mels || n_mels < 1 || !wt_hi || !gs_hi || !re_s || !coef_hi) return NNAB_EINVAL;
  if (precision == NNAB_PREC_3XTF32 && (!wt_lo || !gs_lo || !coef_lo || !im_s)) return NNAB_EINVAL;
  if (ld > INT32_MAX) return NNAB_EINVAL;
  if (kp > 1024) return NNAB_ENOTSUP;  // one TMEM accumulation chain per tile
  RGemmArgs g;
  g.M = F;
  g.N = (int32_t)ld;
  g.K = kp;
  g.a_hi = wt_hi;
  g.a_lo = wt_lo;
  g.lda = kp;
  g.b_hi = gs_hi;
  g.b_lo = gs_lo;
  g.b_mn = 1;
  g.b_row_len = (int32_t)ld;
  g.b_rows = n_mels;
  g.c = coef_hi;
  g.ldc = ld;
  g.splits = 1;
  g.coef_re = re_s;
  g.coef_im = im_s;
  g.coef_lo = coef_lo;
  g.coef_eps = eps;
  return launch_rgemm(g, precision, (cudaStream_t)stream);
}

// Mel layer forward of the trainable layer (gradients.py:69-80): mel = W @ S
// with S the slot-major smoothed magnitude [F][ld] of the training forward, on
// the tcgen05 reduction GEMM, written straight to (B, n_mels, T) from the
// epilogue (no slot-major intermediate).  w: W zero-padded to [n_mels][kp]
// (kp = F rounded up to 32), TF32 hi (+ lo).
extern "C" int nnab_mel_forward_slots(int32_t n_mels, int64_t ld, int32_t kp, const float* w_hi, const float* w_lo,
                                      const float* s_hi, const float* s_lo, int32_t F, int64_t B, int32_t R, int32_t T,
                                      int32_t precision, float* out, void* stream) {
  if (n_mels < 1 || ld < 1 || kp < F || F < 1 || !w_hi || !s_hi || !out || B < 0 || R < T || T < 1)
    return NNAB_EINVAL;
  if (precision == NNAB_PREC_3XTF32 && (!w_lo || !s_lo)) return NNAB_EINVAL;
  if (ld > INT32_MAX || ld < B * R || R % 4) return NNAB_EINVAL;
  if (kp > 2048) return NNAB_ENOTSUP;  // one TMEM chain per tile
  if (B == 0) return NNAB_OK;
  RGemmArgs g;
  g.M = n_mels;
  g.N = (int32_t)ld;
  g.K = kp;
  g.a_hi = w_hi;
  g.a_lo = w_lo;
  g.lda = kp;
  g.b_hi = s_hi;
  g.b_lo = s_lo;
  g.b_mn = 1;
  g.b_row_len = (int32_t)ld;
  g.b_rows = F;
  g.c = out;
  g.ldc = ld;
  g.splits = 1;
  g.frames_B = B;
  g.frames_R = R;
  g.frames_T = T;
  return launch_rgemm(g, precision, (cudaStream_t)stream);
}

// dK[r][m] = sum_slot coef[r][slot] * frames[slot][m]   (gradients.py:129)
extern "C" int nnab_kernel_grad(const nnab_frames* f, const float* coef_hi, const float* coef_lo, int32_t rows,
                                int64_t ld, int32_t precision, float* dk, int64_t ldk, const void* workspace,
                                size_t workspace_bytes, float* partial, int32_t splits, void* stream) {
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  const int split = precision == NNAB_PREC_3XTF32;
  if (!workspace || workspace_bytes < nnab_stft_workspace_bytes(f, precision)) return NNAB_EINVAL;
  const size_t sb = (size_t)((g.B * g.R * g.row_len * 4 + 255) & ~int64_t(255));
  const float* fr_hi = reinterpret_cast<const float*>(workspace);
  const float* fr_lo = split ? reinterpret_cast<const float*>(reinterpret_cast<const char*>(workspace) + sb) : nullptr;
  return nnab_rgemm(rows, g.width, ld, coef_hi, coef_lo, ld, fr_hi, fr_lo, 0, 1, g.row_len, g.B * g.R, dk, ldk, splits,
                    partial, precision, stream);
}

extern "C" int nnab_input_grad(const nnab_frames* f, const float* frame_grads, int64_t ld_fg, float* gx,
                               void* stream) {
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  if (!frame_grads || !gx || ld_fg < g.B * g.R) return NNAB_EINVAL;
  const int64_t total = g.B * g.L;
  if (total == 0) return NNAB_OK;
  input_grad_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(frame_grads, ld_fg, g.B, g.L, g.width, g.hop,
                                                                       g.pad, g.pad_mode, g.T, g.R, gx);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

// ---- 3xF16 kernel gradient (FP32 mode) ----------------------------

// staging: the precision ws16 was staged in -- NNAB_PREC_3XF16 (hi + lo rows) or NNAB_PREC_F16 (hi)
static int f16_views(const nnab_frames* f, const void* ws16, size_t ws16_bytes, int32_t staging, FrameGeom* g,
                     const void** hi, const void** lo, const int32_t** exps) {
  if (staging != NNAB_PREC_3XF16 && staging != NNAB_PREC_F16) return NNAB_EINVAL;
  int rc = staged_views(f, staging, ws16, ws16_bytes, g, hi, lo, exps);
  if (rc) return rc;
  if (g->B > 0 && (!*exps || (staging == NNAB_PREC_3XF16 && !*lo))) return NNAB_EINVAL;
  return NNAB_OK;
}

extern "C" int nnab_mel_dft_coef_f16(const nnab_frames* f, const void* ws16, size_t ws16_bytes, int32_t staging,
                                     int32_t F, int64_t ld,
                                     int32_t kp, const float* wt_hi, const float* wt_lo, const float* gs_hi,
                                     const float* gs_lo, int32_t n_mels, const float* re_s, const float* im_s,
                                     float eps, void* coef_hi, void* coef_lo, int32_t* row_exps, void* stream) {
  FrameGeom g;
  const void *hi, *lo;
  const int32_t* exps;
  int rc = f16_views(f, ws16, ws16_bytes, staging, &g, &hi, &lo, &exps);
  if (rc) return rc;
  // coef_lo given: 3xTF32 coef GEMM from re / im, FP16 hi + lo out (the 3xF16 dK); coef_lo null: TF32
  // coef GEMM from the FP16 unit phasor (im_s null), FP16 hi out (the one-pass FP16 dK)
  const bool split = coef_lo != nullptr;
  if (F < 1 || ld < g.B * g.R || ld % 8 || kp < n_mels || n_mels < 1 || !wt_hi || !gs_hi || !re_s || !coef_hi ||
      !row_exps || (split && (!wt_lo || !gs_lo || !im_s)) || (!split && im_s))
    return NNAB_EINVAL;
  if (ld > INT32_MAX) return NNAB_EINVAL;
  if (kp > 1024) return NNAB_ENOTSUP;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned* gmax = reinterpret_cast<unsigned*>(row_exps + 2 * F);
  NNAB_CUDA_TRY(cudaMemsetAsync(gmax, 0, 4, s));
  if (g.B > 0) {
    const int T = (int)std::min<int64_t>(g.R, g.T);
    clip_absmax_kernel<<<(int)std::min<int64_t>(g.B, 65535), 256, 0, s>>>(gs_hi, gs_lo, g.B, n_mels, ld, g.R, T,
                                                                          exps, gmax);
    NNAB_LAUNCHED();
  }
  row_exp_kernel<<<(F + 127) / 128, 128, 0, s>>>(wt_hi, wt_lo, F, kp, n_mels, gmax, row_exps);
  NNAB_LAUNCHED();
  RGemmArgs a;
  a.M = F;
  a.N = (int32_t)ld;
  a.K = kp;
  a.a_hi = wt_hi;
  a.a_lo = wt_lo;
  a.lda = kp;
  a.b_hi = gs_hi;
  a.b_lo = gs_lo;
  a.b_mn = 1;
  a.b_row_len = (int32_t)ld;
  a.b_rows = n_mels;
  a.c = reinterpret_cast<float*>(coef_hi);
  a.ldc = ld;
  a.splits = 1;
  a.coef_re = re_s;
  a.coef_im = im_s;
  a.coef_lo = reinterpret_cast<float*>(coef_lo);
  a.coef_eps = eps;
  a.coef_f16 = 1;
  a.row_exp = row_exps;
  a.clip_exp = exps;
  a.n_clips = g.B;
  a.clip_R = g.R;
  return launch_rgemm(a, split ? NNAB_PREC_3XTF32 : NNAB_PREC_TF32, s);
}

extern "C" int nnab_dft_coef_f16(const nnab_frames* f, const void* ws16, size_t ws16_bytes, int32_t staging,
                                 const float* g_bft,
                                 const float* re_s, const float* im_s, int32_t F, int32_t T, int64_t ld, float eps,
                                 void* coef_hi, void* coef_lo, int32_t* row_exps, void* stream) {
  FrameGeom g;
  const void *hi, *lo;
  const int32_t* exps;
  int rc = f16_views(f, ws16, ws16_bytes, staging, &g, &hi, &lo, &exps);
  if (rc) return rc;
  // coef_lo given: re / im in, FP16 hi + lo out; null: FP16 hi out, re_s may hold the FP16 unit phasor (im_s null)
  if (!g_bft || !re_s || (coef_lo && !im_s) || !coef_hi || !row_exps || F < 1 || T < 1 || T > g.R ||
      ld < g.B * g.R || ld % 8)
    return NNAB_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned* gmax = reinterpret_cast<unsigned*>(row_exps + 2 * F);
  NNAB_CUDA_TRY(cudaMemsetAsync(gmax, 0, 4, s));
  const int64_t n = g.B * (int64_t)F * T;
  if (n > 0) {
    clip_absmax_kernel<<<(int)std::min<int64_t>(g.B, 65535), 256, 0, s>>>(g_bft, nullptr, g.B, F, T,
                                                                          (int64_t)F * T, T, exps, gmax);
    NNAB_LAUNCHED();
  }
  row_exp_kernel<<<(F + 127) / 128, 128, 0, s>>>(nullptr, nullptr, F, 0, 0, gmax, row_exps);
  NNAB_LAUNCHED();
  const int64_t total = (int64_t)F * ld;
  coef_f16_kernel<<<grid_for(total), 256, 0, s>>>(g_bft, re_s, im_s, F, g.B, T, g.R, ld, eps, exps, row_exps,
                                                   reinterpret_cast<__half*>(coef_hi),
                                                   reinterpret_cast<__half*>(coef_lo));
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_kernel_grad_f16(const nnab_frames* f, const void* coef_hi, const void* coef_lo, int32_t rows,
                                    int64_t ld, const int32_t* row_exps, float* dk, int64_t ldk, const void* ws16,
                                    size_t ws16_bytes, int32_t staging, float* partial, int32_t splits, void* stream) {
  FrameGeom g;
  const void *hi, *lo;
  const int32_t* exps;
  int rc = f16_views(f, ws16, ws16_bytes, staging, &g, &hi, &lo, &exps);
  if (rc) return rc;
  if (!coef_hi || !row_exps || !dk || rows < 1 || ld < g.B * g.R || ld % 8) return NNAB_EINVAL;
  if (coef_lo && staging != NNAB_PREC_3XF16) return NNAB_EINVAL;  // 3xF16 reads the frames' lo rows
  if (g.row_len != g.hop || g.hop % 64) return NNAB_ENOTSUP;  // MN-major 64-column boxes of hop rows
  if (g.B == 0) return NNAB_OK;
  RGemmArgs a;
  a.M = rows;
  a.N = g.width;
  a.K = ld;
  a.a_hi = reinterpret_cast<const float*>(coef_hi);
  a.a_lo = reinterpret_cast<const float*>(coef_lo);  // null: one FP16 pass (coef and frames hi only)
  a.lda = ld;
  a.b_hi = reinterpret_cast<const float*>(hi);
  a.b_lo = coef_lo ? reinterpret_cast<const float*>(lo) : nullptr;
  a.b_mn = 1;
  a.b_row_len = g.row_len;
  a.b_rows = g.B * g.R;
  a.c = dk;
  a.ldc = ldk;
  a.splits = splits;
  a.partial = partial;
  a.row_exp = row_exps;
  return launch_rgemm(a, coef_lo ? NNAB_PREC_3XF16 : NNAB_PREC_F16, (cudaStream_t)stream);
}
