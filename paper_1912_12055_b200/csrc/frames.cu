// Frame staging and bank packing.
//
// The reference materialises every frame (`sliding_window_view(x, M)[::stride]`
// then `ascontiguousarray`, signal.py:181) after padding the clip
// (`np.pad(..., "reflect")`, signal.py:151 via transforms.py:106-107).  Here the
// padded clip is instead laid out ONCE as "hop rows": row r of clip b holds
// padded_b[r*hop, r*hop + hop).  Frame t is then rows t .. t+width/hop-1, so a
// GEMM A-tile for 128 consecutive frames and a 32-sample K block is one
// rectangular TMA box (rows g0+k/hop .., columns k%hop ..): the frames are never
// materialised, and the reflect/zero padding is resolved here with the exact
// np.pad index map (gradients.py:18-25).  When hop does not divide into 32-sample
// K blocks (or hop > width) the rows are whole frames (row_len = width rounded up).
#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {

int frame_geometry(const nnab_frames* f, FrameGeom* g) {
  if (!f || !g) return NNAB_EINVAL;
  if (f->batch < 0 || f->length < 1 || f->width < 1 || f->hop < 1 || f->pad < 0) return NNAB_EINVAL;
  if (f->pad_mode != NNAB_PAD_REFLECT && f->pad_mode != NNAB_PAD_ZERO) return NNAB_EINVAL;
  if (f->pad_mode == NNAB_PAD_REFLECT && f->pad > 0 && f->pad >= f->length) return NNAB_EINVAL;  // signal.py:147
  g->B = f->batch;
  g->L = f->length;
  g->width = f->width;
  g->hop = f->hop;
  g->pad = f->pad;
  g->pad_mode = f->pad_mode;
  g->padded_len = f->length + 2ll * f->pad;
  if (f->width > g->padded_len) return NNAB_EINVAL;  // signal.py:176-177
  int64_t T = (g->padded_len - f->width) / f->hop + 1;
  if (T > (1ll << 30)) return NNAB_ENOTSUP;
  g->T = (int32_t)T;
  g->k_pad = (f->width + 31) / 32 * 32;
  if (f->hop % 32 == 0 && f->hop <= g->k_pad) {
    g->row_len = f->hop;
    g->R = g->T + (g->k_pad + f->hop - 1) / f->hop - 1;
  } else {
    g->row_len = g->k_pad;
    g->R = g->T;
  }
  return NNAB_OK;
}

// rows[(b*R + r)*row_len + c] = padded_b[r*hop + c]  (0 beyond the padded clip),
// TF32-rounded (split=0) or split into tf32 hi + tf32 lo residual (split=1).
// One CTA walks whole rows (no 64-bit divisions per element); interior groups of
// 4 samples are one aligned 16-byte load, the reflect/zero edges go element-wise.
__global__ void __launch_bounds__(256) stage_rows_kernel(const float* __restrict__ x, int64_t B, int64_t L,
                                                         int32_t pad, int32_t mode, int32_t hop, int32_t row_len,
                                                         int32_t R, int64_t padded_len, int split,
                                                         float* __restrict__ hi, float* __restrict__ lo) {
  const int32_t q_per_row = row_len / 4;
  const int64_t rows = B * (int64_t)R;
  const bool aligned_clips = (L % 4) == 0 && (pad % 4) == 0 && (hop % 4) == 0;
  const bool x_aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int per = q_per_row < (int)blockDim.x ? q_per_row : (int)blockDim.x;  // threads per row
  const int rpb = blockDim.x / per;                                           // rows per block step
  const int sub = threadIdx.x / per, lane = threadIdx.x - sub * per;
  if (sub >= rpb) return;
  for (int64_t grow = (int64_t)blockIdx.x * rpb + sub; grow < rows; grow += (int64_t)gridDim.x * rpb) {
    const int64_t b = grow / R;
    const int64_t r = grow - b * R;
    const float* xb = x + b * L;
    float4* hrow = reinterpret_cast<float4*>(hi) + grow * q_per_row;
    float4* lrow = reinterpret_cast<float4*>(lo) + grow * q_per_row;
    for (int32_t q = lane; q < q_per_row; q += per) {
      const int64_t i0 = r * hop + 4 * q;  // padded position of the first sample
      const int64_t j0 = i0 - pad;         // source sample
      float v[4];
      const int64_t ga = b * L + j0;  // absolute source index
      if (aligned_clips && j0 >= 0 && j0 + 3 < L && i0 + 3 < padded_len) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(xb + j0));
        v[0] = w.x;
        v[1] = w.y;
        v[2] = w.z;
        v[3] = w.w;
      } else if (x_aligned && j0 >= 0 && j0 - (ga & 3) + 7 < L && i0 + 3 < padded_len) {
        // interior of a clip whose rows start off a 16-byte boundary (e.g. the CQT
        // pad of 11,341): two aligned loads and a funnel by the misalignment
        const float4* a4 = reinterpret_cast<const float4*>(x + (ga & ~int64_t(3)));
        const float4 w0 = __ldg(a4), w1 = __ldg(a4 + 1);
        const float e[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        const int m = (int)(ga & 3);
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = m == 0 ? e[u] : m == 1 ? e[u + 1] : m == 2 ? e[u + 2] : e[u + 3];
      } else if (x_aligned && mode == NNAB_PAD_REFLECT && i0 + 3 < padded_len &&
                 ((j0 + 3 < 0 && -j0 < L) || (j0 >= L && 2 * (L - 1) - j0 - 3 >= 0))) {
        // a reflected group (np.pad "reflect": one mirror image, left or right):
        // its 4 sources are one descending run -- the same funnel, reversed
        const int64_t a_lo = j0 < 0 ? -j0 - 3 : 2 * (L - 1) - j0 - 3;
        const int64_t gl = b * L + a_lo;
        if (a_lo - (gl & 3) + 7 < L) {
          const float4* a4 = reinterpret_cast<const float4*>(x + (gl & ~int64_t(3)));
          const float4 w0 = __ldg(a4), w1 = __ldg(a4 + 1);
          const float e[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
          const int m = (int)(gl & 3);
#pragma unroll
          for (int u = 0; u < 4; ++u) v[3 - u] = m == 0 ? e[u] : m == 1 ? e[u + 1] : m == 2 ? e[u + 2] : e[u + 3];
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) v[3 - u] = __ldg(xb + a_lo + u);
        }
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + u;
          float sv = 0.f;
          if (i < padded_len) {
            int64_t j = i - pad;
            if (mode == NNAB_PAD_REFLECT) {
              if (j < 0) j = -j;
              if (j >= L) j = 2 * (L - 1) - j;
              sv = __ldg(xb + j);
            } else if (j >= 0 && j < L) {
              sv = __ldg(xb + j);
            }
          }
          v[u] = sv;
        }
      }
      float4 h, l;
      h.x = tf32_rne(v[0]);
      h.y = tf32_rne(v[1]);
      h.z = tf32_rne(v[2]);
      h.w = tf32_rne(v[3]);
      hrow[q] = h;
      if (split) {
        l.x = tf32_rne(v[0] - h.x);
        l.y = tf32_rne(v[1] - h.y);
        l.z = tf32_rne(v[2] - h.z);
        l.w = tf32_rne(v[3] - h.w);
        lrow[q] = l;
      }
    }
  }
}

int stage_frames(const FrameGeom& g, const float* x, float* rows_hi, float* rows_lo, int split, cudaStream_t s) {
  const int64_t rows = g.B * (int64_t)g.R;
  if (rows == 0) return NNAB_OK;
  const int blocks = (int)std::min<int64_t>(rows, (int64_t)num_sms() * 16);
  stage_rows_kernel<<<blocks, 256, 0, s>>>(x, g.B, g.L, g.pad, g.pad_mode, g.hop, g.row_len, g.R, g.padded_len,
                                          split, rows_hi, rows_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

// Bank operand layout: tile n = rows [256n, 256n+256): 128 cosine rows of bins
// 128n.. then the 128 matching sine rows; K zero-padded to k_pad.
__global__ void pack_dft_bank_kernel(const float* __restrict__ h_re, const float* __restrict__ h_im, int32_t n_bins,
                                     int32_t n_fft, int32_t k_pad, int32_t n_tiles, int32_t fold, int32_t split,
                                     float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = (int64_t)n_tiles * 256 * k_pad;
  const int32_t n_body = fold ? n_bins - 1 : n_bins;  // bins held in the regular slots
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / k_pad;
    const int32_t k = (int32_t)(e - row * k_pad);
    const int32_t tile = (int32_t)(row / 256), col = (int32_t)(row % 256);
    const bool is_sin = col >= 128;
    const int32_t bin = tile * 128 + (col & 127);
    float v = 0.f;
    if (k < n_fft) {
      if (fold && tile == 0 && col == 128) {
        v = h_re[(int64_t)(n_bins - 1) * n_fft + k];  // Nyquist cosine in bin 0's (zero) sine slot
      } else if (bin < n_body) {
        v = (is_sin ? h_im : h_re)[(int64_t)bin * n_fft + k];
      }
    }
    const float h = tf32_rne(v);
    hi[e] = h;
    if (split) lo[e] = tf32_rne(v - h);
  }
}

}  // namespace nnab

using namespace nnab;

extern "C" int nnab_dft_bank_tiles(int32_t n_bins, int32_t fold_nyquist) {
  if (n_bins < 1) return 0;
  const int body = fold_nyquist ? n_bins - 1 : n_bins;
  return std::max(1, (body + 127) / 128);
}

extern "C" size_t nnab_dft_bank_bytes(int32_t n_bins, int32_t n_fft, int32_t fold_nyquist) {
  const int64_t k_pad = (n_fft + 31) / 32 * 32;
  return (size_t)nnab_dft_bank_tiles(n_bins, fold_nyquist) * 256 * k_pad * sizeof(float);
}

extern "C" int nnab_pack_dft_bank(const float* h_re, const float* h_im, int32_t n_bins, int32_t n_fft,
                                  int32_t fold_nyquist, int32_t precision, float* packed_hi, float* packed_lo,
                                  void* stream) {
  if (!h_re || !h_im || !packed_hi || n_bins < 1 || n_fft < 1) return NNAB_EINVAL;
  if (fold_nyquist && n_bins < 2) return NNAB_EINVAL;
  const int split = precision == NNAB_PREC_3XTF32;
  if (split && !packed_lo) return NNAB_EINVAL;
  const int32_t k_pad = (n_fft + 31) / 32 * 32;
  const int32_t tiles = nnab_dft_bank_tiles(n_bins, fold_nyquist);
  const int64_t total = (int64_t)tiles * 256 * k_pad;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
  pack_dft_bank_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(h_re, h_im, n_bins, n_fft, k_pad, tiles,
                                                                 fold_nyquist, split, packed_hi, packed_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_frames_geometry(const nnab_frames* f, int32_t* n_frames, int32_t* row_len, int32_t* rows) {
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  if (n_frames) *n_frames = g.T;
  if (row_len) *row_len = g.row_len;
  if (rows) *rows = g.R;
  return NNAB_OK;
}
