// One C-ABI call for spectrogram_vjp (gradients.py:103-149) of a trainable
// DFT-type layer, with or without the Mel stage: the composition
// autograd.DftLayerOp runs from Python (training forward with the saved
// operands, then the backward GEMMs), for C / FFI callers that bind the
// boundary directly.  Like the reference it recomputes the forward.
#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

extern "C" int nnab_stage_frames(const nnab_frames* f, const float* x, int32_t precision, void* workspace,
                                 size_t workspace_bytes, void* stream);

namespace nnab {
namespace {

// dst[c][r] = [h_re; h_im][r][c] for r < 2F, 0 up to ld (the input-gradient
// GEMM's A operand, gradients.py:133-149); TF32 hi (+ lo)
__global__ void transpose_bank_kernel(const float* __restrict__ h_re, const float* __restrict__ h_im, int32_t F,
                                      int32_t n_fft, int32_t ld, int split, float* __restrict__ hi,
                                      float* __restrict__ lo) {
  const int64_t total = (int64_t)n_fft * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / ld;
    const int r = (int)(e - c * ld);
    const float v = r < F ? h_re[(int64_t)r * n_fft + c] : r < 2 * F ? h_im[(int64_t)(r - F) * n_fft + c] : 0.f;
    const float h = tf32_rne(v);
    hi[e] = h;
    if (split) lo[e] = tf32_rne(v - h);
  }
}

size_t al(size_t v) { return (v + 255) & ~size_t(255); }

struct VjpLayout {
  size_t stft, bank3, ph, im, mag, mag_lo, gs, coef, part, ht, fgt, total;
  int32_t kp_2f;
  int64_t ld;
};

int vjp_layout(const nnab_frames* f, int32_t n_bins, int32_t n_mels, int32_t precision, int32_t need_x,
               VjpLayout* o) {
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  const int split = precision == NNAB_PREC_3XTF32;
  const int64_t ld = nnab_slots_ld(f);
  const int64_t F = n_bins, n_fft = g.width;
  const size_t cell = (size_t)F * ld * 4;
  VjpLayout L{};
  L.ld = ld;
  L.kp_2f = (int32_t)((2 * F + 31) / 32 * 32);
  // TF32 convolution layer: 3xTF32 staging (its hi rows are the TF32 frames of dK) and a
  // 3xTF32 bank for the split forward that saves an FP32-accurate phasor
  const bool split_fwd = !split && n_mels == 0;
  L.stft = al(nnab_stft_workspace_bytes(f, split_fwd ? NNAB_PREC_3XTF32 : precision));
  L.bank3 = split_fwd ? 2 * al(nnab_dft_bank_bytes((int32_t)F, (int32_t)n_fft, 0)) : 0;
  L.ph = al(cell);
  L.im = split ? al(cell) : 0;
  L.mag = n_mels > 0 ? al(cell) : 0;
  L.mag_lo = (n_mels > 0 && split) ? al(cell) : 0;
  L.gs = n_mels > 0 ? al((size_t)n_mels * ld * 4) * (split ? 2 : 1) : 0;
  L.coef = al((size_t)2 * F * ld * 4) * (split ? 2 : 1);
  L.part = al(std::max({rgemm_partial_bytes((int32_t)(2 * F), (int32_t)n_fft, ld, 0),
                        n_mels > 0 ? rgemm_partial_bytes(n_mels, (int32_t)F, ld, 0) : (size_t)0,
                        need_x ? rgemm_partial_bytes((int32_t)n_fft, (int32_t)ld, L.kp_2f, 0) : (size_t)0,
                        (size_t)256}));
  L.ht = need_x ? al((size_t)n_fft * L.kp_2f * 4) * (split ? 2 : 1) : 0;
  L.fgt = need_x ? al((size_t)n_fft * ld * 4) : 0;
  L.total = L.stft + L.bank3 + L.ph + L.im + L.mag + L.mag_lo + L.gs + L.coef + L.part + L.ht + L.fgt;
  *o = L;
  return NNAB_OK;
}

int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8); }

}  // namespace
}  // namespace nnab

using namespace nnab;

// Device bytes nnab_layer_vjp needs (n_mels = 0: convolution layer).
extern "C" size_t nnab_layer_vjp_workspace_bytes(const nnab_frames* f, int32_t n_bins, int32_t n_mels,
                                                 int32_t precision, int32_t need_x) {
  VjpLayout L;
  return vjp_layout(f, n_bins, n_mels, precision, need_x, &L) ? 0 : L.total;
}

// spectrogram_vjp (gradients.py:103-149) for the layer "S = sqrt(|bank . frame|^2 + eps)"
// (n_mels = 0) or "W @ S" (n_mels > 0, W = mel_w [n_mels][n_bins], fixed DFT stage).
//   x (B, L) device; packed_hi/lo: the bank packed by nnab_pack_dft_bank (fold 0);
//   h_re/h_im (n_bins, n_fft): the same bank unpacked (for the input gradient);
//   upstream (B, n_mels or n_bins, T);
//   outputs (any may be NULL): d_h (2 n_bins, n_fft) = [dh_re; dh_im] (conv layer),
//   d_w (n_mels, n_bins) (mel layer), d_x (B, L) (conv layer only, like the reference).
// Kernel gradients are summed over the batch.  EINVAL mirrors the reference:
// d_x with a Mel layer (NotImplementedError there), inconsistent sizes.
extern "C" int nnab_layer_vjp(const nnab_frames* f, const float* x, const float* packed_hi, const float* packed_lo,
                              int32_t n_bins, const float* h_re, const float* h_im, const float* mel_w,
                              int32_t n_mels, const float* upstream, float eps, int32_t precision, float* d_h,
                              float* d_w, float* d_x, void* workspace, size_t workspace_bytes, void* stream) {
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  const int split = precision == NNAB_PREC_3XTF32;
  if (precision != NNAB_PREC_TF32 && !split) return NNAB_EINVAL;
  if (!x || !packed_hi || (split && !packed_lo) || !upstream || n_bins < 1 || n_mels < 0) return NNAB_EINVAL;
  if (n_mels > 0 && (!mel_w || d_h || d_x)) return NNAB_EINVAL;  // mel layer: weights gradient only
  if (d_x && (!h_re || !h_im)) return NNAB_EINVAL;
  VjpLayout Lo;
  if ((rc = vjp_layout(f, n_bins, n_mels, precision, d_x != nullptr, &Lo))) return rc;
  if (!workspace || workspace_bytes < Lo.total) return NNAB_EINVAL;
  if (g.B == 0) return NNAB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ld = Lo.ld, F = n_bins, n_fft = g.width;
  char* p = reinterpret_cast<char*>(workspace);
  auto take = [&](size_t n) { char* r = p; p += n; return n ? reinterpret_cast<float*>(r) : nullptr; };
  void* ws = take(Lo.stft);
  float* bank3 = take(Lo.bank3);
  float* ph = take(Lo.ph);
  float* im = take(Lo.im);
  float* mag = take(Lo.mag);
  float* mag_lo = take(Lo.mag_lo);
  float* gs = take(Lo.gs);
  float* coef = take(Lo.coef);
  float* part = take(Lo.part);
  float* ht = take(Lo.ht);
  float* fgt = take(Lo.fgt);
  auto lo_of = [&](float* a, size_t bytes) {  // the lo half of a hi/lo allocation (3xTF32)
    return split ? reinterpret_cast<float*>(reinterpret_cast<char*>(a) + bytes / 2) : nullptr;
  };

  // forward with the saved operands (gradients.py:61-80).  TF32 convolution layer with the
  // unpacked bank at hand: the forward runs 3xTF32 and saves the TF32-backward format, so
  // the phasor re/S, im/S weighing every frame is FP32-accurate where |X| is small
  if (Lo.bank3 && h_re && h_im) {
    const size_t bb = Lo.bank3 / 2;
    float* b3_lo = reinterpret_cast<float*>(reinterpret_cast<char*>(bank3) + bb);
    if ((rc = nnab_pack_dft_bank(h_re, h_im, n_bins, (int32_t)n_fft, 0, NNAB_PREC_3XTF32, bank3, b3_lo, stream)))
      return rc;
    if ((rc = nnab_stage_frames(f, x, NNAB_PREC_3XTF32, ws, Lo.stft, stream))) return rc;
    if ((rc = nnab_stft_forward_train_staged(f, bank3, b3_lo, n_bins, 0, NNAB_PREC_3XTF32,
                                             NNAB_OUT_SMOOTH_MAG | NNAB_SAVE_PHASOR, 1.f, eps, nullptr, 0, 0, nullptr,
                                             nullptr, ph, nullptr, mag, ld, ws, Lo.stft, stream)))
      return rc;
  } else {
    if ((rc = nnab_stage_frames(f, x, precision, ws, Lo.stft, stream))) return rc;
    if ((rc = nnab_stft_forward_train_staged(f, packed_hi, packed_lo, n_bins, 0, precision, NNAB_OUT_SMOOTH_MAG,
                                             1.f, eps, nullptr, 0, 0, nullptr, nullptr, ph, im, mag, ld, ws, Lo.stft,
                                             stream)))
      return rc;
  }
  const float* coef_lo = split ? lo_of(coef, Lo.coef) : nullptr;
  if (n_mels > 0) {
    // mel layer (gradients.py:118-121): dW = g @ S^T; g to slots fused with the operand split
    float* gs_lo = lo_of(gs, Lo.gs);
    if ((rc = nnab_grad_to_slots_split(upstream, g.B, n_mels, g.T, g.R, ld, precision, gs, gs_lo, stream))) return rc;
    if (split) {
      if ((rc = nnab_tf32_split(mag, F * ld, precision, mag, mag_lo, stream))) return rc;
    }
    if (d_w && (rc = nnab_rgemm(n_mels, n_bins, ld, gs, gs_lo, ld, mag, mag_lo, ld, 0, 0, 0, d_w, n_bins, 0, part,
                                precision, stream)))
      return rc;
    return NNAB_OK;
  }
  // convolution layer (gradients.py:125-129): coef = g*re/S, g*im/S, then dh = coef @ frames
  if ((rc = nnab_dft_coef(nullptr, upstream, ph, im, n_bins, g.B, g.T, g.R, ld, eps, precision, coef,
                          const_cast<float*>(coef_lo), stream)))
    return rc;
  if (d_h && (rc = nnab_kernel_grad(f, coef, coef_lo, 2 * n_bins, ld, precision, d_h, n_fft, ws, Lo.stft, part, 0,
                                    stream)))
    return rc;
  if (d_x) {
    // input gradient (gradients.py:133-149): frame grads^T = h^T @ coef, overlap-add, pad fold
    float* ht_lo = lo_of(ht, Lo.ht);
    const int64_t n = (int64_t)n_fft * Lo.kp_2f;
    transpose_bank_kernel<<<blocks_for(n), 256, 0, s>>>(h_re, h_im, n_bins, (int32_t)n_fft, Lo.kp_2f, split, ht,
                                                        ht_lo);
    NNAB_LAUNCHED();
    if ((rc = nnab_rgemm((int32_t)n_fft, (int32_t)ld, Lo.kp_2f, ht, ht_lo, Lo.kp_2f, coef, coef_lo, ld, 1,
                         (int32_t)ld, 2 * n_bins, fgt, ld, 0, part, precision, stream)))
      return rc;
    if ((rc = nnab_input_grad(f, fgt, ld, d_x, stream))) return rc;
  }
  return NNAB_OK;
}
