/*
 * nnab -- B200 (sm_100a) spectrogram kernels behind a plain C ABI.
 *
 * This is the drop-in boundary for the `spectro` reference's hot path
 * (/root/reference/pkg/src/spectro).  The reference is pure Python/NumPy, so
 * its "FFI" is the call a Python caller makes; every entry point below names
 * the reference function it replaces (file:line, relative to
 * pkg/src/spectro/).  The Python host mirror in paper_1912_12055_b200/ binds
 * these symbols with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - All float pointers are DEVICE pointers (caller-allocated) unless a
 *    function says otherwise; execution is stream-ordered on `stream`
 *    (a cudaStream_t passed as void*).  No call allocates device memory:
 *    scratch comes from a caller-supplied workspace sized by the matching
 *    *_workspace_bytes() query.
 *  - Calls are re-entrant and hold no global mutable state.
 *  - Return value: NNAB_OK or an NNAB_E* code; nnab_strerror() names it.
 *    NNAB_EINVAL mirrors the reference's ValueError cases (reflect pad >=
 *    signal length signal.py:147-150, kernel longer than padded signal
 *    signal.py:176-177, hop < 1 signal.py:178-179, CQT hop divisibility
 *    transforms.py:253-257).
 *  - Signals are float32 (B, L) row-major; spectrogram outputs are
 *    (B, F, T) row-major float32 (complex outputs: interleaved (re, im)
 *    float pairs, i.e. complex64), matching nnAudio's (batch, freq, time).
 */
#ifndef NNAB_H
#define NNAB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NNAB_OK 0
#define NNAB_EINVAL 1   /* bad argument (reference raises ValueError) */
#define NNAB_ECUDA 2    /* CUDA runtime / driver error */
#define NNAB_ENOTSUP 3  /* configuration not supported by the sm_100a kernels */
#define NNAB_ENODEV 4   /* no sm_100 device */

#define NNAB_PAD_REFLECT 0 /* np.pad(..., "reflect"): mirror without the edge sample */
#define NNAB_PAD_ZERO 1    /* "constant_zero" */

#define NNAB_OUT_MAGNITUDE 0 /* hypot(re, im)            transforms.py:86-93 */
#define NNAB_OUT_POWER 1     /* re^2 + im^2                                 */
#define NNAB_OUT_COMPLEX 2   /* re - i*im (interleaved complex64)            */
#define NNAB_OUT_MEL 3       /* W @ |X|^power            transforms.py:164-172 */
#define NNAB_OUT_SMOOTH_MAG 4 /* sqrt(re^2+im^2+eps)      gradients.py:61-67 */
/* flag, OR-ed into NNAB_OUT_MAGNITUDE / NNAB_OUT_POWER / NNAB_OUT_MEL of the
 * STFT entry points: the fused epilogue writes log(value + eps) (log
 * compression, north_star item 3; the reference has no log op, so parity is
 * log of the parity-checked value).  With it, eps is the log offset only (the
 * Mel magnitude is the plain sqrt(re^2 + im^2)). */
#define NNAB_OUT_LOG 0x100
/* flag, OR-ed into the out_kind of nnab_stft_forward_train_staged: save the
 * TF32-backward format (FP16 unit phasor re/S, im/S in save_re, TF32-rounded |X|
 * in save_mag) from a split-precision forward (3xTF32 / 3xF16), so the phasor
 * that weighs every frame in the kernel gradient is FP32-accurate even where
 * |X| is small, while the backward GEMMs stay TF32. */
#define NNAB_SAVE_PHASOR 0x200
/* flag (split modes without NNAB_SAVE_PHASOR): save_mag is [2][n_bins][ld], the
 * TF32 hi of |X| then its TF32 residual -- the 3xTF32 operand pair of the Mel
 * layer's forward W @ S and dW = g S^T, with no separate split pass. */
#define NNAB_SAVE_MAG_SPLIT 0x400

#define NNAB_PREC_TF32 0  /* one TF32 tcgen05 pass (peak-normalised error <= 1e-3) */
#define NNAB_PREC_3XTF32 1 /* hi/lo split, 3 passes (<= 1e-5, FP32-equivalent) */
/* FP16 operands under exact power-of-two scales (per clip for the signal, per
 * bank for the kernels) so every operand sits in FP16's normal range: the same
 * 11-bit significand as TF32 at twice the tcgen05 rate (kind::f16, FP32
 * accumulate); the scales are undone exactly in the epilogue.  STFT / Mel and
 * CQT1992v2 (hybrid E-GEMM + schedule). */
#define NNAB_PREC_F16 2   /* one FP16 pass (<= 1e-3) */
#define NNAB_PREC_3XF16 3 /* FP16 hi/lo split, 3 passes (<= 1e-5) */

/* A strided-correlation ("conv1d with a kernel bank") problem:
 * out[r, t] = sum_m padded[t*hop + m] * bank[r, m]   (signal.py:159-183)  */
typedef struct nnab_frames {
  int64_t batch;    /* B clips */
  int64_t length;   /* L samples per clip */
  int32_t width;    /* kernel width M (n_fft, or the CQT bank width) */
  int32_t hop;      /* stride between frames */
  int32_t pad;      /* samples padded on each side (n_fft//2 when centred) */
  int32_t pad_mode; /* NNAB_PAD_* */
} nnab_frames;

/* ---------------------------------------------------------------- misc */
int nnab_version(void);
const char* nnab_strerror(int code);
/* last CUDA error string recorded by a failing call on this thread */
const char* nnab_last_error(void);
/* kernels this library has launched in the process (all threads) */
uint64_t nnab_launch_count(void);
/* number of frames T and the staging layout for a problem; NNAB_EINVAL for
 * the reference's ValueError cases. */
int nnab_frames_geometry(const nnab_frames* f, int32_t* n_frames, int32_t* row_len, int32_t* rows_per_clip);

/* --------------------------------------------------- bank preparation
 * Pack a DFT bank (h_re, h_im: (n_bins, n_fft) float32 device rows,
 * kernels.py:137-146) into the GEMM operand layout: tiles of 256 rows
 * (128 cos rows, 128 sin rows), K padded to a multiple of 32, TF32-rounded.
 * With 3xTF32 a second (lo) array receives the rounding residual.
 * fold_nyquist: bins 0 and n_bins-1 have all-zero sine rows (the default
 * integer-bin bank), so bin n_bins-1's cosine row takes the sine slot of bin 0
 * and the bank tiles exactly (1025 bins -> 8 tiles).                    */
int nnab_dft_bank_tiles(int32_t n_bins, int32_t fold_nyquist);
size_t nnab_dft_bank_bytes(int32_t n_bins, int32_t n_fft, int32_t fold_nyquist);
/* bytes of each packed array (hi, and lo for the split modes) for `precision`:
 * the FP16 modes store halves (K padded to 64) plus a 256-byte trailer in the
 * hi array holding the bank's scale exponent; = nnab_dft_bank_bytes for TF32. */
size_t nnab_dft_bank_bytes_prec(int32_t n_bins, int32_t n_fft, int32_t fold_nyquist, int32_t precision);
int nnab_pack_dft_bank(const float* h_re, const float* h_im, int32_t n_bins, int32_t n_fft,
                       int32_t fold_nyquist, int32_t precision, float* packed_hi, float* packed_lo,
                       void* stream);

/* ------------------------------------------------------- STFT / Mel
 * Stft.__call__ (transforms.py:130-144), MelSpec.__call__ (transforms.py:164-172),
 * TrainableLayer.spectrogram for DFT banks (gradients.py:61-67, out_kind
 * NNAB_OUT_SMOOTH_MAG with eps).
 *  x          (B, L) float32
 *  packed_*   from nnab_pack_dft_bank (lo only for 3xTF32, else may be NULL)
 *  mel_w      (n_mels, mel_ld) float32, zero-padded rows (NNAB_OUT_MEL only)
 *  mel_band   optional int32 pairs [lo, hi) of mel rows touching each 32-bin
 *             chunk (NULL = dense W)
 *  out        (B, n_bins, T) float32 | (B, n_bins, T, 2) | (B, n_mels, T)   */
size_t nnab_stft_workspace_bytes(const nnab_frames* f, int32_t precision);
int nnab_stft_forward(const nnab_frames* f, const float* x, const float* packed_hi, const float* packed_lo,
                      int32_t n_bins, int32_t fold_nyquist, int32_t precision, int32_t out_kind, float power,
                      float eps, const float* mel_w, int32_t n_mels, int32_t mel_ld, const int32_t* mel_band,
                      float* out, void* workspace, size_t workspace_bytes, void* stream);

/* The two phases of nnab_stft_forward, for callers that reuse staged frames
 * (the backward pass re-reads them for the kernel gradient) or time the GEMM
 * alone.  Stage: pad (np.pad index map, signal.py:151 / gradients.py:18-25)
 * and lay the clips out as hop rows in `workspace`, TF32-rounded (3xTF32: hi
 * and lo halves).  Staged forward: the tcgen05 GEMM + fused epilogue on them. */
int nnab_stage_frames(const nnab_frames* f, const float* x, int32_t precision, void* workspace,
                      size_t workspace_bytes, void* stream);
int nnab_stft_forward_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo, int32_t n_bins,
                             int32_t fold_nyquist, int32_t precision, int32_t out_kind, float power, float eps,
                             const float* mel_w, int32_t n_mels, int32_t mel_ld, const int32_t* mel_band,
                             float* out, const void* workspace, size_t workspace_bytes, void* stream);

/* Host-buffer end-to-end variant (the call a CPU caller of the reference
 * makes): x_host and out_host are pinned host buffers; the batch is streamed
 * through the device in chunks so H2D, compute and D2H overlap.  All device
 * buffers (x chunk, workspace, out chunk) come from `device_scratch`. */
size_t nnab_stft_host_scratch_bytes(const nnab_frames* f, int32_t precision, int32_t out_rows,
                                    int64_t chunk_clips);
int nnab_stft_forward_host(const nnab_frames* f, const float* x_host, const float* packed_hi,
                           const float* packed_lo, int32_t n_bins, int32_t fold_nyquist, int32_t precision,
                           int32_t out_kind, float power, float eps, const float* mel_w, int32_t n_mels,
                           int32_t mel_ld, const int32_t* mel_band, float* out_host, int64_t chunk_clips,
                           void* device_scratch, size_t scratch_bytes, void* stream);

/* spectrogram_vjp (gradients.py:103-149) in one call, recomputing the forward
 * like the reference: convolution layer (n_mels = 0; d_h = [dh_re; dh_im]
 * (2 n_bins, n_fft), optional d_x (B, L)) or Mel layer over a fixed DFT stage
 * (n_mels > 0; d_w (n_mels, n_bins); d_h / d_x must be NULL, the reference
 * raises NotImplementedError for the Mel input gradient).  packed_*: the bank
 * from nnab_pack_dft_bank (fold 0); h_re / h_im: the same bank unpacked (needed
 * for d_x; in TF32 mode they also let the convolution layer's forward run
 * 3xTF32 so the phasor re/S, im/S that weighs every frame's gradient is
 * FP32-accurate where |X| is small -- NULL keeps the one-pass TF32 forward);
 * upstream (B, rows, T).  Kernel gradients are summed over the batch. */
size_t nnab_layer_vjp_workspace_bytes(const nnab_frames* f, int32_t n_bins, int32_t n_mels, int32_t precision,
                                      int32_t need_x);
int nnab_layer_vjp(const nnab_frames* f, const float* x, const float* packed_hi, const float* packed_lo,
                   int32_t n_bins, const float* h_re, const float* h_im, const float* mel_w, int32_t n_mels,
                   const float* upstream, float eps, int32_t precision, float* d_h, float* d_w, float* d_x,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------- signal primitives
 * The reference's signal.py primitives as standalone device ops (the
 * transforms fuse them into their own kernels).  Device pointers, stream-ordered. */
/* pad_signal (signal.py:138-156): x (B, L) -> y (B, L + left + right), mode
 * NNAB_PAD_REFLECT / NNAB_PAD_ZERO, bit-exact; EINVAL for negative pads or a
 * reflect pad >= L (the reference's ValueErrors). */
int nnab_pad_signal(const float* x, int64_t B, int64_t L, int64_t left, int64_t right, int32_t mode, float* y,
                    void* stream);
/* downsample2 (signal.py:232-247): reflect pad (n_taps-1)/2, np.convolve-valid
 * with the (device) taps, keep even samples: y (B, ceil(L/2)); EINVAL for an
 * even n_taps or L < n_taps. */
int nnab_downsample2(const float* x, int64_t B, int64_t L, const float* taps, int32_t n_taps, float* y,
                     void* stream);

/* ------------------------------------------------------- trainable layers
 * TrainableLayer / spectrogram_vjp (gradients.py:28-149) on the device.
 * Frame slots: clip b, frame t -> slot b*R + t (R = rows per clip from
 * nnab_frames_geometry); slot-major arrays are [rows][ld], ld = nnab_slots_ld. */
int64_t nnab_slots_ld(const nnab_frames* f);
/* Training forward on staged frames: out = smoothed magnitude sqrt(re^2+im^2+eps)
 * (NNAB_OUT_SMOOTH_MAG, gradients.py:61-67) or W @ that (NNAB_OUT_MEL,
 * gradients.py:69-80); also stores re, im and (if save_mag) S, slot-major.
 * TF32 only: save_im = NULL stores the unit phasor (re/S, im/S) instead, as
 * packed FP16 pairs (one 32-bit word per (bin, slot) in save_re) -- all the
 * backward's coef step needs; nnab_dft_coef / nnab_mel_dft_coef then take
 * im_s = NULL and re_s = that phasor array. */
int nnab_stft_forward_train_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo,
                                   int32_t n_bins, int32_t fold_nyquist, int32_t precision, int32_t out_kind,
                                   float power, float eps, const float* mel_w, int32_t n_mels, int32_t mel_ld,
                                   const int32_t* mel_band, float* out, float* save_re, float* save_im,
                                   float* save_mag, int64_t ld, const void* workspace, size_t workspace_bytes,
                                   void* stream);
/* (B, rows, T) -> slot-major [rows][ld], zero on non-frame slots */
int nnab_grad_to_slots(const float* g_brt, int64_t B, int32_t rows, int32_t T, int32_t R, int64_t ld, float* out,
                       void* stream);
/* the same, fused with the GEMM-operand split: hi = TF32(g) (+ lo = TF32(g - hi) in 3xTF32) */
int nnab_grad_to_slots_split(const float* g_brt, int64_t B, int32_t rows, int32_t T, int32_t R, int64_t ld,
                             int32_t precision, float* hi, float* lo, void* stream);
/* slot-major [rows][ld] -> (B, rows, T) */
int nnab_from_slots(const float* src, int64_t B, int32_t rows, int32_t T, int32_t R, int64_t ld, float* out_brt,
                    void* stream);
/* coef = dS*re/S (rows 0..F-1) and dS*im/S (rows F..2F-1), gradients.py:127-128;
 * dS from ds_slots ([F][ld]) or g_bft ((B, F, T)); TF32 hi (+ lo residual). */
int nnab_dft_coef(const float* ds_slots, const float* g_bft, const float* re_s, const float* im_s, int32_t F,
                  int64_t B, int32_t T, int32_t R, int64_t ld, float eps, int32_t precision, float* coef_hi,
                  float* coef_lo, void* stream);
/* Mel layer forward of the trainable layer (gradients.py:69-80): W @ S on the
 * slot-major smoothed magnitude S [F][ld] (save_mag of the training forward),
 * written as (B, n_mels, T).  w = W zero-padded to [n_mels][kp], kp = F
 * rounded up to 32 (<= 2048, else NNAB_ENOTSUP); R % 4 == 0. */
int nnab_mel_forward_slots(int32_t n_mels, int64_t ld, int32_t kp, const float* w_hi, const float* w_lo,
                           const float* s_hi, const float* s_lo, int32_t F, int64_t B, int32_t R, int32_t T,
                           int32_t precision, float* out, void* stream);
/* Joint mel + trainable STFT backward: dS = W^T g computed on the tensor cores
 * with the coef step (gradients.py:125-128) in the GEMM epilogue, so dS never
 * reaches HBM.  wt = W^T zero-padded to [F][kp] (kp = n_mels rounded up to 32,
 * <= 1024), gs = upstream grad in slot layout [n_mels][ld]; writes coef [2F][ld]
 * like nnab_dft_coef(ds_slots = W^T g). */
int nnab_mel_dft_coef(int32_t F, int64_t ld, int32_t kp, const float* wt_hi, const float* wt_lo, const float* gs_hi,
                      const float* gs_lo, int32_t n_mels, const float* re_s, const float* im_s, float eps,
                      int32_t precision, float* coef_hi, float* coef_lo, void* stream);
/* dst[c][r] = src[r][c] zero-padded to ld rows, TF32 hi (+ lo) */
int nnab_transpose_pad(const float* src, int32_t rows, int32_t cols, int32_t ld, int32_t precision, float* hi,
                       float* lo, void* stream);
int nnab_tf32_split(const float* src, int64_t n, int32_t precision, float* hi, float* lo, void* stream);
/* C[M][N] = sum_k A[M][k] B(k, N) on tcgen05; B K-major (b_mn = 0: row n at
 * b + n*ldb) or MN-major ((k, n) at rows[k + n/b_row_len][n % b_row_len]);
 * split-K partials (deterministic fixed-order sum) in `partial`. */
size_t nnab_rgemm_partial_bytes(int32_t M, int32_t N, int64_t K, int32_t splits);
int nnab_rgemm(int32_t M, int32_t N, int64_t K, const float* a_hi, const float* a_lo, int64_t lda, const float* b_hi,
               const float* b_lo, int64_t ldb, int32_t b_mn, int32_t b_row_len, int64_t b_rows, float* c,
               int64_t ldc, int32_t splits, float* partial, int32_t precision, void* stream);
/* dK = coef @ frames (gradients.py:129) with the frames read from the staged rows */
int nnab_kernel_grad(const nnab_frames* f, const float* coef_hi, const float* coef_lo, int32_t rows, int64_t ld,
                     int32_t precision, float* dk, int64_t ldk, const void* workspace, size_t workspace_bytes,
                     float* partial, int32_t splits, void* stream);
/* FP32-mode (<= 1e-5) kernel gradient on FP16 tensor cores (3xF16): the coef
 * operand is written as FP16 hi/lo of coef * 2^(row_exps[m] - e_b) (e_b: clip b's
 * staging exponent), the frames are the 3xF16 training forward's staged rows
 * (ws16: its nnab_stage_frames workspace, staged in `staging` = NNAB_PREC_3XF16, or
 * NNAB_PREC_F16 for the one-pass form; hop % 64 == 0), and
 * the GEMM's epilogue multiplies row m by 2^-row_exps[m].  row_exps: int32[2F + 1]
 * (the last word is scratch).  coef_hi/coef_lo: FP16 [2F][ld]; ld % 8 == 0.
 * Replaces nnab_dft_coef / nnab_mel_dft_coef + nnab_kernel_grad in NNAB_PREC_3XTF32
 * (gradients.py:125-129); the row exponent comes from a bound on |dS| (no pass over coef).
 * coef_lo = NULL: one FP16 pass (11-bit operands, the TF32 mode's accuracy): coef hi only,
 * the frames' hi rows only; the coef inputs may then be TF32 (wt_lo / gs_lo NULL) and
 * re_s the FP16 unit phasor of a TF32-backward forward (im_s NULL). */
int nnab_mel_dft_coef_f16(const nnab_frames* f, const void* ws16, size_t ws16_bytes, int32_t staging, int32_t F, int64_t ld,
                          int32_t kp, const float* wt_hi, const float* wt_lo, const float* gs_hi, const float* gs_lo,
                          int32_t n_mels, const float* re_s, const float* im_s, float eps, void* coef_hi,
                          void* coef_lo, int32_t* row_exps, void* stream);
int nnab_dft_coef_f16(const nnab_frames* f, const void* ws16, size_t ws16_bytes, int32_t staging, const float* g_bft,
                      const float* re_s, const float* im_s, int32_t F, int32_t T, int64_t ld, float eps,
                      void* coef_hi, void* coef_lo, int32_t* row_exps, void* stream);
int nnab_kernel_grad_f16(const nnab_frames* f, const void* coef_hi, const void* coef_lo, int32_t rows, int64_t ld,
                         const int32_t* row_exps, float* dk, int64_t ldk, const void* ws16, size_t ws16_bytes,
                         int32_t staging, float* partial, int32_t splits, void* stream);
/* dx: overlap-add of frame grads ([tap][ld] = h^T @ coef) folded through the
 * pad index map (gradients.py:133-149); deterministic gather, (B, L) out. */
int nnab_input_grad(const nnab_frames* f, const float* frame_grads_t, int64_t ld, float* gx, void* stream);

/* ------------------------------------------------------- CQT1992v2
 * Cqt1992v2.__call__ (transforms.py:201-208 via _complex_conv 175-186) and
 * TrainableLayer.spectrogram for CQT banks (gradients.py:61-67).
 * Bank: k_re/k_im (n_bins, width) float32 device rows (kernels.py:361-402),
 * packed with re/im rows of each bin interleaved.  `schedule` (device, from
 * nnab_cqt_schedule over each row's non-zero support) lists the K blocks in
 * longest-first order with the MMA width each needs.
 * out: (B, n_bins, T) float32, or complex64 re + i*im for NNAB_OUT_COMPLEX. */
int nnab_cqt_bank_tiles(int32_t n_bins);
size_t nnab_cqt_bank_bytes(int32_t n_bins, int32_t width);
/* bytes of each packed schedule-bank array for `precision` (FP16 modes: halves, K
 * padded to 64, plus a 256-byte scale trailer in the hi array) */
size_t nnab_cqt_bank_bytes_prec(int32_t n_bins, int32_t width, int32_t precision);
int nnab_pack_cqt_bank(const float* k_re, const float* k_im, int32_t n_bins, int32_t width, int32_t precision,
                       float* packed_hi, float* packed_lo, void* stream);
/* host-only: support[2*bin], support[2*bin+1] = non-zero column range [begin, end)
 * of each row; table_host capacity n_tiles * width/16 + 16 entries. */
int nnab_cqt_schedule(const int32_t* support, int32_t n_bins, int32_t width, int32_t precision,
                      uint32_t* table_host, int32_t* n_entries);
int nnab_cqt1992v2_forward(const nnab_frames* f, const float* x, const float* packed_hi, const float* packed_lo,
                           int32_t n_bins, const uint32_t* schedule, int32_t n_entries, int32_t precision,
                           int32_t out_kind, float eps, float* out, void* workspace, size_t workspace_bytes,
                           void* stream);
/* GEMM phase only, on frames already staged by nnab_stage_frames */
int nnab_cqt1992v2_forward_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo,
                                  int32_t n_bins, const uint32_t* schedule, int32_t n_entries, int32_t precision,
                                  int32_t out_kind, float eps, float* out, const void* workspace,
                                  size_t workspace_bytes, void* stream);

/* CQT1992v2 as a hop-offset GEMM ("E-GEMM", csrc/cqt1992_egemm.cu):
 * E[s][(row, r)] = sum_c rows[s][c] K[row][hop r + c] over the (row, r) pairs a
 * row's support touches, D[s][row] = sum_r E[s + r][(row, r)] in a shared-memory
 * ring, fused magnitude.  Same result as nnab_cqt1992v2_forward (TF32 only).
 * nnab_cqt_egemm_plan (host) groups whole bins' columns (<= 256 per group,
 * sorted by r): col_table [max_groups*256] = row_local << 8 | r (0xFFFF
 * unused), group_rows [max_groups*64] = bank row 2*bin (+1 for Im) or -1. */
int nnab_cqt_egemm_plan(const int32_t* support, int32_t n_bins, int32_t width, int32_t hop, int32_t max_groups,
                        uint16_t* col_table, int32_t* group_rows, uint32_t* run_table /* [max_groups*4*65] */,
                        int32_t* n_groups, int32_t* r_max);
size_t nnab_cqt_egemm_bank_bytes(int32_t n_groups, int32_t hop);
/* the same for `precision` (FP16 modes: halves plus a 256-byte scale trailer) */
size_t nnab_cqt_egemm_bank_bytes_prec(int32_t n_groups, int32_t hop, int32_t precision);
int nnab_pack_cqt_egemm(const float* k_re, const float* k_im, int32_t width, int32_t hop, const uint16_t* col_table,
                        const int32_t* group_rows, int32_t n_groups, int32_t precision, float* packed_hi,
                        float* packed_lo, void* stream);
int nnab_cqt1992v2_egemm_staged(const nnab_frames* f, const float* packed_hi, const uint16_t* col_table,
                                const int32_t* group_rows, const uint32_t* run_table, int32_t n_groups,
                                int32_t r_max, int32_t n_bins,
                                int32_t out_kind, float eps, float* out, const void* workspace,
                                size_t workspace_bytes, void* stream);
/* CQT1992v2 hybrid: bins [0, n_long) on the E-GEMM (eg_bank/col_table/
 * group_rows/n_groups/r_max from nnab_cqt_egemm_plan + nnab_pack_cqt_egemm over
 * those bins), bins [n_long, n_bins) on the per-K-block schedule (sched_bank and
 * schedule of those rows at the same width), both from one staging of the
 * frames; out (B, n_bins, T).  TF32, or 3xTF32 with the *_lo banks (the
 * E-GEMM then runs as CTA pairs with main + correction accumulators).
 * Replaces the reference's single DGEMM (transforms.py:175-208). */
int nnab_cqt1992v2_hybrid_staged(const nnab_frames* f, const float* eg_bank, const float* eg_bank_lo,
                                 const uint16_t* col_table, const int32_t* group_rows, int32_t n_groups,
                                 int32_t r_max, const float* sched_bank, const float* sched_bank_lo,
                                 const uint32_t* schedule, int32_t n_entries, int32_t n_long, int32_t n_bins,
                                 int32_t precision, int32_t out_kind, float eps, float* out, const void* workspace,
                                 size_t workspace_bytes, void* stream);
int nnab_cqt1992v2_hybrid_forward(const nnab_frames* f, const float* x, const float* eg_bank,
                                  const float* eg_bank_lo, const uint16_t* col_table, const int32_t* group_rows,
                                  int32_t n_groups, int32_t r_max, const float* sched_bank,
                                  const float* sched_bank_lo, const uint32_t* schedule, int32_t n_entries,
                                  int32_t n_long, int32_t n_bins, int32_t precision, int32_t out_kind, float eps,
                                  float* out, void* workspace, size_t workspace_bytes, void* stream);
/* pinned host (B, L) -> pinned host (B, n_bins, T); scratch: nnab_cqt1992v2_host_scratch_bytes(precision) */
int nnab_cqt1992v2_hybrid_forward_host(const nnab_frames* f, const float* x_host, const float* eg_bank,
                                       const float* eg_bank_lo, const uint16_t* col_table, const int32_t* group_rows,
                                       int32_t n_groups, int32_t r_max, const float* sched_bank,
                                       const float* sched_bank_lo, const uint32_t* schedule, int32_t n_entries,
                                       int32_t n_long, int32_t n_bins, int32_t precision, int32_t out_kind,
                                       float eps, float* out_host, int64_t chunk_clips, void* device_scratch,
                                       size_t scratch_bytes, void* stream);

/* Host-buffer end-to-end variant of nnab_cqt1992v2_forward (pinned x_host ->
 * pinned out_host, chunks of clips streamed through the device with H2D /
 * compute / D2H overlap); device buffers come from `device_scratch`. */
size_t nnab_cqt1992v2_host_scratch_bytes(const nnab_frames* f, int32_t precision, int32_t n_bins, int32_t out_kind,
                                         int64_t chunk_clips);
int nnab_cqt1992v2_forward_host(const nnab_frames* f, const float* x_host, const float* packed_hi,
                                const float* packed_lo, int32_t n_bins, const uint32_t* schedule, int32_t n_entries,
                                int32_t precision, int32_t out_kind, float eps, float* out_host, int64_t chunk_clips,
                                void* device_scratch, size_t scratch_bytes, void* stream);

/* ------------------------------------------------------- CQT2010v2
 * Cqt2010v2.__call__ (transforms.py:290-313, 319-323): early_stages x
 * downsample2 (signal.py:232-247), then per octave alpha: downsample2 (alpha>0)
 * and the centred complex conv with the top-octave bank (n_filters, width) at
 * hop kernel_hop >> alpha; rows scattered to first_bin + j - alpha*bins_per_octave.
 * taps: the (odd, symmetric) anti-alias FIR, HOST float32 (n_taps values).
 * out (B, n_bins, T) with T = the shortest octave's frame count (returned).
 * precision NNAB_PREC_TF32: the fused tensor-core chain (half-band FIR as a
 * TMEM-resident Toeplitz MMA, the whole clip in shared memory) when the clip
 * fits; NNAB_PREC_3XTF32 (and configurations outside that envelope): FP32
 * CUDA-core stage kernels. */
size_t nnab_cqt2010v2_workspace_bytes(int64_t B, int64_t L, int32_t early_stages);
int nnab_cqt2010v2_forward(const float* x, int64_t B, int64_t L, const float* taps, int32_t n_taps,
                           const float* k_re, const float* k_im, int32_t n_filters, int32_t width,
                           int32_t early_stages, int32_t n_octaves, int32_t kernel_hop, int32_t first_bin,
                           int32_t bins_per_octave, int32_t n_bins, int32_t pad_mode, int32_t out_kind,
                           int32_t precision, float* out, int32_t* n_frames_out, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Host-buffer end-to-end variant of nnab_cqt2010v2_forward (same pipeline as
 * nnab_stft_forward_host); T = the frame count nnab_cqt2010v2_forward reports. */
size_t nnab_cqt2010v2_host_scratch_bytes(int64_t L, int32_t early_stages, int32_t n_bins, int32_t T, int32_t out_kind,
                                         int64_t chunk_clips);
int nnab_cqt2010v2_forward_host(const float* x_host, int64_t B, int64_t L, const float* taps, int32_t n_taps,
                                const float* k_re, const float* k_im, int32_t n_filters, int32_t width,
                                int32_t early_stages, int32_t n_octaves, int32_t kernel_hop, int32_t first_bin,
                                int32_t bins_per_octave, int32_t n_bins, int32_t pad_mode, int32_t out_kind,
                                int32_t precision, float* out_host, int64_t chunk_clips, void* device_scratch,
                                size_t scratch_bytes, void* stream);

/* ------------------------------------------------------- file formats (csrc/io.cu)
 * WAV ingestion (wavio.py:19-68): the data chunk's bytes on the device ->
 * mono float32 (PCM16 / 32768, channel mean); equals float32(reference).
 * format 1 = PCM 16-bit, 3 = IEEE float 32-bit. */
int nnab_decode_wav(const void* payload, int64_t n_frames, int32_t channels, int32_t format, float* out,
                    void* stream);
/* SpecFile payload (specfile.py:26-43): float32 cells -> float64 on the device. */
int nnab_widen_f64(const float* src, int64_t n, double* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NNAB_H */
