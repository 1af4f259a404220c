// Host-side internals shared by the libnnab translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "../../include/nnab.h"

namespace nnab {

// Record a CUDA error for nnab_last_error() and map it to NNAB_ECUDA.
int cuda_fail(cudaError_t e, const char* where);
#define NNAB_CUDA_TRY(expr)                              \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
  } while (0)

// Count every libnnab kernel launch (nnab_launch_count) and check it.
void note_launch();
#define NNAB_LAUNCHED()                    \
  do {                                     \
    note_launch();                         \
    NNAB_CUDA_TRY(cudaGetLastError());     \
  } while (0)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
int make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                 uint32_t box_inner, uint32_t box_outer, int swizzle_bytes, int elem_bytes = 4);

int num_sms();

// Staging layout for frames: see frames.cu.
struct FrameGeom {
  int64_t B, L;
  int32_t width, hop, pad, pad_mode;
  int32_t T;         // frames per clip
  int32_t k_pad;     // width rounded up to 32
  int32_t row_len;   // TMA row (hop in hop-row mode, k_pad in framed mode)
  int32_t R;         // staged rows per clip
  int64_t padded_len;
};
// kalign: K-block alignment of the staged rows in elements (32 for the fp32 /
// TF32 operand modes, 64 for FP16: one 128-byte swizzle row)
int frame_geometry(const nnab_frames* f, FrameGeom* g, int kalign = 32);

inline bool prec_is_f16(int p) { return p == NNAB_PREC_F16 || p == NNAB_PREC_3XF16; }
inline bool prec_is_split(int p) { return p == NNAB_PREC_3XTF32 || p == NNAB_PREC_3XF16; }
inline int prec_kalign(int p) { return prec_is_f16(p) ? 64 : 32; }
inline bool prec_valid(int p) { return p >= NNAB_PREC_TF32 && p <= NNAB_PREC_3XF16; }

int stage_frames(const FrameGeom& g, const float* x, float* rows_hi, float* rows_lo, int split,
                 cudaStream_t s);
// atomicMax of |a|, |b| over n elements into *out as ordered float bits (the FP16 bank
// packers' peak; *out zeroed by the caller) (frames.cu)
int launch_bank_absmax(const float* a, const float* b, int64_t n, unsigned int* out, cudaStream_t s);
// FP16 hop rows scaled per clip by 2^exps[b] (frames.cu)
int stage_frames_f16(const FrameGeom& g, const float* x, void* rows_hi, void* rows_lo, int32_t* exps, int split,
                     cudaStream_t s);

struct StftGemmArgs {
  const float* a_hi;  // staged rows (B*R, row_len) -- fp32, or FP16 in the F16 modes
  const float* a_lo;
  const float* b_hi;  // packed bank (n_tiles*256, k_pad)
  const float* b_lo;
  const int32_t* a_exp = nullptr;  // F16 modes: per-clip scale exponent of the staged rows
  const int32_t* b_exp = nullptr;  // F16 modes: the bank's scale exponent (pack trailer)
  int32_t n_tiles;
  int32_t n_bins;
  int32_t fold;
  int32_t out_kind;
  float power;
  float eps;
  const float* mel_w;
  int32_t n_mels, mel_ld;
  const int32_t* mel_band;
  float* out;
  const uint32_t* kb_tab = nullptr;  // CQT long-bank schedule (device), see stft_gemm.cu
  int32_t n_tab = 0;
  int32_t b_box = 256;
  int32_t pairs = 0;
  int32_t out_bins = 0;  // pairs mode: bins per clip of the output (0 = n_bins; the caller offsets out)
  float *save_re = nullptr, *save_im = nullptr, *save_mag = nullptr;  // training forward (slot-major)
  float* save_mag_lo = nullptr;  // NNAB_SAVE_MAG_SPLIT: save_mag TF32 hi, this the lo residual
  int64_t ld_slots = 0;
  int32_t save_phasor = 0;  // saves in the TF32-backward format whatever the forward's operand mode
};

// Pointers into a staged-frames workspace of `precision` (capi.cu): rows hi / lo,
// per-clip exponents (FP16 modes), and the geometry with the precision's K alignment.
int staged_views(const nnab_frames* f, int32_t precision, const void* workspace, size_t workspace_bytes,
                 FrameGeom* g, const void** hi, const void** lo, const int32_t** exps);
int launch_stft_gemm(const FrameGeom& g, const StftGemmArgs& a, int precision, cudaStream_t s);
// cosine (= sine) rows per DFT-layout bank tile (frames.cu): 128, or fewer for a one-tile bank
int dft_half(int32_t n_bins, int32_t fold_nyquist);

// Reduction GEMM C[M][N] = sum_k A[M][K] B(K, N)  (rgemm.cu)
struct RGemmArgs {
  int32_t M = 0, N = 0;
  int64_t K = 0;                            // multiple of 32 (16 in 3xTF32)
  const float *a_hi = nullptr, *a_lo = nullptr;
  int64_t lda = 0;                          // floats
  const float *b_hi = nullptr, *b_lo = nullptr;
  int64_t ldb = 0;                          // K-major B: floats per row n
  int32_t b_mn = 0;                         // 1: (k, n) at rows[k + n / b_row_len][n % b_row_len]
  int32_t b_row_len = 0;
  int64_t b_rows = 0;
  float* c = nullptr;
  int64_t ldc = 0;
  int32_t splits = 0;                       // 0 = auto
  float* partial = nullptr;                 // split-K scratch (rgemm_partial_bytes)
  float alpha = 1.f;
  // coef epilogue (dS GEMM of the joint mel + STFT layer): instead of C = dS,
  // write coef rows f: dS*re/S and f + M: dS*im/S (tf32 hi [/lo]) at
  // coef[(f or f+M) * ldc + slot]; re/im are [M][ldc] (gradients.py:127-128)
  const float *coef_re = nullptr, *coef_im = nullptr;
  float* coef_lo = nullptr;
  float coef_eps = 0.f;
  // frames output (mel forward of the training layer): column n = slot b*R + t is
  // written to c[(b*M + m)*T + t] for t < T (the (B, M, T) layout), nothing else
  int64_t frames_B = 0;
  int32_t frames_R = 0, frames_T = 0;
  // 3xF16 kernel gradient (precision NNAB_PREC_3XF16): a_hi/a_lo and b_hi/b_lo are FP16
  // (lda in halves, B the MN-major staged hop rows); C rows are scaled by 2^-row_exp[m]
  const int32_t* row_exp = nullptr;
  // coef epilogue in FP16 (3xTF32 coef GEMM, coef_f16 = 1): c / coef_lo are FP16 hi/lo of
  // coef * 2^(row_exp[row] - clip_exp[slot / clip_R]) (0 past n_clips); ldc in halves
  const int32_t* clip_exp = nullptr;
  int64_t n_clips = 0;
  int32_t clip_R = 0, coef_f16 = 0;
};
size_t rgemm_partial_bytes(int32_t M, int32_t N, int64_t K, int32_t splits);
// fused tensor-core CQT2010v2 (cqt2010_tc.cu); NNAB_ENOTSUP outside its envelope
int launch_cqt2010_tc(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, const float* k_re,
                      const float* k_im, int n_filt, int width, int early_stages, int n_oct, int kernel_hop,
                      int first_bin, int bpo, int n_bins, int pad_mode, int out_kind, int T, float* out,
                      cudaStream_t st);
int launch_rgemm(const RGemmArgs& g, int precision, cudaStream_t s);
// CQT2010v2 batched path (cqt2010_tc.cu): the fused kernel as a per-clip front (stages
// 1-2), then per octave a CONV and a HALVE launch over all clips through level buffers
// in `workspace` (cqt2010_levels_bytes); NNAB_ENOTSUP outside the envelope / without room
size_t cqt2010_levels_bytes(int64_t B, int64_t L, const float* taps, int n_taps, int n_filt, int width,
                            int early_stages, int n_oct, int kernel_hop, int T, int pad_mode);
int launch_cqt2010_levels(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, const float* k_re,
                          const float* k_im, int n_filt, int width, int early_stages, int n_oct, int kernel_hop,
                          int first_bin, int bpo, int n_bins, int pad_mode, int out_kind, int T, float* out,
                          void* workspace, size_t workspace_bytes, cudaStream_t st, int mode);
// CQT2010v2 front (cqt2010_front.cu): stages 1-2 of every clip -> the octave-0 level buffer
// (FP16 in the clip's scale 2^-exps[b], reflect margins); NNAB_ENOTSUP outside its envelope
// the conv-bank images the back end reads (cqt2010_prep_kernel's work), written by the front
// launch instead of a launch of their own
struct CqtPrepArgs {
  uint4 *toep_img = nullptr, *filt_img = nullptr;
  const float *k_re = nullptr, *k_im = nullptr;
  int n_filt = 0, width = 0, shift = 0, nconv = 0, kc = 0, filt_log2 = 0;
};
int launch_cqt2010_front(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, __half* lv0,
                         int32_t lv0_stride, int32_t* exps, int32_t* flags, int32_t* list, int32_t* list_n,
                         cudaStream_t st, const CqtPrepArgs* prep = nullptr);
// CQT2010v2 back end (cqt2010_back.cu): the octave chain and every octave's conv of clip
// groups in one launch (level 0 written by the front, the conv bank image by the prep kernel)
struct CqtBackArgs {
  int n_oct;
  int64_t B;
  const float* taps;
  int n_taps;
  __half* lv[12];
  int32_t n[12], stride[12], h[12], copies[12], U[12], rs[12];
  int pad_al, T, n_bins, first_bin, bpo, n_filt, out_kind;
  const int32_t* exps;
  const uint4* filt_img;
  float* out;
};
int launch_cqt2010_back(const CqtBackArgs& g, cudaStream_t st);
// CQT2010v2 octave chain (cqt2010_chain.cu): halvings of levels 0 -> n_oct - 1 for all clips
// (level 0 written), with margins and the conv's shifted copies; NNAB_ENOTSUP outside it
int launch_cqt2010_chain(int64_t B, int n_oct, __half* const* lv, const int32_t* stride, const int32_t* n,
                         const int32_t* h, const int32_t* copies, const float* taps, int n_taps, cudaStream_t st);

}  // namespace nnab
