// CQT1992v2: the long complex time-domain bank (kernels.py:361-402) applied by
// centred strided correlation (transforms.py:175-186, 201-208).
//
// The bank is 84 complex rows of width even(N_0) = 22,682 at the default
// config, but row k is non-zero only on its centred support of N_k samples
// (N_83 = 188).  The same tcgen05 GEMM as the STFT runs it, with:
//  * re/im rows of each bin interleaved (2j, 2j+1) and bins ordered longest
//    first, so the rows active in any 32-sample K block form a prefix;
//  * a per-K-block schedule (kblock, N = rows of that prefix rounded to 16)
//    so each MMA only spans the active rows -- 4.5x fewer MMA cycles than
//    the dense bank -- processed longest-first so the first MMA of a tile
//    initialises every accumulator column.
#include <cuda_fp16.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {

__global__ void pack_cqt_bank_kernel(const float* __restrict__ k_re, const float* __restrict__ k_im, int32_t n_bins,
                                     int32_t width, int32_t k_pad, int32_t n_tiles, int32_t split,
                                     float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = (int64_t)n_tiles * 256 * k_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / k_pad;
    const int32_t k = (int32_t)(e - row * k_pad);
    const int32_t tile = (int32_t)(row / 256), col = (int32_t)(row % 256);
    const int32_t bin = tile * 128 + col / 2;
    float v = 0.f;
    if (k < width && bin < n_bins) v = ((col & 1) ? k_im : k_re)[(int64_t)bin * width + k];
    const float h = tf32_rne(v);
    hi[e] = h;
    if (split) lo[e] = tf32_rne(v - h);
  }
}

// FP16 schedule bank: the same layout in halves (K padded to 64) scaled by 2^e_h
// (trailer[1], from the bank peak in trailer[0], launch_bank_absmax)
__global__ void pack_cqt_bank_f16_kernel(const float* __restrict__ k_re, const float* __restrict__ k_im,
                                         int32_t n_bins, int32_t width, int32_t k_pad, int32_t n_tiles, int32_t split,
                                         __half* __restrict__ hi, __half* __restrict__ lo,
                                         int32_t* __restrict__ trailer) {
  const float pk = __uint_as_float(static_cast<unsigned int>(trailer[0]));
  int ex = 0;
  if (pk > 0.f && pk < INFINITY) frexpf(pk, &ex);
  const int e = pk > 0.f ? max(-100, min(100, 15 - ex)) : 0;
  const float sc = ldexpf(1.f, e);
  if (blockIdx.x == 0 && threadIdx.x == 0) trailer[1] = e;
  const int64_t total = (int64_t)n_tiles * 256 * k_pad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / k_pad;
    const int32_t k = (int32_t)(i - row * k_pad);
    const int32_t tile = (int32_t)(row / 256), col = (int32_t)(row % 256);
    const int32_t bin = tile * 128 + col / 2;
    float v = 0.f;
    if (k < width && bin < n_bins) v = ((col & 1) ? k_im : k_re)[(int64_t)bin * width + k];
    v *= sc;
    const __half h = __float2half_rn(v);
    hi[i] = h;
    if (split) lo[i] = __float2half_rn(v - __half2float(h));
  }
}

}  // namespace nnab

using namespace nnab;

extern "C" int nnab_cqt_bank_tiles(int32_t n_bins) { return std::max(1, (n_bins + 127) / 128); }

extern "C" size_t nnab_cqt_bank_bytes_prec(int32_t n_bins, int32_t width, int32_t precision) {
  if (!prec_is_f16(precision)) return nnab_cqt_bank_bytes(n_bins, width);
  const int64_t k_pad = (width + 63) / 64 * 64;
  const size_t data = (size_t)nnab_cqt_bank_tiles(n_bins) * 256 * k_pad * 2;
  return ((data + 255) & ~size_t(255)) + 256;  // + trailer: [0] peak bits, [1] scale exponent
}

extern "C" size_t nnab_cqt_bank_bytes(int32_t n_bins, int32_t width) {
  const int64_t k_pad = (width + 31) / 32 * 32;
  return (size_t)nnab_cqt_bank_tiles(n_bins) * 256 * k_pad * sizeof(float);
}

extern "C" int nnab_pack_cqt_bank(const float* k_re, const float* k_im, int32_t n_bins, int32_t width,
                                  int32_t precision, float* packed_hi, float* packed_lo, void* stream) {
  if (!k_re || !k_im || !packed_hi || n_bins < 1 || width < 1) return NNAB_EINVAL;
  if (!prec_valid(precision)) return NNAB_EINVAL;
  const int split = prec_is_split(precision);
  if (split && !packed_lo) return NNAB_EINVAL;
  if (prec_is_f16(precision)) {
    cudaStream_t s = (cudaStream_t)stream;
    const int32_t k_pad = (width + 63) / 64 * 64;
    const int32_t tiles = nnab_cqt_bank_tiles(n_bins);
    const int64_t total = (int64_t)tiles * 256 * k_pad;
    int32_t* trailer = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(packed_hi) +
                                                  nnab_cqt_bank_bytes_prec(n_bins, width, precision) - 256);
    NNAB_CUDA_TRY(cudaMemsetAsync(trailer, 0, 8, s));
    int rc = launch_bank_absmax(k_re, k_im, (int64_t)n_bins * width, reinterpret_cast<unsigned int*>(trailer), s);
    if (rc) return rc;
    pack_cqt_bank_f16_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 8192), 256, 0, s>>>(
        k_re, k_im, n_bins, width, k_pad, tiles, split, reinterpret_cast<__half*>(packed_hi),
        reinterpret_cast<__half*>(packed_lo), trailer);
    NNAB_LAUNCHED();
    return NNAB_OK;
  }
  const int32_t k_pad = (width + 31) / 32 * 32;
  const int32_t tiles = nnab_cqt_bank_tiles(n_bins);
  const int64_t total = (int64_t)tiles * 256 * k_pad;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8192);
  pack_cqt_bank_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(k_re, k_im, n_bins, width, k_pad, tiles, split,
                                                                 packed_hi, packed_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

// Host-side schedule.  support[2*bin] = first non-zero column, support[2*bin+1]
// = one past the last (an all-zero row has begin >= end).  Writes, per tile,
// entries (kblock << 16 | N) sorted by N descending into table_host
// (capacity n_tiles * ceil(k_pad / block)) and the per-tile entry count into
// *n_entries (multi-tile banks must have equal counts per tile).
extern "C" int nnab_cqt_schedule(const int32_t* support, int32_t n_bins, int32_t width, int32_t precision,
                                 uint32_t* table_host, int32_t* n_entries) {
  if (!support || !table_host || !n_entries || n_bins < 1 || width < 1) return NNAB_EINVAL;
  if (!prec_valid(precision)) return NNAB_EINVAL;
  // K-block elements of the GEMM's stage rows: TF32 32 (3xTF32 16), FP16 64 (3xF16 32)
  const int bk = (prec_is_f16(precision) ? 64 : 32) / (prec_is_split(precision) ? 2 : 1);
  const int32_t k_pad = (width + prec_kalign(precision) - 1) / prec_kalign(precision) * prec_kalign(precision);
  const int nkb = k_pad / bk;
  const int tiles = nnab_cqt_bank_tiles(n_bins);
  std::vector<std::vector<uint32_t>> per_tile(tiles);
  size_t longest = 0;
  for (int t = 0; t < tiles; ++t) {
    const int b0 = t * 128, b1 = std::min(n_bins, b0 + 128);
    std::vector<std::pair<int, int>> e;  // (N, kb)
    int max_rows = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      const int k0 = kb * bk, k1 = k0 + bk;
      int active = 0;  // 1 + highest bin (within tile) touching [k0, k1)
      for (int b = b0; b < b1; ++b)
        if (support[2 * b] < support[2 * b + 1] && support[2 * b] < k1 && support[2 * b + 1] > k0) active = b - b0 + 1;
      if (active == 0) continue;
      const int n = std::min(256, (2 * active + 15) / 16 * 16);
      max_rows = std::max(max_rows, n);
      e.push_back({n, kb});
    }
    if (e.empty()) e.push_back({16, 0});  // all-zero tile: one MMA to zero the accumulator
    std::stable_sort(e.begin(), e.end(), [](auto& a, auto& b) { return a.first > b.first; });
    // the first MMA must cover every column the epilogue reads
    e[0].first = std::max(e[0].first, std::min(256, (2 * (b1 - b0) + 15) / 16 * 16));
    for (auto& x : e) per_tile[t].push_back(((uint32_t)x.second << 16) | (uint32_t)x.first);
    longest = std::max(longest, per_tile[t].size());
  }
  for (int t = 0; t < tiles; ++t) {
    if (per_tile[t].size() != longest) return NNAB_ENOTSUP;  // multi-tile banks must share a schedule length
  }
  for (int t = 0; t < tiles; ++t)
    std::copy(per_tile[t].begin(), per_tile[t].end(), table_host + (size_t)t * longest);
  *n_entries = (int32_t)longest;
  return NNAB_OK;
}

extern "C" int nnab_cqt1992v2_forward(const nnab_frames* f, const float* x, const float* packed_hi,
                                      const float* packed_lo, int32_t n_bins, const uint32_t* schedule,
                                      int32_t n_entries, int32_t precision, int32_t out_kind, float eps, float* out,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  if (!x) return NNAB_EINVAL;
  int rc = nnab_stage_frames(f, x, precision, workspace, workspace_bytes, stream);
  if (rc) return rc;
  return nnab_cqt1992v2_forward_staged(f, packed_hi, packed_lo, n_bins, schedule, n_entries, precision, out_kind,
                                       eps, out, workspace, workspace_bytes, stream);
}

namespace nnab {
// The scheduled long-bank GEMM on staged frames; out_bins = bins per clip of
// the (possibly larger) output this bank's rows are written into.
int cqt_schedule_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo, int32_t n_bins,
                        const uint32_t* schedule, int32_t n_entries, int32_t precision, int32_t out_kind, float eps,
                        float* out, int32_t out_bins, const void* workspace, size_t workspace_bytes,
                        cudaStream_t s);
}  // namespace nnab

extern "C" int nnab_cqt1992v2_forward_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo,
                                             int32_t n_bins, const uint32_t* schedule, int32_t n_entries,
                                             int32_t precision, int32_t out_kind, float eps, float* out,
                                             const void* workspace, size_t workspace_bytes, void* stream) {
  return nnab::cqt_schedule_staged(f, packed_hi, packed_lo, n_bins, schedule, n_entries, precision, out_kind, eps,
                                   out, n_bins, workspace, workspace_bytes, (cudaStream_t)stream);
}

int nnab::cqt_schedule_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo, int32_t n_bins,
                              const uint32_t* schedule, int32_t n_entries, int32_t precision, int32_t out_kind,
                              float eps, float* out, int32_t out_bins, const void* workspace,
                              size_t workspace_bytes, cudaStream_t s) {
  if (!prec_valid(precision)) return NNAB_EINVAL;
  FrameGeom g;
  const void *rows_hi, *rows_lo;
  const int32_t* exps;
  int rc = staged_views(f, precision, workspace, workspace_bytes, &g, &rows_hi, &rows_lo, &exps);
  if (rc) return rc;
  const int split = prec_is_split(precision);
  if (!packed_hi || (split && !packed_lo) || !out || !schedule || n_entries < 1 || n_bins < 1)
    return NNAB_EINVAL;
  if (out_kind != NNAB_OUT_MAGNITUDE && out_kind != NNAB_OUT_POWER && out_kind != NNAB_OUT_COMPLEX &&
      out_kind != NNAB_OUT_SMOOTH_MAG)
    return NNAB_EINVAL;
  if (g.B == 0) return NNAB_OK;
  if (out_bins < n_bins) return NNAB_EINVAL;
  StftGemmArgs a{};
  a.a_hi = reinterpret_cast<const float*>(rows_hi);
  a.a_lo = reinterpret_cast<const float*>(rows_lo);
  a.a_exp = exps;
  if (prec_is_f16(precision))
    a.b_exp = reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(packed_hi) +
                                               nnab_cqt_bank_bytes_prec(n_bins, g.width, precision) - 256) + 1;
  a.b_hi = packed_hi;
  a.b_lo = packed_lo;
  a.n_tiles = nnab_cqt_bank_tiles(n_bins);
  a.n_bins = n_bins;
  a.fold = 0;
  a.out_kind = out_kind;
  a.power = 1.f;
  a.eps = eps;
  a.out = out;
  a.kb_tab = schedule;
  a.n_tab = n_entries;
  a.b_box = std::min(256, (2 * std::min(n_bins, 128) + 15) / 16 * 16);
  a.pairs = 1;
  a.out_bins = out_bins;
  return launch_stft_gemm(g, a, precision, s);
}
