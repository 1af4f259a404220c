// STFT / Mel forward: one persistent warp-specialised tcgen05 GEMM per call.
//
// Replaces the reference's per-clip DGEMM `frames @ kernels.T`
// (signal.py:181-182 via transforms.py:130-144) and the follow-on
// magnitude / power / complex finish (transforms.py:86-93) and Mel projection
// `weights @ |X|^power` (transforms.py:164-172), fused into the epilogue.
//
//   D[slot, col] = sum_k rows[slot + k/row_len, k%row_len] * bank[col, k]
//
// M = frame slots (128 per tile, spanning clips), N = 256 bank rows per tile
// (128 cosine + 128 sine rows of the same 128 bins, so magnitude needs no
// cross-CTA exchange), K = kernel width.  Operands arrive by TMA (128-byte
// swizzle, 32-sample K blocks; 64-byte swizzle + 16-sample blocks in 3xTF32
// mode where each stage carries hi and lo halves), accumulate in TMEM (two
// 256-column accumulators so the epilogue of tile n overlaps the MMAs of n+1),
// and the epilogue warps read TMEM with tcgen05.ld.
//
// Warp roles (256 threads, one CTA per SM):
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer (one elected lane)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: thread = accumulator row = one frame slot
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {

namespace {

constexpr int kBM = 128;
constexpr int kBN = 256;  // 128 bins x {cos, sin}
constexpr int kThreads = 256;
constexpr int kMelRows = 128;  // mel accumulator rows resident in smem

// kP: NNAB_PREC_* (TF32, 3xTF32, F16, 3xF16)
template <int kP, bool kPair>
struct Cfg {
  static constexpr bool kSplit = kP == NNAB_PREC_3XTF32 || kP == NNAB_PREC_3XF16;
  static constexpr bool kHalf = kP == NNAB_PREC_F16 || kP == NNAB_PREC_3XF16;
  static constexpr int ELEM = kHalf ? 2 : 4;              // operand bytes
  static constexpr int SWZ = kSplit ? 64 : 128;           // swizzle span = bytes of one K block row
  static constexpr int BK = SWZ / ELEM;                   // elements per K block (TF32 32|16, FP16 64|32)
  static constexpr int KSTEPS = SWZ / 32;                 // MMAs per K block (32 bytes of K each)
  static constexpr int A_BYTES = kBM * SWZ;               // 16 KB | 8 KB
  // a CTA pair splits the N = 256 bank rows: each CTA stages 128 of them
  static constexpr int B_BYTES = (kPair ? kBN / 2 : kBN) * SWZ;
  static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * (kSplit ? 2 : 1);  // 48 KB | 32 KB (pair)
  // unsplit: two 256-column accumulators (double buffer).  Split: one buffer of
  // main (hi*hi) + correction (hi*lo + lo*hi) accumulators.  Keeping the large
  // hi*hi chain apart from the small cross terms cuts the number of
  // accumulate steps the big partial sums go through by 3x, which is what
  // bounds the split modes' accuracy (the tensor-core FP32 accumulate is not RNE).
  static constexpr int NUM_ACC = kSplit ? 1 : 2;
  static constexpr int ACC_STRIDE = kSplit ? 512 : 256;
  static constexpr uint32_t idesc(uint32_t M, uint32_t N) { return kHalf ? idesc_f16(M, N) : idesc_tf32(M, N); }
};

NNAB_DEV void mma_any(bool half, bool pair, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (half) {
    if (pair) mma_f16_pair(d, a, b, idesc, acc);
    else mma_f16(d, a, b, idesc, acc);
  } else {
    if (pair) mma_tf32_pair(d, a, b, idesc, acc);
    else mma_tf32(d, a, b, idesc, acc);
  }
}

struct Params {
  int64_t B;
  int32_t T, R, row_len, kblocks, n_mtiles, n_tiles, n_bins, fold, out_kind;
  float power, eps;
  const float* mel_w;
  int32_t n_mels, mel_ld;
  const int32_t* mel_band;
  float* out;
  // CQT1992v2 long-bank schedule: per N tile, n_tab entries (kblock << 16 | N),
  // longest-first so the first MMA (N = max) initialises every used column.
  const uint32_t* kb_tab;
  int32_t n_tab, b_box, pairs, out_bins;
  int32_t half;  // DFT-layout tiles: cosine (= sine) rows per tile (dft_half)
  float log_eps;  // >= 0: outputs are log(value + log_eps) (NNAB_OUT_LOG)
  int32_t stages;  // smem pipeline depth (4, or 3 when the Mel accumulator takes 64 KB)
  // FP16 modes: epilogue scale 2^-(a_exp[clip] + *b_exp) undoes the operand scales (null: 1)
  const int32_t* a_exp;
  const int32_t* b_exp;
  // training forward: re, im and smoothed magnitude per (bin, slot) saved in
  // slot-major layout [bin][ld_slots] for the backward GEMMs (may be null)
  float *save_re, *save_im, *save_mag, *save_mag_lo;
  int64_t ld_slots;
  int32_t save_phasor;  // 1: save the TF32-backward format (FP16 unit phasor + TF32 |X|) in any operand mode
  int32_t stage_acc;    // kE8: stage the accumulators in shared memory and release TMEM before the processing
};

NNAB_DEV uint64_t make_sdesc(const void* p, int swz_bytes) {
  // K-major, rows of swz_bytes, 8-row atoms of 8*swz_bytes
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * swz_bytes) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(swz_bytes == 128 ? 2 : 4) << 61;
  return d;
}

// log compression of an output value (NNAB_OUT_LOG); log_eps < 0: off
NNAB_DEV float log_out(float v, float log_eps) { return log_eps >= 0.f ? logf(v + log_eps) : v; }

NNAB_DEV float finish(float re, float im, int kind, float power, float eps) {
  const float p = fmaf(re, re, im * im);
  if (kind == NNAB_OUT_POWER) return p;
  if (kind == NNAB_OUT_SMOOTH_MAG) return fast_sqrt(p + eps);
  if (kind == NNAB_OUT_MEL) {  // eps = 0 for MelSpec, 1e-12 for the trainable layer (gradients.py:69-74)
    if (power == 1.f) return fast_sqrt(p + eps);
    if (power == 2.f) return p + eps;
    return powf(fast_sqrt(p + eps), power);
  }
  return fast_sqrt(p);
}

// kE8 (split modes, non-Mel outputs): 8 epilogue warps, two per TMEM lane quarter on
// alternate 32-column chunks.  The split modes have one accumulator buffer, so the
// MMAs of tile n + 1 wait for tile n's epilogue; halving its time raises the tensor
// pipe's active share.
template <int kP, bool kPair, bool kE8 = false>
__global__ void __launch_bounds__(kE8 ? kThreads + 128 : kThreads, 1)
    stft_gemm_kernel(const __grid_constant__ CUtensorMap tm_a_hi, const __grid_constant__ CUtensorMap tm_a_lo,
                     const __grid_constant__ CUtensorMap tm_b_hi, const __grid_constant__ CUtensorMap tm_b_lo,
                     const Params p) {
  using C = Cfg<kP, kPair>;
  constexpr bool kSplit = C::kSplit;
  const bool mel = p.out_kind == NNAB_OUT_MEL;
  const int stages = p.stages;
  const uint32_t rank = kPair ? cluster_ctarank() : 0;  // 0 = leader (issues the pair's MMAs)

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* mel_acc = reinterpret_cast<float*>(smem + stages * C::STAGE_BYTES);  // [kMelRows][kBM]
  // kE8 + stage_acc: the fp32 (re | im) staging tile [kBM][256] (16-byte chunks XOR-swizzled by row) in its place
  float* stage_acc = mel_acc;
  // kE8 + Mel + stage_acc: |X| staging [kBM][128] after the Mel accumulator, then the
  // folded Nyquist |X| per row
  float* mag_stage = mel_acc + kMelRows * kBM;
  float* nyq_stage = mag_stage + kBM * 128;
  const size_t extra = mel ? kMelRows * kBM * 4 + ((kE8 && p.stage_acc) ? kBM * 128 * 4 + kBM * 4 : 0)
                           : (kE8 && p.stage_acc) ? kBM * kBN * 4 : 0;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + stages * C::STAGE_BYTES + extra);
  uint64_t* full = bars;            // [stages]  (pair: only the leader's are used)
  uint64_t* empty = bars + 8;       // [stages]
  uint64_t* tmem_full = bars + 16;  // [2]
  uint64_t* tmem_empty = bars + 18; // [2]       (pair: the leader's counts both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_a_hi);
    tma_prefetch(&tm_b_hi);
    if (kSplit) {
      tma_prefetch(&tm_a_lo);
      tma_prefetch(&tm_b_lo);
    }
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], (kPair ? 2 : 1) * (kE8 ? 8 : 4));  // one arrive per epilogue warp (of both CTAs)
    }
    fence_barrier_init();
  }
  if (kPair) cluster_sync();  // the peer's TMA / arrives target the leader's barriers
  if (warp == 2) {
    if (kPair) tmem_alloc_pair<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  if (mel) {
    for (int i = threadIdx.x; i < kMelRows * kBM; i += blockDim.x) mel_acc[i] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // M-tile walk: one CTA per M tile, or one pair per two consecutive M tiles
  const int m_start = kPair ? (int)cluster_id_x() : (int)blockIdx.x;
  const int m_step = kPair ? (int)nclusters_x() : (int)gridDim.x;
  const int m_end = kPair ? (p.n_mtiles + 1) / 2 : p.n_mtiles;

  const int nt = p.n_tiles;
  const int n_iter = p.kb_tab ? p.n_tab : p.kblocks;
  const int b_rows = kPair ? p.b_box / 2 : p.b_box;  // bank rows this CTA stages per K block
  const uint32_t stage_tx = (uint32_t)(C::A_BYTES + b_rows * C::SWZ) * (kSplit ? 2 : 1) * (kPair ? 2 : 1);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      for (int mi = m_start; mi < m_end; mi += m_step) {
        const int mt = kPair ? 2 * mi + (int)rank : mi;
        for (int n = 0; n < nt; ++n) {
          for (int it = 0; it < n_iter; ++it) {
            const uint32_t e = p.kb_tab ? __ldg(p.kb_tab + n * p.n_tab + it) : 0u;
            const int kb = p.kb_tab ? (int)(e >> 16) : it;
            // pair: the peer stages bank rows [N/2, N) of this K block's MMA width N
            const int tile_rows = (p.pairs || p.kb_tab) ? kBN : 2 * p.half;  // DFT layout: 2 hb rows per tile
            const int b_row = n * tile_rows +
                              (kPair && rank ? (p.kb_tab ? (int)(e & 0xffffu) / 2 : tile_rows / 2) : 0);
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = smem + s * C::STAGE_BYTES;
            const int k = kb * C::BK;
            const int a_col = k % p.row_len;
            const int a_row = mt * kBM + k / p.row_len;
            if (kPair) {
              const uint32_t fb = mapa(&full[s], 0);
              if (rank == 0) mbar_expect_tx(&full[s], stage_tx);
              tma_load_2d_pair(st, &tm_a_hi, fb, a_col, a_row, keep);
              tma_load_2d_pair(st + C::A_BYTES, &tm_b_hi, fb, k, b_row, keep);
              if (kSplit) {
                tma_load_2d_pair(st + C::A_BYTES + C::B_BYTES, &tm_a_lo, fb, a_col, a_row, keep);
                tma_load_2d_pair(st + 2 * C::A_BYTES + C::B_BYTES, &tm_b_lo, fb, k, b_row, keep);
              }
            } else {
              mbar_expect_tx(&full[s], stage_tx);
              tma_load_2d_hint(st, &tm_a_hi, &full[s], a_col, a_row, keep);
              tma_load_2d_hint(st + C::A_BYTES, &tm_b_hi, &full[s], k, b_row, keep);
              if (kSplit) {
                tma_load_2d_hint(st + C::A_BYTES + C::B_BYTES, &tm_a_lo, &full[s], a_col, a_row, keep);
                tma_load_2d_hint(st + 2 * C::A_BYTES + C::B_BYTES, &tm_b_lo, &full[s], k, b_row, keep);
              }
            }
            if (++s == stages) { s = 0; ph ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (rank == 0 && elect_one()) {
      constexpr uint32_t kM = kPair ? 2 * kBM : kBM;
      const uint32_t idesc_full = C::idesc(kM, (p.pairs || p.kb_tab) ? kBN : 2 * p.half);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int mi = m_start; mi < m_end; mi += m_step) {
        for (int n = 0; n < nt; ++n) {
          mbar_wait(&tmem_empty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + acc * C::ACC_STRIDE;
          for (int kb = 0; kb < n_iter; ++kb) {
            uint32_t idesc = idesc_full;
            if (p.kb_tab) idesc = C::idesc(kM, __ldg(p.kb_tab + n * p.n_tab + kb) & 0xffffu);
            mbar_wait(&full[s], ph);
            tc_fence_after();
            uint8_t* st = smem + s * C::STAGE_BYTES;
            const uint64_t a_hi = make_sdesc(st, C::SWZ);
            const uint64_t b_hi = make_sdesc(st + C::A_BYTES, C::SWZ);
#pragma unroll
            for (int k = 0; k < C::KSTEPS; ++k) {
              const uint64_t off = (uint64_t)((k * 32) >> 4);  // 32 bytes along K per MMA
              const uint64_t a_lo = make_sdesc(st + C::A_BYTES + C::B_BYTES, C::SWZ);
              const uint64_t b_lo = make_sdesc(st + 2 * C::A_BYTES + C::B_BYTES, C::SWZ);
              mma_any(C::kHalf, kPair, d, a_hi + off, b_hi + off, idesc, (kb | k) != 0);
              if (kSplit) {
                mma_any(C::kHalf, kPair, d + kBN, a_hi + off, b_lo + off, idesc, (kb | k) != 0);
                mma_any(C::kHalf, kPair, d + kBN, a_lo + off, b_hi + off, idesc, 1);
              }
            }
            if (kPair) mma_commit_pair(&empty[s], 0x3);
            else mma_commit(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
          }
          if (kPair) mma_commit_pair(&tmem_full[acc], 0x3);
          else mma_commit(&tmem_full[acc]);
          if (++acc == C::NUM_ACC) { acc = 0; aph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = (warp - 4) & 3;  // TMEM lane quarter
    const int hsel = kE8 ? (int)((warp - 4) >> 2) : 0;
    // kE8: chunks hsel, hsel + 2; with a Mel output both warps of a lane quarter read every
    // chunk and each accumulates half of every chunk's Mel band rows (each (row, mel) sum
    // keeps the 4-warp order: deterministic, and no second accumulator)
    const int CSTEP = (kE8 && !mel) ? 2 : 1;
    const int c_first = (kE8 && !mel) ? hsel : 0;
    // DFT-layout tiles: hb cosine columns then hb sine columns (hb = 128, or the bin count
    // rounded up to 8 for a one-tile bank of <= 120 bins), nch 32-column chunks of each
    const int hb = p.half, nch = (p.half + 31) / 32;
    const uint32_t row = q * 32 + lane;
    const int kind = p.out_kind;
    const int F = p.n_bins;
    int acc = 0;
    uint32_t aph = 0;
    const uint32_t empty_addr0 = kPair ? mapa(&tmem_empty[0], 0) : smem_u32(&tmem_empty[0]);
    // |X| for the backward GEMMs: TF32 for a TF32 backward; fp32 in the split modes, or
    // (save_mag_lo) already split into the 3xTF32 operand pair
    auto save_mag = [&](int64_t o, float pw) {
      if (!kSplit || p.save_phasor) {
        p.save_mag[o] = tf32_rne(fast_sqrt(pw));
      } else {
        const float m = sqrtf(pw);
        if (p.save_mag_lo) {
          const float h = tf32_rne(m);
          p.save_mag[o] = h;
          p.save_mag_lo[o] = tf32_rne(m - h);
        } else {
          p.save_mag[o] = m;
        }
      }
    };
    auto release_acc = [&](int a) {  // one arrive per warp on the (leader's) tmem_empty
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(empty_addr0 + 8 * a);
    };
    for (int mi = m_start; mi < m_end; mi += m_step) {
      const int mt = kPair ? 2 * mi + (int)rank : mi;
      const int64_t g = (int64_t)mt * kBM + row;
      const int64_t b = g / p.R;
      const int t = (int)(g - b * p.R);
      const bool valid = b < p.B && t < p.T;
      float nyq_val = 0.f;
      // FP16 modes: undo the operand scales (exact powers of two)
      const float osc = (C::kHalf && p.a_exp) ? ldexpf(1.f, -(__ldg(p.a_exp + min(b, p.B - 1)) + __ldg(p.b_exp))) : 1.f;
      for (int n = 0; n < nt; ++n) {
        mbar_wait(&tmem_full[acc], aph);
        tc_fence_after();
        const uint32_t tb = tmem_base + ((q * 32) << 16) + acc * C::ACC_STRIDE;
        if (kE8 && mel && p.stage_acc) {
          // Mel with the magnitudes staged: the warp pair of a lane quarter turns its two
          // chunks into |X| in shared memory and frees TMEM, then each warp projects every
          // chunk onto its parity's Mel rows while the next tile's MMAs run
          float4* mrow = reinterpret_cast<float4*>(mag_stage) + row * 32;
          const int sw = (int)(row & 7);
          asm volatile("bar.sync %0, 64;" ::"r"(1 + (int)q) : "memory");  // the pair is done reading the staging
#pragma unroll 1
          for (int c = hsel; c < nch; c += 2) {
            float re[32], im[32], cre[32], cim[32];
            tmem_ld32(tb + c * 32, re);
            tmem_ld32(tb + hb + c * 32, im);
            tmem_ld32(tb + kBN + c * 32, cre);
            tmem_ld32(tb + kBN + hb + c * 32, cim);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              re[j] = (re[j] + cre[j]) * osc;
              im[j] = (im[j] + cim[j]) * osc;
            }
            if (p.fold && n == 0 && c == 0) {
              nyq_stage[row] = finish(im[0], 0.f, kind, p.power, p.eps);  // cosine row of bin F-1 in bin 0's sine slot
              im[0] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              mrow[(c * 8 + j) ^ sw] = make_float4(
                  finish(re[4 * j], im[4 * j], kind, p.power, p.eps), finish(re[4 * j + 1], im[4 * j + 1], kind, p.power, p.eps),
                  finish(re[4 * j + 2], im[4 * j + 2], kind, p.power, p.eps),
                  finish(re[4 * j + 3], im[4 * j + 3], kind, p.power, p.eps));
          }
          release_acc(acc);
          if (++acc == C::NUM_ACC) { acc = 0; aph ^= 1; }
          asm volatile("bar.sync %0, 64;" ::"r"(1 + (int)q) : "memory");  // both halves staged
          if (p.fold && n == 0) nyq_val = nyq_stage[row];
#pragma unroll 1
          for (int c = 0; c < nch; ++c) {
            float m32[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 v4 = mrow[(c * 8 + j) ^ sw];
              m32[4 * j] = v4.x, m32[4 * j + 1] = v4.y, m32[4 * j + 2] = v4.z, m32[4 * j + 3] = v4.w;
            }
            const int bin0 = n * hb + c * 32;
            const int ch = bin0 >> 5;
            const int lo = p.mel_band ? p.mel_band[2 * ch] : 0;
            const int hi = p.mel_band ? p.mel_band[2 * ch + 1] : p.n_mels;
            int m = lo + ((lo ^ hsel) & 1);
            for (; m + 2 < hi; m += 4) {
              const float4* w0 = reinterpret_cast<const float4*>(p.mel_w + (int64_t)m * p.mel_ld + bin0);
              const float4* w1 = reinterpret_cast<const float4*>(p.mel_w + (int64_t)(m + 2) * p.mel_ld + bin0);
              float4 wa[8], wb[8];
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                wa[j4] = __ldg(w0 + j4);
                wb[j4] = __ldg(w1 + j4);
              }
              float a = mel_acc[m * kBM + row], a2 = mel_acc[(m + 2) * kBM + row];
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                a = fmaf(wa[j4].x, m32[4 * j4 + 0], a);
                a2 = fmaf(wb[j4].x, m32[4 * j4 + 0], a2);
                a = fmaf(wa[j4].y, m32[4 * j4 + 1], a);
                a2 = fmaf(wb[j4].y, m32[4 * j4 + 1], a2);
                a = fmaf(wa[j4].z, m32[4 * j4 + 2], a);
                a2 = fmaf(wb[j4].z, m32[4 * j4 + 2], a2);
                a = fmaf(wa[j4].w, m32[4 * j4 + 3], a);
                a2 = fmaf(wb[j4].w, m32[4 * j4 + 3], a2);
              }
              mel_acc[m * kBM + row] = a;
              mel_acc[(m + 2) * kBM + row] = a2;
            }
            if (m < hi) {
              const float4* w = reinterpret_cast<const float4*>(p.mel_w + (int64_t)m * p.mel_ld + bin0);
              float a = mel_acc[m * kBM + row];
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 wv = __ldg(w + j4);
                a = fmaf(wv.x, m32[4 * j4 + 0], a);
                a = fmaf(wv.y, m32[4 * j4 + 1], a);
                a = fmaf(wv.z, m32[4 * j4 + 2], a);
                a = fmaf(wv.w, m32[4 * j4 + 3], a);
              }
              mel_acc[m * kBM + row] = a;
            }
          }
          continue;
        }
        if (p.pairs) {
          // columns (2j, 2j+1) = (re, im) of bin 128n + j; complex value re + i*im
          const int bins_here = min(128, F - n * 128);
          const int nc = (2 * bins_here + 31) / 32;
#pragma unroll 1
          for (int c = 0; c < nc; ++c) {
            float v[32];
            tmem_ld32(tb + c * 32, v);
            if (kSplit) {
              float cv[32];
              tmem_ld32(tb + kBN + c * 32, cv);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += cv[j];
            } else {
              tmem_ld_wait();
            }
            if (C::kHalf) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= osc;
            }
            if (valid) {
              const int bin0 = n * 128 + c * 16;
              const int64_t ob = b * (int64_t)p.out_bins;
              if (kind == NNAB_OUT_COMPLEX) {
                float2* o = reinterpret_cast<float2*>(p.out);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (bin0 + j < F) o[(ob + bin0 + j) * p.T + t] = make_float2(v[2 * j], v[2 * j + 1]);
              } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (bin0 + j < F) p.out[(ob + bin0 + j) * p.T + t] = finish(v[2 * j], v[2 * j + 1], kind, p.power, p.eps);
              }
            }
          }
          release_acc(acc);
          if (++acc == C::NUM_ACC) { acc = 0; aph ^= 1; }
          continue;
        }
        // kE8 + stage_acc: copy this warp's chunks (main + correction, scaled) to its rows of
        // the staging tile and release TMEM at once, so the next tile's MMAs overlap the
        // processing below (the split modes have one accumulator buffer)
        float4* srow = reinterpret_cast<float4*>(stage_acc) + row * 64;
        const int sw = (int)(row & 7);
        if (kE8 && p.stage_acc) {
#pragma unroll 1
          for (int c = c_first; c < nch; c += CSTEP) {
            float re[32], im[32], cre[32], cim[32];
            tmem_ld32(tb + c * 32, re);
            tmem_ld32(tb + hb + c * 32, im);
            tmem_ld32(tb + kBN + c * 32, cre);
            tmem_ld32(tb + kBN + hb + c * 32, cim);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              srow[(c * 8 + j) ^ sw] = make_float4((re[4 * j] + cre[4 * j]) * osc, (re[4 * j + 1] + cre[4 * j + 1]) * osc,
                                                   (re[4 * j + 2] + cre[4 * j + 2]) * osc,
                                                   (re[4 * j + 3] + cre[4 * j + 3]) * osc);
              srow[(32 + c * 8 + j) ^ sw] =
                  make_float4((im[4 * j] + cim[4 * j]) * osc, (im[4 * j + 1] + cim[4 * j + 1]) * osc,
                              (im[4 * j + 2] + cim[4 * j + 2]) * osc, (im[4 * j + 3] + cim[4 * j + 3]) * osc);
            }
          }
          release_acc(acc);
        }
#pragma unroll 1
        for (int c = c_first; c < nch; c += CSTEP) {
          float re[32], im[32];
          if (kE8 && p.stage_acc) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 a = srow[(c * 8 + j) ^ sw], b = srow[(32 + c * 8 + j) ^ sw];
              re[4 * j] = a.x, re[4 * j + 1] = a.y, re[4 * j + 2] = a.z, re[4 * j + 3] = a.w;
              im[4 * j] = b.x, im[4 * j + 1] = b.y, im[4 * j + 2] = b.z, im[4 * j + 3] = b.w;
            }
          } else {
          tmem_ld32(tb + c * 32, re);
          tmem_ld32(tb + hb + c * 32, im);
          if (kSplit) {
            float cre[32], cim[32];
            tmem_ld32(tb + kBN + c * 32, cre);
            tmem_ld32(tb + kBN + hb + c * 32, cim);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              re[j] += cre[j];
              im[j] += cim[j];
            }
          } else {
            tmem_ld_wait();
          }
          if (C::kHalf) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              re[j] *= osc;
              im[j] *= osc;
            }
          }
          }  // TMEM read
          const int bin0 = n * hb + c * 32;
          float nyq_re = 0.f;
          if (p.fold && n == 0 && c == 0) {
            nyq_re = im[0];  // cosine row of bin F-1 sits in bin 0's sine slot
            im[0] = 0.f;
          }
          if (p.save_re && (!kE8 || !mel || hsel == 0)) {  // slot-major copies for the backward (coalesced)
            const int64_t slot = (int64_t)mt * kBM + row;
            if (slot < p.ld_slots) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int bin = bin0 + j;
                if (bin < F - p.fold) {
                  const int64_t o = (int64_t)bin * p.ld_slots + slot;
                  const float pw = fmaf(re[j], re[j], im[j] * im[j]) + p.eps;
                  if (p.save_im && !p.save_phasor) {
                    p.save_re[o] = re[j];
                    p.save_im[o] = im[j];
                  } else {  // TF32 backward: the unit phasor (re/S, im/S) as packed FP16 (what coef needs)
                    const float inv = rsqrtf(pw);
                    const __half2 ph = __floats2half2_rn(re[j] * inv, im[j] * inv);
                    reinterpret_cast<__half2*>(p.save_re)[o] = ph;
                  }
                  if (p.save_mag)  // GEMM operand of dW: TF32-rounded for a TF32 backward, fp32 (split later) in 3xTF32
                    save_mag(o, pw);
                }
              }
              if (p.fold && n == 0 && c == 0) {
                const int64_t o = (int64_t)(F - 1) * p.ld_slots + slot;
                const float pw = nyq_re * nyq_re + p.eps;
                if (p.save_im && !p.save_phasor) {
                  p.save_re[o] = nyq_re;
                  p.save_im[o] = 0.f;
                } else {
                  reinterpret_cast<__half2*>(p.save_re)[o] = __floats2half2_rn(nyq_re * rsqrtf(pw), 0.f);
                }
                if (p.save_mag) save_mag(o, pw);
              }
            }
          }
          if (kind == NNAB_OUT_MEL) {
            float m32[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) m32[j] = finish(re[j], im[j], kind, p.power, p.eps);
            const int ch = bin0 >> 5;
            const int lo = p.mel_band ? p.mel_band[2 * ch] : 0;
            const int hi = p.mel_band ? p.mel_band[2 * ch + 1] : p.n_mels;
            // kE8: this warp owns the Mel rows of parity hsel (fixed per row, so every
            // (row, mel) sum is updated by one thread in chunk order)
            const int mst = kE8 ? 2 : 1;
            // two mel rows per step: independent FMA chains and all 16 weight
            // loads of both rows in flight before the first use
            int m = kE8 ? lo + ((lo ^ hsel) & 1) : lo;
            for (; m + mst < hi; m += 2 * mst) {
              const float4* w0 = reinterpret_cast<const float4*>(p.mel_w + (int64_t)m * p.mel_ld + bin0);
              const float4* w1 = reinterpret_cast<const float4*>(p.mel_w + (int64_t)(m + mst) * p.mel_ld + bin0);
              float4 wa[8], wb[8];
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                wa[j4] = __ldg(w0 + j4);
                wb[j4] = __ldg(w1 + j4);
              }
              float a = mel_acc[m * kBM + row], a2 = mel_acc[(m + mst) * kBM + row];
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                a = fmaf(wa[j4].x, m32[4 * j4 + 0], a);
                a2 = fmaf(wb[j4].x, m32[4 * j4 + 0], a2);
                a = fmaf(wa[j4].y, m32[4 * j4 + 1], a);
                a2 = fmaf(wb[j4].y, m32[4 * j4 + 1], a2);
                a = fmaf(wa[j4].z, m32[4 * j4 + 2], a);
                a2 = fmaf(wb[j4].z, m32[4 * j4 + 2], a2);
                a = fmaf(wa[j4].w, m32[4 * j4 + 3], a);
                a2 = fmaf(wb[j4].w, m32[4 * j4 + 3], a2);
              }
              mel_acc[m * kBM + row] = a;
              mel_acc[(m + mst) * kBM + row] = a2;
            }
            if (m < hi) {
              const float4* w = reinterpret_cast<const float4*>(p.mel_w + (int64_t)m * p.mel_ld + bin0);
              float a = mel_acc[m * kBM + row];
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 wv = __ldg(w + j4);
                a = fmaf(wv.x, m32[4 * j4 + 0], a);
                a = fmaf(wv.y, m32[4 * j4 + 1], a);
                a = fmaf(wv.z, m32[4 * j4 + 2], a);
                a = fmaf(wv.w, m32[4 * j4 + 3], a);
              }
              mel_acc[m * kBM + row] = a;
            }
            if (p.fold && n == 0 && c == 0) nyq_val = finish(nyq_re, 0.f, kind, p.power, p.eps);
          } else if (valid && p.out) {  // out == null: training forward that only saves slots
            const int64_t ob = b * (int64_t)F;
            if (kind == NNAB_OUT_COMPLEX) {
              float2* o = reinterpret_cast<float2*>(p.out);
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (bin0 + j < F - p.fold) o[(ob + bin0 + j) * p.T + t] = make_float2(re[j], -im[j]);
              if (p.fold && n == 0 && c == 0) o[(ob + F - 1) * p.T + t] = make_float2(nyq_re, 0.f);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (bin0 + j < F - p.fold)
                  p.out[(ob + bin0 + j) * p.T + t] = log_out(finish(re[j], im[j], kind, p.power, p.eps), p.log_eps);
              if (p.fold && n == 0 && c == 0)
                p.out[(ob + F - 1) * p.T + t] = log_out(finish(nyq_re, 0.f, kind, p.power, p.eps), p.log_eps);
            }
          }
        }
        if (!(kE8 && p.stage_acc)) release_acc(acc);
        if (++acc == C::NUM_ACC) { acc = 0; aph ^= 1; }
      }
      if (kind == NNAB_OUT_MEL) {
        if (p.fold) {  // Nyquist bin's mel contribution
          const int ch = (F - 1) >> 5;
          const int lo = p.mel_band ? p.mel_band[2 * ch] : 0;
          const int hi = p.mel_band ? p.mel_band[2 * ch + 1] : p.n_mels;
          for (int m = kE8 ? lo + ((lo ^ hsel) & 1) : lo; m < hi; m += kE8 ? 2 : 1)
            mel_acc[m * kBM + row] = fmaf(__ldg(p.mel_w + (int64_t)m * p.mel_ld + F - 1), nyq_val, mel_acc[m * kBM + row]);
        }
        if (kE8) {  // both halves of the band rows are in: the warp pair syncs on a named barrier
          asm volatile("bar.sync %0, 64;" ::"r"(1 + (int)q) : "memory");
        }
        for (int m = kE8 ? hsel : 0; m < p.n_mels; m += kE8 ? 2 : 1) {
          if (valid) p.out[(b * p.n_mels + m) * (int64_t)p.T + t] = log_out(mel_acc[m * kBM + row], p.log_eps);
          mel_acc[m * kBM + row] = 0.f;
        }
        if (kE8) asm volatile("bar.sync %0, 64;" ::"r"(1 + (int)q) : "memory");  // zeroed before the next tile's adds
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();  // the peer's TMEM is written by the leader's MMAs until the end
  tc_fence_after();
  if (warp == 2) {
    if (kPair) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

template <int kP, bool kPair, bool kE8 = false>
int launch_impl(const FrameGeom& g, const StftGemmArgs& a, cudaStream_t s) {
  using C = Cfg<kP, kPair>;
  constexpr bool kSplit = C::kSplit;
  const bool mel = (a.out_kind & ~NNAB_OUT_LOG) == NNAB_OUT_MEL;
  if (mel && (a.n_mels < 1 || a.n_mels > kMelRows || !a.mel_w || a.mel_ld % 4 != 0)) return NNAB_ENOTSUP;
  if (g.row_len % C::BK != 0 || g.k_pad % C::BK != 0) return NNAB_ENOTSUP;
  if (C::kHalf && (!a.a_exp || !a.b_exp)) return NNAB_EINVAL;
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  const uint64_t rows_total = (uint64_t)g.B * g.R;
  // DFT-layout banks: tiles of 2 hb rows (hb = dft_half: 128, or fewer for a one-tile bank)
  const int hb = (a.pairs || a.kb_tab) ? 128 : dft_half(a.n_bins, a.fold);
  const uint64_t bank_rows = (uint64_t)a.n_tiles * ((a.pairs || a.kb_tab) ? kBN : 2 * hb);
  const int b_box = a.b_box > 0 ? a.b_box : 2 * hb;
  if (b_box % 16 != 0 || b_box > kBN) return NNAB_EINVAL;
  const int b_rows = kPair ? b_box / 2 : b_box;  // each CTA of a pair stages half the bank rows
  constexpr int E = C::ELEM;
  int rc = make_tmap_2d(&ta_hi, a.a_hi, g.row_len, rows_total, (uint64_t)g.row_len * E, C::BK, kBM, C::SWZ, E);
  if (!rc) rc = make_tmap_2d(&tb_hi, a.b_hi, g.k_pad, bank_rows, (uint64_t)g.k_pad * E, C::BK, b_rows, C::SWZ, E);
  if (!rc && kSplit) rc = make_tmap_2d(&ta_lo, a.a_lo, g.row_len, rows_total, (uint64_t)g.row_len * E, C::BK, kBM, C::SWZ, E);
  if (!rc && kSplit) rc = make_tmap_2d(&tb_lo, a.b_lo, g.k_pad, bank_rows, (uint64_t)g.k_pad * E, C::BK, b_rows, C::SWZ, E);
  if (rc) return rc;
  if (!kSplit) {
    ta_lo = ta_hi;
    tb_lo = tb_hi;
  }
  Params p{};
  p.B = g.B;
  p.T = g.T;
  p.R = g.R;
  p.row_len = g.row_len;
  p.kblocks = g.k_pad / C::BK;
  p.n_mtiles = (int32_t)((rows_total + kBM - 1) / kBM);
  p.n_tiles = a.n_tiles;
  p.n_bins = a.n_bins;
  p.fold = a.fold;
  p.out_kind = a.out_kind & ~NNAB_OUT_LOG;
  p.log_eps = (a.out_kind & NNAB_OUT_LOG) ? a.eps : -1.f;
  p.power = a.power;
  p.eps = (a.out_kind & NNAB_OUT_LOG) ? 0.f : a.eps;
  p.mel_w = a.mel_w;
  p.n_mels = a.n_mels;
  p.mel_ld = a.mel_ld;
  p.mel_band = a.mel_band;
  p.out = a.out;
  p.kb_tab = a.kb_tab;
  p.save_re = a.save_re;
  p.save_im = a.save_im;
  p.save_mag = a.save_mag;
  p.save_mag_lo = a.save_mag_lo;
  p.ld_slots = a.ld_slots;
  p.a_exp = a.a_exp;
  p.b_exp = a.b_exp;
  if (a.save_re && a.pairs) return NNAB_EINVAL;
  p.save_phasor = a.save_phasor;
  if (a.save_re && !a.save_im && kSplit && !a.save_phasor) return NNAB_EINVAL;  // 3x modes save re / im
  p.n_tab = a.n_tab;
  p.b_box = b_box;
  p.half = hb;
  p.pairs = a.pairs;
  p.out_bins = a.out_bins > 0 ? a.out_bins : a.n_bins;
  if (a.kb_tab && (a.n_tab < 1 || mel)) return NNAB_EINVAL;
  if (kE8 && a.pairs) return NNAB_EINVAL;  // the pairs loop: 4 warps
  if (p.n_mtiles == 0) return NNAB_OK;
  // as many pipeline stages as fit next to the Mel accumulator (<= 8)
  static const bool stage_env = [] {
    const char* e = getenv("NNAB_STFT_STAGE_ACC");
    return !(e && e[0] == '0');
  }();
  // staging: the re | im tile, or (Mel, no slot saves) the |X| tile next to the Mel accumulator
  p.stage_acc = kE8 && kSplit && stage_env && !(mel && a.save_re);  // one buffer (split modes) only
  const size_t mel_bytes = mel ? (size_t)kMelRows * kBM * 4 + (p.stage_acc ? (size_t)kBM * 128 * 4 + kBM * 4 : 0)
                               : p.stage_acc ? (size_t)kBM * kBN * 4 : 0;
  constexpr size_t kBudget = 227 * 1024 - 1024 - 256;  // max dynamic smem - alignment slack - barriers
  int stages = (int)std::min<size_t>(8, (kBudget - mel_bytes) / C::STAGE_BYTES);
  if (const char* e = getenv("NNAB_DEBUG_STAGES")) stages = std::max(2, std::min(stages, atoi(e)));
  p.stages = stages;
  const size_t smem = 1024 + (size_t)stages * C::STAGE_BYTES + mel_bytes + 256;
  auto kern = stft_gemm_kernel<kP, kPair, kE8>;
  constexpr int threads = kE8 ? kThreads + 128 : kThreads;
  NNAB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (!kPair) {
    const int grid = std::min(p.n_mtiles, num_sms());
    kern<<<grid, threads, smem, s>>>(ta_hi, ta_lo, tb_hi, tb_lo, p);
  } else {
    const int pairs = (p.n_mtiles + 1) / 2;
    const int grid = 2 * std::min(pairs, num_sms() / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    NNAB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta_hi, ta_lo, tb_hi, tb_lo, p));
  }
  NNAB_LAUNCHED();
  return NNAB_OK;
}

}  // namespace

int launch_stft_gemm(const FrameGeom& g, const StftGemmArgs& a, int precision, cudaStream_t s) {
  // CTA pairs (cta_group::2, M = 256) by default; NNAB_CTA_PAIR=0 selects one CTA per M tile
  static const bool pair = [] {
    const char* e = getenv("NNAB_CTA_PAIR");
    return !(e && e[0] == '0');
  }();
  static const bool e8 = [] {  // NNAB_STFT_E8=0: 4 epilogue warps in the split modes too
    const char* e = getenv("NNAB_STFT_E8");
    return !(e && e[0] == '0');
  }();
  static const bool e8_f16 = [] {
    const char* e = getenv("NNAB_STFT_E8_F16");
    return e && e[0] == '1';
  }();
  switch (precision) {
    case NNAB_PREC_TF32: return pair ? launch_impl<NNAB_PREC_TF32, true>(g, a, s) : launch_impl<NNAB_PREC_TF32, false>(g, a, s);
    case NNAB_PREC_3XTF32: return pair ? launch_impl<NNAB_PREC_3XTF32, true>(g, a, s) : launch_impl<NNAB_PREC_3XTF32, false>(g, a, s);
    case NNAB_PREC_F16:
      // the fused Mel projection on 8 epilogue warps: opt-in (NNAB_STFT_E8_F16=1), measured neutral
      // (Mel 2.04-2.10 vs 2.09 ms, power 2 2.33-2.42 vs 2.40-2.42: the two accumulator buffers already
      // hide the 4-warp epilogue)
      if (pair && e8_f16 && (a.out_kind & ~NNAB_OUT_LOG) == NNAB_OUT_MEL && !a.pairs)
        return launch_impl<NNAB_PREC_F16, true, true>(g, a, s);
      return pair ? launch_impl<NNAB_PREC_F16, true>(g, a, s) : launch_impl<NNAB_PREC_F16, false>(g, a, s);
    case NNAB_PREC_3XF16:
      if (pair && e8 && !a.pairs)
        return launch_impl<NNAB_PREC_3XF16, true, true>(g, a, s);
      return pair ? launch_impl<NNAB_PREC_3XF16, true>(g, a, s) : launch_impl<NNAB_PREC_3XF16, false>(g, a, s);
    default: return NNAB_EINVAL;
  }
}

}  // namespace nnab
