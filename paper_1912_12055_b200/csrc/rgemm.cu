// Reduction GEMM for the backward pass (gradients.py:103-149):
//
//   C[m, n] = sum_k A[m, k] * B(k, n)        (fp32 out, TF32 or 3xTF32 in)
//
// A is K-major in global memory (row m, k contiguous).  B is either K-major
// (row n, k contiguous) or MN-major, where element (k, n) lives at
// rows[k + n / b_row_len][n % b_row_len] -- with b_row_len = hop that is the
// staged hop-row frame layout, so the kernel-gradient GEMM
// dK = coef @ frames (gradients.py:127-129) reads frames straight from the
// forward's staging buffer (never materialised).  The reduction runs over
// all frame slots of the batch (277,890 at the default config); output tiles
// of 128 x 256 are spread over persistent CTAs, optionally split along K into
// `splits` deterministic partial tiles (summed in a fixed order afterwards).
//
// Warp roles as in stft_gemm.cu: TMA producer, MMA issuer, TMEM allocator,
// 4 epilogue warps (thread = output row).
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

// Split-K count for a reduction with `units` CTAs per split: the smallest count whose work
// units fill whole waves of the persistent grid to >= 90 % (a TF32 CQT kernel gradient has 90
// CTAs per split: 3 splits -> 1.82 of 2 waves instead of 0.61 of 1; its 3xTF32 form 178: 3 ->
// 3.6 of 4 instead of 1.2 of 2).
int auto_splits(int64_t units, int64_t kb) {
  const int n = num_sms();
  int best = 1;
  double best_e = 0.;
  for (int s = 1; s <= 16 && s <= kb; ++s) {
    const double w = (double)units * s / n, e = w / std::ceil(w);
    if (w >= 0.9 && e >= 0.9) return s;
    if (w >= 0.9 && e > best_e) { best_e = e; best = s; }
  }
  return best_e > 0. ? best : std::max(1, (int)std::min<int64_t>(kb, n / std::max<int64_t>(1, units)));
}

constexpr int kBM = 128, kBN = 256, kThreads = 256, kStages = 4;

// 3xF16 TMEM accumulation chunk (K per chain before the FP32 drain into C); NNAB_RGEMM_F16_CHUNK
int f16_chunk() {
  static const int c = [] {
    const char* e = getenv("NNAB_RGEMM_F16_CHUNK");
    const int v = e ? atoi(e) : 2048;
    return v >= 64 && v % 64 == 0 ? v : 2048;
  }();
  return c;
}
constexpr int kStg = 36;  // epilogue transpose row stride (floats)
// 3xF16 epilogue: per warp two 32 x 32 fp32 staging tiles (128-byte swizzle) that TMA
// stores / reduce-adds into C
constexpr int kF16Stg = 4 * 2 * 4096;

// kF16 (CTA pairs only): FP16 operands, 64 K per stage; with kSplit (3xF16) a stage holds
// A hi | A lo | this CTA's half of B hi | of B lo, without (one FP16 pass) A | B half.
template <bool kSplit, bool kF16 = false>
struct RCfg {
  static constexpr int BK = kF16 ? 64 : kSplit ? 16 : 32;
  static constexpr int EB = kF16 ? 2 : 4;  // element bytes
  static constexpr int SWZ = BK * EB;
  static constexpr int A_BYTES = kBM * BK * EB;
  static constexpr int B_BYTES = kBN * BK * EB;
  static constexpr int STAGE = kF16 ? (kSplit ? 2 : 1) * (A_BYTES + B_BYTES / 2) : (A_BYTES + B_BYTES) * (kSplit ? 2 : 1);
  // pipeline stages: 3 of 64 KB (3xF16), 6 of 32 KB (FP16) next to the drain staging
  static constexpr int NST_F16 = kSplit ? 3 : 6;
  static constexpr int NUM_ACC = kSplit ? 1 : 2;
  static constexpr int ACC_STRIDE = kSplit ? 512 : 256;
};

struct RParams {
  int32_t M, N;
  int64_t K;
  int32_t m_tiles, n_tiles, splits;
  int64_t k_per_split;  // multiple of BK
  int64_t k_chunk;      // TMEM accumulation chunk (multiple of BK); chunks are summed in fp32 in C
  int32_t b_mn, b_row_len;
  float* C;             // [splits][M][ldc]
  int64_t ldc, split_stride;
  const float *re, *im;  // coef epilogue (RGemmArgs::coef_re): C is coef_hi; im null: re holds FP16 phasor pairs
  float* c_lo;
  float eps;
  int64_t fB;  // frames output (RGemmArgs::frames_R > 0)
  int32_t fR, fT;
  const int32_t* row_exp;   // RGemmArgs::row_exp
  const int32_t* clip_exp;  // RGemmArgs::clip_exp (coef_f16)
  int64_t n_clips;
  int32_t clip_R, coef_f16;
  int32_t c_split_rows;  // kF16: rows of C (its tensor map) per split (0: C is the output)
};

NNAB_DEV float4 tf32_hi4(float4 a) { return make_float4(tf32_rne(a.x), tf32_rne(a.y), tf32_rne(a.z), tf32_rne(a.w)); }
NNAB_DEV float4 tf32_lo4(float4 a) {
  return make_float4(tf32_rne(a.x - tf32_rne(a.x)), tf32_rne(a.y - tf32_rne(a.y)), tf32_rne(a.z - tf32_rne(a.z)),
                     tf32_rne(a.w - tf32_rne(a.w)));
}
// coef pair (gradients.py:127-128), same arithmetic as coef_kernel: MUFU
// rsqrt (rel. error < 2^-22, far below the TF32 rounding of the result) instead
// of IEEE sqrt + two divisions -- the epilogue's 4 warps are issue-bound on those
NNAB_DEV void coef_store(float d, float r, float i, float eps, float& cr, float& ci) {
  const float inv = rsqrtf(fmaf(r, r, i * i) + eps);
  const float di = d * inv;
  cr = di * r;
  ci = di * i;
}

// FP16 hi = RN(v), lo = RN(v - hi) of four values, packed in pairs
NNAB_DEV void split_f16x4(float a, float b, float c, float d, uint2& hi, uint2& lo) {
  const __half2 h0 = __floats2half2_rn(a, b), h1 = __floats2half2_rn(c, d);
  const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
  const __half2 l0 = __floats2half2_rn(a - f0.x, b - f0.y), l1 = __floats2half2_rn(c - f1.x, d - f1.y);
  hi = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
  lo = make_uint2(*reinterpret_cast<const uint32_t*>(&l0), *reinterpret_cast<const uint32_t*>(&l1));
}

// 2^-clip_exp of the clips owning slots n .. n + 3 (0 past the last clip): one division
// when R >= 4 (the four slots then span at most two clips); |clip_exp| <= 100
NNAB_DEV void clip_scales(const RParams& p, int n, float* es) {
  const int b0 = n / p.clip_R, r0 = n - b0 * p.clip_R;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int b = p.clip_R >= 4 ? b0 + (r0 + j >= p.clip_R ? 1 : 0) : (n + j) / p.clip_R;
    es[j] = b < p.n_clips ? __int_as_float((127 - p.clip_exp[b]) << 23) : 0.f;
  }
}

NNAB_DEV uint64_t kdesc(const void* p, int swz) {
  uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * swz) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(swz == 128 ? 2 : 4) << 61;
  return d;
}
// MN-major FP16, 128-byte swizzle: K-rows of 128 B (64 MN elements), 8-row atoms
// SBO = 1024 B apart along K, 64-element MN atoms LBO apart.
NNAB_DEV uint64_t mndesc_f16(uint32_t addr, uint32_t lbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// MN-major TF32 uses the "128B_BASE32B" layout (32-byte units swizzled in a
// 128-byte row, 4 K-rows per atom; TMA SWIZZLE_128B_ATOM_32B): K-rows of 128 B
// (32 MN elements), SBO = 4 rows = 512 B between K groups, MN atoms LBO apart.
NNAB_DEV uint64_t mndesc(const void* p, int /*swz*/, uint32_t lbo) {
  uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}

// kPair (TF32): a cluster of two CTAs computes a 256 x 256 tile with
// cta_group::2 MMAs -- each CTA stages its own 128 A rows and HALF of the B tile,
// so the B bytes pulled from L2 per MAC halve (the long kernel-gradient
// reduction dK = coef @ frames is L2-bandwidth bound at 128 x 256 per CTA).
// kWide (with kPair): 256 x 512 tiles -- two N=256 MMAs per K step into all
// 512 TMEM columns (one accumulator), a quarter less L2 traffic per MAC again.
// kE8: the coef epilogues (nnab_mel_dft_coef: TF32 phasor, also with FP16 output; 3xTF32 with FP16
// output) on 8 epilogue warps (384 threads, 3 stages): their HBM-latency-bound loads get twice the
// warps in flight.
// kF16: the FP16 kernel gradient (nnab_kernel_grad_f16), 3xF16 with kSplit, else one FP16 pass --
// A = coef rows scaled by 2^(row_exp - clip_exp) as FP16 (hi/lo), B = the FP16 forward's staged frames (MN-major
// hop rows, x 2^clip_exp); the epilogue undoes 2^row_exp.
template <bool kSplit, bool kPair, bool kWide, bool kE8 = false, bool kF16 = false>
__global__ void __launch_bounds__(kE8 ? 384 : kThreads, 1)
    rgemm_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                 const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                 const __grid_constant__ CUtensorMap tc, const RParams p) {
  using C = RCfg<kSplit, kF16>;
  static_assert(!kF16 || (kPair && !kWide && !kE8), "FP16 kernel gradient: CTA-pair tiles");
  static_assert(!kWide || (kPair && !kSplit), "wide tiles are a TF32 pair mode");
  constexpr int TBN = kWide ? 2 * kBN : kBN;     // tile columns
  constexpr int NACC = kWide ? 1 : C::NUM_ACC;   // TMEM accumulators
  constexpr int kBNc = kPair ? kBN / 2 : kBN;  // B columns this CTA stages per MMA
  constexpr int kHalves = kWide ? 2 : 1;       // N=256 MMAs per K step
  constexpr int NST = kF16 ? C::NST_F16 : kE8 ? 3 : kStages;  // pipeline stages
  constexpr int kEW = kE8 ? 8 : 4;              // epilogue warps
  static_assert(!kE8 || !kWide, "8-warp epilogue: coef GEMMs only");
  const uint32_t rank = kPair ? cluster_ctarank() : 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * C::STAGE + (kF16 ? kF16Stg : 0));
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* tfull = bars + 2 * NST;
  uint64_t* tempty = bars + 2 * NST + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * NST + 4);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], (kPair ? 2 : 1) * kEW * 32);  // pair: the leader's counts both CTAs' threads
    }
    fence_barrier_init();
  }
  if (kPair) cluster_sync();
  if (warp == 2) {
    if (kPair) tmem_alloc_pair<512>(tslot);
    else tmem_alloc<512>(tslot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // work items: (m tile, n tile, split); a pair walks pair-tiles (two m tiles) by cluster
  const int m_units = kPair ? (p.m_tiles + 1) / 2 : p.m_tiles;
  const int n_work = m_units * p.n_tiles * p.splits;
  const int w_start = kPair ? (int)cluster_id_x() : (int)blockIdx.x;
  const int w_step = kPair ? (int)nclusters_x() : (int)gridDim.x;

  if (warp == 0) {
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_last();
      for (int w = w_start; w < n_work; w += w_step) {
        const int sp = w % p.splits, tile = w / p.splits;
        const int mt = (tile / p.n_tiles) * (kPair ? 2 : 1) + (int)rank, nt = tile % p.n_tiles;
        const int64_t k_lo = sp * p.k_per_split;
        const int64_t k_hi = (k_lo + p.k_per_split < p.K) ? k_lo + p.k_per_split : p.K;
        for (int64_t k = k_lo; k < k_hi; k += C::BK) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * C::STAGE;
          if constexpr (kF16) {
            const uint32_t fb = mapa(&full[s], 0);
            if (rank == 0) mbar_expect_tx(&full[s], 2 * C::STAGE);
            constexpr int kAs = kSplit ? 2 : 1;  // A slabs before the B half
            tma_load_2d_pair(st, &ta_hi, fb, (int)k, mt * kBM, pol);
            if (kSplit) tma_load_2d_pair(st + C::A_BYTES, &ta_lo, fb, (int)k, mt * kBM, pol);
            const int nb = nt * kBN + (int)rank * kBNc;
            int col = nb % p.b_row_len, row = (int)(k + nb / p.b_row_len);
#pragma unroll
            for (int j = 0; j < kBNc / 64; ++j) {  // boxes of {64 n, 64 k}: 8 KB, one MN atom column
              tma_load_2d_pair(st + kAs * C::A_BYTES + j * 8192, &tb_hi, fb, col, row, pol);
              if (kSplit) tma_load_2d_pair(st + kAs * C::A_BYTES + C::B_BYTES / 2 + j * 8192, &tb_lo, fb, col, row, pol);
              if ((col += 64) == p.b_row_len) col = 0, ++row;  // b_row_len % 64 == 0
            }
            if (++s == NST) { s = 0; ph ^= 1; }
            continue;
          } else if (kPair) {  // both CTAs' bytes complete on the leader's barrier
            const uint32_t fb = mapa(&full[s], 0);
            if (rank == 0)
              mbar_expect_tx(&full[s], 2 * (C::A_BYTES + kHalves * C::B_BYTES / 2) * (kSplit ? 2 : 1));
            tma_load_2d_pair(st, &ta_hi, fb, (int)k, mt * kBM, pol);
            if (kSplit) tma_load_2d_pair(st + C::A_BYTES + C::B_BYTES, &ta_lo, fb, (int)k, mt * kBM, pol);
#pragma unroll
            for (int h = 0; h < kHalves; ++h) {  // this CTA's half of each MMA's 256 columns
              const int nb = nt * TBN + h * kBN + (int)rank * kBNc;
              uint8_t* sb = st + C::A_BYTES + h * (C::B_BYTES / 2);
              uint8_t* sb_lo = st + 2 * C::A_BYTES + C::B_BYTES;  // 3xTF32 (never wide)
              if (!p.b_mn) {
                tma_load_2d_pair(sb, &tb_hi, fb, (int)k, nb, pol);
                if (kSplit) tma_load_2d_pair(sb_lo, &tb_lo, fb, (int)k, nb, pol);
              } else {
                int col = nb % p.b_row_len, row = (int)(k + nb / p.b_row_len);
#pragma unroll 1
                for (int j = 0; j < kBNc / 32; ++j) {
                  tma_load_2d_pair(sb + j * C::BK * 128, &tb_hi, fb, col, row, pol);
                  if (kSplit) tma_load_2d_pair(sb_lo + j * C::BK * 128, &tb_lo, fb, col, row, pol);
                  if ((col += 32) == p.b_row_len) col = 0, ++row;  // b_row_len % 32 == 0
                }
              }
            }
            if (++s == NST) { s = 0; ph ^= 1; }
            continue;
          }
          mbar_expect_tx(&full[s], C::STAGE);
          tma_load_2d(st, &ta_hi, &full[s], (int)k, mt * kBM);
          if (kSplit) tma_load_2d(st + C::A_BYTES + C::B_BYTES, &ta_lo, &full[s], (int)k, mt * kBM);
          if (!p.b_mn) {
            tma_load_2d(st + C::A_BYTES, &tb_hi, &full[s], (int)k, nt * kBN);
            if (kSplit) tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES, &tb_lo, &full[s], (int)k, nt * kBN);
          } else {
            // kBN/32 boxes of {32 n, BK k}; box j lands at j * (BK rows * 128 B)
#pragma unroll 1
            for (int j = 0; j < kBN / 32; ++j) {
              const int n0 = nt * kBN + j * 32;
              const int col = n0 % p.b_row_len;
              const int row = (int)(k + n0 / p.b_row_len);
              tma_load_2d(st + C::A_BYTES + j * C::BK * 128, &tb_hi, &full[s], col, row);
              if (kSplit)
                tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES + j * C::BK * 128, &tb_lo, &full[s], col, row);
            }
          }
          if (++s == NST) { s = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {
      const uint32_t idesc = idesc_tf32(kPair ? 2 * kBM : kBM, kBN) | (p.b_mn ? (1u << 16) : 0u);
      (void)idesc;
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int w = w_start; w < n_work; w += w_step) {
        const int sp = w % p.splits;
        const int64_t k_lo = sp * p.k_per_split;
        const int64_t k_hi = (k_lo + p.k_per_split < p.K) ? k_lo + p.k_per_split : p.K;
        for (int64_t kc = k_lo; kc < k_hi; kc += p.k_chunk) {
          const int64_t kc_hi = (kc + p.k_chunk < k_hi) ? kc + p.k_chunk : k_hi;
          mbar_wait(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tbase + (NACC > 1 ? acc * C::ACC_STRIDE : 0);
          bool first = true;
          for (int64_t k = kc; k < kc_hi; k += C::BK) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            uint8_t* st = smem + s * C::STAGE;
            if constexpr (kF16) {
              constexpr uint32_t idf = idesc_f16(2 * kBM, kBN) | (1u << 16);  // B MN-major
              const uint32_t sa = smem_u32(st), sb = sa + (kSplit ? 2 : 1) * C::A_BYTES;
#pragma unroll
              for (int kk = 0; kk < C::BK / 16; ++kk) {
                const uint64_t a = sdesc_kmajor_sw128_addr(sa + kk * 32);
                const uint64_t b = mndesc_f16(sb + kk * 2048, 8192);  // 16 K rows = two 8-row atoms
                mma_f16_pair(d, a, b, idf, first ? 0u : 1u);
                if (kSplit) {
                  const uint64_t a_lo = sdesc_kmajor_sw128_addr(sa + C::A_BYTES + kk * 32);
                  const uint64_t b_lo = mndesc_f16(sb + C::B_BYTES / 2 + kk * 2048, 8192);
                  mma_f16_pair(d + kBN, a, b_lo, idf, first ? 0u : 1u);
                  mma_f16_pair(d + kBN, a_lo, b, idf, 1u);
                }
                first = false;
              }
              mma_commit_pair(&empty[s], 0x3);
              if (++s == NST) { s = 0; ph ^= 1; }
              continue;
            }
            const uint64_t a = kdesc(st, C::SWZ);
            const uint64_t a_lo = kdesc(st + C::A_BYTES + C::B_BYTES, C::SWZ);
            // MN-major B: the kBN/32 boxes are C::BK*128 bytes apart (LBO)
            const uint64_t b = p.b_mn ? mndesc(st + C::A_BYTES, 128, C::BK * 128) : kdesc(st + C::A_BYTES, C::SWZ);
            const uint64_t b_lo = p.b_mn ? mndesc(st + 2 * C::A_BYTES + C::B_BYTES, 128, C::BK * 128)
                                         : kdesc(st + 2 * C::A_BYTES + C::B_BYTES, C::SWZ);
#pragma unroll
            for (int kk = 0; kk < C::BK / 8; ++kk) {
              const uint64_t ao = (uint64_t)((kk * 32) >> 4);
              const uint64_t bo = p.b_mn ? (uint64_t)((kk * 1024) >> 4) : ao;  // MN-major: next 8 K rows
              if (kPair) {
                mma_tf32_pair(d, a + ao, b + bo, idesc, first ? 0u : 1u);
                if (kWide)  // second 256 columns: B half staged B_BYTES/2 further on
                  mma_tf32_pair(d + kBN, a + ao, b + bo + (uint64_t)((C::B_BYTES / 2) >> 4), idesc, first ? 0u : 1u);
                if (kSplit) {
                  mma_tf32_pair(d + kBN, a + ao, b_lo + bo, idesc, first ? 0u : 1u);
                  mma_tf32_pair(d + kBN, a_lo + ao, b + bo, idesc, 1u);
                }
              } else {
                mma_tf32(d, a + ao, b + bo, idesc, first ? 0u : 1u);
                if (kSplit) {
                  mma_tf32(d + kBN, a + ao, b_lo + bo, idesc, first ? 0u : 1u);
                  mma_tf32(d + kBN, a_lo + ao, b + bo, idesc, 1u);
                }
              }
              first = false;
            }
            if (kPair) mma_commit_pair(&empty[s], 0x3);
            else mma_commit(&empty[s]);
            if (++s == NST) { s = 0; ph ^= 1; }
          }
          if (kPair) mma_commit_pair(&tfull[acc], 0x3);
          else mma_commit(&tfull[acc]);
          if (++acc == NACC) { acc = 0; aph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // Epilogue: TMEM row = thread, so each 32-column chunk goes through a
    // per-warp shared-memory transpose (32 rows x 36-float stride, conflict-free
    // for float4) and leaves as float4 runs of 8 lanes per row: every global
    // access is a full 128-byte line instead of 32 rows x 16 B.
    const uint32_t ew = warp - 4, q = ew & 3;  // TMEM lane quarter
    if constexpr (kF16) {
      // Drain per TMEM chunk: main + correction accumulators -> registers (thread = row),
      // x 2^-row_exp, into a swizzled staging tile, then TMA: the split's first chunk
      // stores, later ones reduce-add in L2 (no read-modify-write round trip through the
      // SM).  TMEM is released right after the last tcgen05.ld, so the MMAs of the next
      // chunk overlap the stores.  Chunk d's reduce-adds are issued only after chunk
      // d - 1's completed: a fixed summation order (deterministic).
      uint8_t* stg16 = smem + NST * C::STAGE + ew * 8192;
      const uint32_t tempty0 = mapa(&tempty[0], 0);
      uint32_t aph = 0;
      int acc = 0;  // TMEM accumulator (one pass: double-buffered; 3xF16: main + correction)
      for (int w = w_start; w < n_work; w += w_step) {
        const int sp = w % p.splits, tile = w / p.splits;
        const int mt = (tile / p.n_tiles) * 2 + (int)rank, nt = tile % p.n_tiles;
        const int64_t k_lo = sp * p.k_per_split;
        const int64_t k_hi = (k_lo + p.k_per_split < p.K) ? k_lo + p.k_per_split : p.K;
        const int m_base = mt * kBM + (int)q * 32;
        const int crow = sp * p.c_split_rows + m_base;
        const int m = m_base + (int)lane;
        const float rs = m < p.M ? __int_as_float((127 - p.row_exp[m]) << 23) : 0.f;
        for (int64_t kc = k_lo; kc < k_hi; kc += p.k_chunk) {
          const bool first_chunk = kc == k_lo;
          mbar_wait(&tfull[acc], aph);
          tc_fence_after();
          const uint32_t tb = tbase + ((q * 32) << 16) + (NACC > 1 ? acc * C::ACC_STRIDE : 0);
          if (lane == 0) bulk_wait_all();  // the previous chunk's stores / adds have landed
          __syncwarp();
#pragma unroll 1
          for (int c = 0; c < kBN / 32; ++c) {
            float v[32], u[32];
            tmem_ld32(tb + c * 32, v);
            if (kSplit) {
              tmem_ld32(tb + kBN + c * 32, u);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) u[j] = 0.f;
            }
            tmem_ld_wait();
            if (c == kBN / 32 - 1) {  // accumulators read: the next chunk's MMAs may start
              tc_fence_before();
              mbar_arrive_cluster(tempty0 + 8 * acc);
            }
            uint8_t* buf = stg16 + (c & 1) * 4096;
            if (c >= 2) {
              if (lane == 0) bulk_wait_read_n<1>();  // chunk c - 2's copy has read this buffer
              __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                  make_float4((v[4 * j] + u[4 * j]) * rs, (v[4 * j + 1] + u[4 * j + 1]) * rs,
                              (v[4 * j + 2] + u[4 * j + 2]) * rs, (v[4 * j + 3] + u[4 * j + 3]) * rs);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && m_base < p.M) {  // a pair's rows past M: nothing (they would reach the next split)
              const int col = nt * kBN + c * 32;
              if (first_chunk) tma_store_2d(&tc, buf, col, crow);
              else tma_reduce_add_2d(&tc, buf, col, crow);
              bulk_commit();
            }
          }
          if (++acc == NACC) { acc = 0; aph ^= 1; }
        }
      }
      if (lane == 0) bulk_wait_all();
      __syncwarp();
    } else {
    const int hsel = kE8 ? (int)(ew >> 2) : 0;  // kE8: warps 4-7 even chunks, 8-11 odd ones
    constexpr int CSTEP = kE8 ? 2 : 1;
    float* stg = reinterpret_cast<float*>(smem + NST * C::STAGE + 128) + ew * 32 * kStg;
    const int sr = (int)(lane >> 3), sc = (int)(lane & 7) * 4;  // this lane's (row in 4, float4 column)
    int acc = 0;
    uint32_t aph = 0;
    const uint32_t tempty0 = kPair ? mapa(&tempty[0], 0) : smem_u32(&tempty[0]);
    const bool vec = (p.ldc % 4) == 0;
    for (int w = w_start; w < n_work; w += w_step) {
      const int sp = w % p.splits, tile = w / p.splits;
      const int mt = (tile / p.n_tiles) * (kPair ? 2 : 1) + (int)rank, nt = tile % p.n_tiles;
      const int64_t k_lo = sp * p.k_per_split;
      const int64_t k_hi = (k_lo + p.k_per_split < p.K) ? k_lo + p.k_per_split : p.K;
      const int m_base = mt * kBM + (int)q * 32;
      float rsv[8];  // coef_f16: this thread's rows' 2^row_exp (rows m_base + 4 it + sr)
      if (p.coef_f16) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int m = m_base + it * 4 + sr;
          rsv[it] = m < p.M ? __int_as_float((127 + p.row_exp[m]) << 23) : 0.f;
        }
      }
      float* cbase = p.C + sp * p.split_stride;
      for (int64_t kc = k_lo; kc < k_hi; kc += p.k_chunk) {
        const bool first_chunk = kc == k_lo;  // later chunks add into C in fixed order: deterministic
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t tb = tbase + ((q * 32) << 16) + (NACC > 1 ? acc * C::ACC_STRIDE : 0);
        // phasor coef epilogue: chunk c + 1's phasor loads are in flight while chunk c
        // is drained (the epilogue is HBM-latency bound with 4 warps per SM)
        const bool phasor = !kSplit && (kE8 || (p.re && !p.im));  // split modes save re and im
        uint4 ph_cur[8], ph_nxt[8];
        auto load_ph = [&](int c, uint4* dst) {
          const int n = nt * TBN + c * 32 + sc;
          const bool full4 = vec && n + 4 <= p.N;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int m = m_base + it * 4 + sr;
            if (m < p.M && full4) dst[it] = __ldcs(reinterpret_cast<const uint4*>(p.re + (int64_t)m * p.ldc + n));
          }
        };
        if (phasor) load_ph(hsel, ph_cur);
#pragma unroll 1
        for (int c = hsel; c < TBN / 32; c += CSTEP) {
          if (phasor && c + CSTEP < TBN / 32) load_ph(c + CSTEP, ph_nxt);
          float v[32];
          tmem_ld32(tb + c * 32, v);
          if (kSplit) {
            float u[32];
            tmem_ld32(tb + kBN + c * 32, u);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += u[j];
          } else {
            tmem_ld_wait();
          }
          __syncwarp();  // the previous chunk's reads of stg are done
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(stg + lane * kStg + 4 * j) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          __syncwarp();
          const int n = nt * TBN + c * 32 + sc;
          if (n >= p.N || m_base >= p.M) {
            if (phasor) {
#pragma unroll
              for (int it = 0; it < 8; ++it) ph_cur[it] = ph_nxt[it];
            }
            continue;
          }
          const bool full4 = vec && n + 4 <= p.N;
          float4 d[8];
#pragma unroll
          for (int it = 0; it < 8; ++it) d[it] = *reinterpret_cast<const float4*>(stg + (it * 4 + sr) * kStg + sc);
          if (phasor) {  // coef epilogue from the saved unit phasor (re/S, im/S) in FP16 pairs
            uint4 ph[8];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              ph[it] = ph_cur[it];
              ph_cur[it] = ph_nxt[it];
            }
            float es[4] = {0.f, 0.f, 0.f, 0.f};  // coef_f16: 2^-clip_exp per column
            if (p.coef_f16) clip_scales(p, n, es);
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int m = m_base + it * 4 + sr;
              if (m >= p.M) continue;
              const int64_t o = (int64_t)m * p.ldc + n, o2 = o + (int64_t)p.M * p.ldc;
              if (p.coef_f16) {  // one-pass FP16 kernel-gradient operand: coef * 2^(row_exp - clip_exp)
                const float rs = rsv[it];
                const float dv[4] = {d[it].x, d[it].y, d[it].z, d[it].w};
                __half* ch = reinterpret_cast<__half*>(p.C);
                float cr[4], ci[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  float2 f = make_float2(0.f, 0.f);
                  if (full4) f = __half22float2(reinterpret_cast<const __half2*>(&ph[it])[j]);
                  else if (n + j < p.N) f = __half22float2(reinterpret_cast<const __half2*>(p.re)[o + j]);
                  cr[j] = dv[j] * f.x * es[j] * rs;
                  ci[j] = dv[j] * f.y * es[j] * rs;
                }
                const __half2 r01 = __floats2half2_rn(cr[0], cr[1]), r23 = __floats2half2_rn(cr[2], cr[3]);
                const __half2 i01 = __floats2half2_rn(ci[0], ci[1]), i23 = __floats2half2_rn(ci[2], ci[3]);
                if (full4) {
                  __stcs(reinterpret_cast<uint2*>(ch + o), make_uint2(*reinterpret_cast<const uint32_t*>(&r01),
                                                                      *reinterpret_cast<const uint32_t*>(&r23)));
                  __stcs(reinterpret_cast<uint2*>(ch + o2), make_uint2(*reinterpret_cast<const uint32_t*>(&i01),
                                                                       *reinterpret_cast<const uint32_t*>(&i23)));
                } else {
#pragma unroll
                  for (int j = 0; j < 4; ++j)
                    if (n + j < p.N) {
                      ch[o + j] = __float2half_rn(cr[j]);
                      ch[o2 + j] = __float2half_rn(ci[j]);
                    }
                }
                continue;
              }
              if (full4) {
                const __half2* h2 = reinterpret_cast<const __half2*>(&ph[it]);
                const float2 f0 = __half22float2(h2[0]), f1 = __half22float2(h2[1]), f2 = __half22float2(h2[2]),
                             f3 = __half22float2(h2[3]);
                const float4 hr = make_float4(d[it].x * f0.x, d[it].y * f1.x, d[it].z * f2.x, d[it].w * f3.x);
                const float4 hi = make_float4(d[it].x * f0.y, d[it].y * f1.y, d[it].z * f2.y, d[it].w * f3.y);
                __stcs(reinterpret_cast<float4*>(p.C + o), tf32_hi4(hr));
                __stcs(reinterpret_cast<float4*>(p.C + o2), tf32_hi4(hi));
              } else {
                const float dv[4] = {d[it].x, d[it].y, d[it].z, d[it].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  if (n + j >= p.N) continue;
                  const float2 f = __half22float2(reinterpret_cast<const __half2*>(p.re)[o + j]);
                  p.C[o + j] = tf32_rne(dv[j] * f.x);
                  p.C[o2 + j] = tf32_rne(dv[j] * f.y);
                }
              }
            }
          } else if constexpr (!kE8 || kSplit) {
          if (p.re) {  // coef epilogue: the dS tile never leaves the SM
            float4 rr[8], ii[8];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int m = m_base + it * 4 + sr;
              const int64_t o = (int64_t)m * p.ldc + n;
              if (m < p.M && full4) {
                rr[it] = __ldcs(reinterpret_cast<const float4*>(p.re + o));  // read once: stream
                ii[it] = __ldcs(reinterpret_cast<const float4*>(p.im + o));
              }
            }
            if (p.coef_f16) {  // FP16 hi/lo of coef * 2^(row_exp[m] - clip_exp[slot]) (3xF16 dK operand)
              float es[4];
              clip_scales(p, n, es);
              __half* ch = reinterpret_cast<__half*>(p.C);
              __half* cl = reinterpret_cast<__half*>(p.c_lo);
#pragma unroll
              for (int it = 0; it < 8; ++it) {
                const int m = m_base + it * 4 + sr;
                if (m >= p.M) continue;
                const float rs = rsv[it];  // |row_exp| <= 125
                const int64_t o = (int64_t)m * p.ldc + n, o2 = o + (int64_t)p.M * p.ldc;
                const float dv[4] = {d[it].x, d[it].y, d[it].z, d[it].w};
                float cr[4], ci[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  float r_, i_;
                  if (full4) {
                    r_ = j == 0 ? rr[it].x : j == 1 ? rr[it].y : j == 2 ? rr[it].z : rr[it].w;
                    i_ = j == 0 ? ii[it].x : j == 1 ? ii[it].y : j == 2 ? ii[it].z : ii[it].w;
                  } else {
                    r_ = n + j < p.N ? p.re[o + j] : 0.f;
                    i_ = n + j < p.N ? p.im[o + j] : 0.f;
                  }
                  coef_store(dv[j], r_, i_, p.eps, cr[j], ci[j]);
                  cr[j] *= es[j] * rs;
                  ci[j] *= es[j] * rs;
                }
                uint2 hr, lr, hi4, li4;
                split_f16x4(cr[0], cr[1], cr[2], cr[3], hr, lr);
                split_f16x4(ci[0], ci[1], ci[2], ci[3], hi4, li4);
                if (full4) {
                  __stcs(reinterpret_cast<uint2*>(ch + o), hr);
                  __stcs(reinterpret_cast<uint2*>(cl + o), lr);
                  __stcs(reinterpret_cast<uint2*>(ch + o2), hi4);
                  __stcs(reinterpret_cast<uint2*>(cl + o2), li4);
                } else {
                  const uint32_t w4[4][2] = {{hr.x, hr.y}, {lr.x, lr.y}, {hi4.x, hi4.y}, {li4.x, li4.y}};
                  __half* dst[4] = {ch + o, cl + o, ch + o2, cl + o2};
#pragma unroll
                  for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                      if (n + j < p.N)
                        dst[a][j] = __ushort_as_half((unsigned short)(w4[a][j >> 1] >> (16 * (j & 1))));
                }
              }
            } else {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int m = m_base + it * 4 + sr;
              if (m >= p.M) continue;
              const int64_t o = (int64_t)m * p.ldc + n, o2 = o + (int64_t)p.M * p.ldc;
              if (full4) {
                float4 hr, hi;
                coef_store(d[it].x, rr[it].x, ii[it].x, p.eps, hr.x, hi.x);
                coef_store(d[it].y, rr[it].y, ii[it].y, p.eps, hr.y, hi.y);
                coef_store(d[it].z, rr[it].z, ii[it].z, p.eps, hr.z, hi.z);
                coef_store(d[it].w, rr[it].w, ii[it].w, p.eps, hr.w, hi.w);
                if (kSplit) {
                  __stcs(reinterpret_cast<float4*>(p.c_lo + o), tf32_lo4(hr));
                  __stcs(reinterpret_cast<float4*>(p.c_lo + o2), tf32_lo4(hi));
                }
                __stcs(reinterpret_cast<float4*>(p.C + o), tf32_hi4(hr));
                __stcs(reinterpret_cast<float4*>(p.C + o2), tf32_hi4(hi));
              } else {
                const float dv[4] = {d[it].x, d[it].y, d[it].z, d[it].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  if (n + j >= p.N) continue;
                  float cr, ci;
                  coef_store(dv[j], p.re[o + j], p.im[o + j], p.eps, cr, ci);
                  p.C[o + j] = tf32_rne(cr);
                  p.C[o2 + j] = tf32_rne(ci);
                  if (kSplit) {
                    p.c_lo[o + j] = tf32_rne(cr - tf32_rne(cr));
                    p.c_lo[o2 + j] = tf32_rne(ci - tf32_rne(ci));
                  }
                }
              }
            }
            }  // !coef_f16
          } else if (p.fR) {  // one chunk, no split: the slot tile lands in (B, M, T) directly
            const int64_t b = n / p.fR;  // R % 4 == 0: the lane's 4 slots share a clip
            const int t0 = (int)(n - b * p.fR);
            if (b < p.fB) {
#pragma unroll
              for (int it = 0; it < 8; ++it) {
                const int m = m_base + it * 4 + sr;
                if (m >= p.M) continue;
                float* orow = p.C + (b * p.M + m) * (int64_t)p.fT;
                const float dv[4] = {d[it].x, d[it].y, d[it].z, d[it].w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  if (t0 + j < p.fT && n + j < p.N) orow[t0 + j] = dv[j];
              }
            }
          } else {
            // the running sum lives in C (L2): all loads are in flight before any add
            float4 cur[8];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int m = m_base + it * 4 + sr;
              cur[it] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (!first_chunk && m < p.M && full4)
                cur[it] = *reinterpret_cast<const float4*>(cbase + (int64_t)m * p.ldc + n);
            }
            if (p.row_exp) {  // undo the operand's per-row 2^row_exp (exact)
#pragma unroll
              for (int it = 0; it < 8; ++it) {
                const int m = m_base + it * 4 + sr;
                if (m >= p.M) continue;
                const float rs = __int_as_float((127 - p.row_exp[m]) << 23);
                d[it] = make_float4(d[it].x * rs, d[it].y * rs, d[it].z * rs, d[it].w * rs);
              }
            }
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int m = m_base + it * 4 + sr;
              if (m >= p.M) continue;
              float* crow = cbase + (int64_t)m * p.ldc + n;
              if (full4) {
                *reinterpret_cast<float4*>(crow) = make_float4(cur[it].x + d[it].x, cur[it].y + d[it].y,
                                                               cur[it].z + d[it].z, cur[it].w + d[it].w);
              } else {
                const float dv[4] = {d[it].x, d[it].y, d[it].z, d[it].w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  if (n + j < p.N) crow[j] = first_chunk ? dv[j] : crow[j] + dv[j];
              }
            }
          }
          }  // !kE8
        }
        tc_fence_before();
        if (kPair) mbar_arrive_cluster(tempty0 + 8 * acc);
        else mbar_arrive(&tempty[acc]);
        if (++acc == NACC) { acc = 0; aph ^= 1; }
      }
    }
    }  // !kF16
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();  // the peer's TMEM is written by the leader's MMAs until the end
  tc_fence_after();
  if (warp == 2) {
    if (kPair) tmem_dealloc_pair<512>(tbase);
    else tmem_dealloc<512>(tbase);
  }
}

// out[m][n] = sum_s parts[s][m][n] in a fixed order (deterministic split-K)
__global__ void sum_splits_kernel(const float* __restrict__ parts, int32_t splits, int64_t stride, int32_t M,
                                  int32_t N, int64_t ldp, float* __restrict__ out, int64_t ldo, float alpha) {
  const int64_t total = (int64_t)M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / N, n = e - m * N;
    float a = 0.f;
    for (int s = 0; s < splits; ++s) a += parts[s * stride + m * ldp + n];
    out[m * ldo + n] = alpha * a;
  }
}

template <bool kSplit, bool kPair, bool kWide = false, bool kE8 = false, bool kF16 = false>
int launch(const RGemmArgs& g, cudaStream_t st) {
  using C = RCfg<kSplit, kF16>;
  constexpr int kBNc = kPair ? kBN / 2 : kBN;
  constexpr int TBN = kWide ? 2 * kBN : kBN;
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  int rc = NNAB_OK;
  if (kF16) {  // K need not be a multiple of BK: the tail boxes are zero-filled past K and b_rows
    if (g.lda % 8 || !g.b_mn || g.b_row_len % 64 || (kSplit && (!g.a_lo || !g.b_lo)) || !g.row_exp)
      return NNAB_EINVAL;
    rc = make_tmap_2d(&ta_hi, g.a_hi, g.K, g.M, (uint64_t)g.lda * 2, 64, kBM, 128, 2);
    if (!rc && kSplit) rc = make_tmap_2d(&ta_lo, g.a_lo, g.K, g.M, (uint64_t)g.lda * 2, 64, kBM, 128, 2);
    if (!rc) rc = make_tmap_2d(&tb_hi, g.b_hi, g.b_row_len, g.b_rows, (uint64_t)g.b_row_len * 2, 64, 64, 128, 2);
    if (!rc && kSplit)
      rc = make_tmap_2d(&tb_lo, g.b_lo, g.b_row_len, g.b_rows, (uint64_t)g.b_row_len * 2, 64, 64, 128, 2);
  } else if (g.K % C::BK || g.lda % 4 || (g.b_mn && g.b_row_len % 32) || (!g.b_mn && g.ldb % 4)) {
    return NNAB_EINVAL;
  } else {
  rc = make_tmap_2d(&ta_hi, g.a_hi, g.K, g.M, (uint64_t)g.lda * 4, C::BK, kBM, C::SWZ);
  if (!rc && kSplit) rc = make_tmap_2d(&ta_lo, g.a_lo, g.K, g.M, (uint64_t)g.lda * 4, C::BK, kBM, C::SWZ);
  if (!g.b_mn) {
    if (!rc) rc = make_tmap_2d(&tb_hi, g.b_hi, g.K, g.N, (uint64_t)g.ldb * 4, C::BK, kBNc, C::SWZ);
    if (!rc && kSplit) rc = make_tmap_2d(&tb_lo, g.b_lo, g.K, g.N, (uint64_t)g.ldb * 4, C::BK, kBNc, C::SWZ);
  } else {
    // rows of b_row_len floats; b_rows rows in total; boxes of 32 columns x BK rows, 128-byte swizzle
    if (!rc) rc = make_tmap_2d(&tb_hi, g.b_hi, g.b_row_len, g.b_rows, (uint64_t)g.b_row_len * 4, 32, C::BK, -128);
    if (!rc && kSplit)
      rc = make_tmap_2d(&tb_lo, g.b_lo, g.b_row_len, g.b_rows, (uint64_t)g.b_row_len * 4, 32, C::BK, -128);
  }
  }
  if (rc) return rc;
  if (!kSplit) {
    ta_lo = ta_hi;
    tb_lo = tb_hi;
  }
  RParams p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.m_tiles = (g.M + kBM - 1) / kBM;
  p.n_tiles = (g.N + TBN - 1) / TBN;
  const int tiles = p.m_tiles * p.n_tiles;
  const int units = (kPair ? (p.m_tiles + 1) / 2 * 2 : p.m_tiles) * p.n_tiles;  // CTAs per split
  const int64_t kb = (g.K + C::BK - 1) / C::BK;
  int splits = (g.coef_re || g.frames_R) ? 1 : g.splits > 0 ? g.splits : auto_splits(units, kb);
  splits = (int)std::min<int64_t>(splits, kb);
  p.k_per_split = (kb + splits - 1) / splits * C::BK;
  p.splits = (int)((g.K + p.k_per_split - 1) / p.k_per_split);
  // one FP16 pass: its 11-bit operands dwarf the accumulate steps' error, so long chains (as wide TF32)
  p.k_chunk = (kF16 ? (kSplit ? f16_chunk() : 8192) : kSplit ? 1024 : kWide ? 8192 : 2048);  // accumulate steps per TMEM
                                                    // chain (wide: no second accumulator, so drain less often)
  // the epilogues that write final values (frames output, coef) need one TMEM chain per tile:
  // up to 2,048 K in every mode (a 3xTF32 Mel forward over 1,025 bins has K = 1,056)
  if ((g.frames_R || g.coef_re) && kb * C::BK <= 2048) p.k_chunk = std::max<int64_t>(p.k_chunk, kb * C::BK);
  p.b_mn = g.b_mn;
  p.b_row_len = g.b_mn ? g.b_row_len : 1 << 30;
  p.re = g.coef_re;
  p.im = g.coef_im;
  p.c_lo = g.coef_lo;
  p.eps = g.coef_eps;
  p.fB = g.frames_B;
  p.fR = g.frames_R;
  p.fT = g.frames_T;
  p.row_exp = g.row_exp;
  p.clip_exp = g.clip_exp;
  p.n_clips = g.n_clips;
  p.clip_R = g.clip_R;
  p.coef_f16 = g.coef_f16;
  // coef_f16: 3xTF32 from re / im (FP16 hi + lo out) or TF32 from the FP16 unit phasor (hi only)
  if (p.coef_f16 && (kF16 || !p.re || (kSplit && (!p.im || !p.c_lo)) || !p.row_exp || !p.clip_exp || p.clip_R < 1 ||
                     g.ldc % 4))
    return NNAB_EINVAL;
  if (p.fR && (p.fR % 4 || p.splits != 1 || kb > p.k_chunk / C::BK || g.alpha != 1.f || p.re)) return NNAB_EINVAL;
  if (p.re && (p.splits != 1 || kb > p.k_chunk / C::BK || g.alpha != 1.f)) return NNAB_EINVAL;  // one TMEM chain
  const bool direct = p.splits == 1 && g.alpha == 1.f && (!kF16 || g.ldc % 4 == 0);  // kF16: TMA row stride
  p.C = direct ? g.c : g.partial;
  p.ldc = direct ? g.ldc : (int64_t)p.n_tiles * TBN;
  p.split_stride = (int64_t)p.m_tiles * kBM * p.ldc;
  if (!direct && !g.partial) return NNAB_EINVAL;
  CUtensorMap tc = ta_hi;
  p.c_split_rows = 0;
  if (kF16) {  // C (or the split partials) as a 2-D fp32 tensor, 32 x 32 boxes, 128-byte swizzle
    if (direct) rc = make_tmap_2d(&tc, p.C, g.N, g.M, (uint64_t)p.ldc * 4, 32, 32, 128, 4);
    else {
      p.c_split_rows = p.m_tiles * kBM;
      rc = make_tmap_2d(&tc, p.C, p.ldc, (uint64_t)p.splits * p.c_split_rows, (uint64_t)p.ldc * 4, 32, 32, 128, 4);
    }
    if (rc) return rc;
  }
  const size_t smem = 1024 + (kF16 ? C::NST_F16 : kE8 ? 3 : kStages) * C::STAGE + 128 +
                      (kF16 ? kF16Stg : (kE8 ? 8 : 4) * 32 * kStg * 4);
  constexpr int threads = kE8 ? 384 : kThreads;
  auto k = rgemm_kernel<kSplit, kPair, kWide, kE8, kF16>;
  NNAB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  (void)tiles;
  if (!kPair) {
    const int grid = std::min(units * p.splits, num_sms());
    k<<<grid, threads, smem, st>>>(ta_hi, ta_lo, tb_hi, tb_lo, tc, p);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min(units * p.splits, num_sms() / 2 * 2));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    NNAB_CUDA_TRY(cudaLaunchKernelEx(&cfg, k, ta_hi, ta_lo, tb_hi, tb_lo, tc, p));
  }
  NNAB_LAUNCHED();
  if (!direct) {
    const int64_t total = (int64_t)g.M * g.N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
    sum_splits_kernel<<<blocks, 256, 0, st>>>(g.partial, p.splits, p.split_stride, g.M, g.N, p.ldc, g.c, g.ldc,
                                              g.alpha);
    NNAB_LAUNCHED();
  }
  return NNAB_OK;
}

}  // namespace

size_t rgemm_partial_bytes(int32_t M, int32_t N, int64_t K, int32_t splits) {
  const int64_t mt = (M + kBM - 1) / kBM;
  const int64_t nt = (N + 2 * kBN - 1) / (2 * kBN) * 2;  // 256-column tiles, even: covers the wide layout
  if (splits <= 0) {  // auto split count: the largest any tile form picks
    const int64_t kb = std::max<int64_t>(1, K / 16), kb64 = std::max<int64_t>(1, (K + 63) / 64);
    const int64_t u_single = mt * ((N + kBN - 1) / kBN), u_pair = (mt + 1) / 2 * 2 * ((N + kBN - 1) / kBN),
                  u_wide = (mt + 1) / 2 * 2 * (nt / 2);
    splits = std::max(auto_splits(u_single, kb), std::max(auto_splits(u_pair, kb), auto_splits(u_wide, kb)));
    splits = std::max(splits, auto_splits(u_pair, kb64));  // 3xF16 (64 K per block)
  }
  return (size_t)splits * mt * kBM * nt * kBN * sizeof(float);
}

// TF32 reductions over more than one m tile use the CTA-pair form: measured
// 6.77 -> 4.46 ms on the 2050 x 2048 x 283,200 kernel gradient, never slower on
// smaller shapes (tools/dbg_rgemm_pair.py).  NNAB_RGEMM_PAIR=0 forces single CTAs.
int launch_rgemm(const RGemmArgs& g, int precision, cudaStream_t s) {
  static const int pair_env = [] {
    const char* e = getenv("NNAB_RGEMM_PAIR");
    return e ? e[0] - '0' : 1;
  }();
  const bool pair_ok = pair_env != 0;
  if (precision == NNAB_PREC_3XTF32) {  // CTA pairs too (the long reductions are L2-bound)
    const bool pair = pair_ok && (pair_env >= 2 || g.M > kBM);
    static const bool e8_split = [] {
      const char* e = getenv("NNAB_COEF_E8");
      return !(e && e[0] == '0');
    }();
    // the FP16-output coef epilogue is ALU-latency bound on 4 warps: twice the warps
    if (pair && e8_split && g.coef_f16) return launch<true, true, false, true>(g, s);
    return pair ? launch<true, true>(g, s) : launch<true, false>(g, s);
  }
  if (precision == NNAB_PREC_3XF16) return launch<true, true, false, false, true>(g, s);
  if (precision == NNAB_PREC_F16) return launch<false, true, false, false, true>(g, s);
  if (precision == NNAB_PREC_TF32) {
    const bool pair = pair_ok && (pair_env >= 2 || g.M > kBM);  // one m tile: the peer would idle
    const bool wide = pair && !g.coef_re && (pair_env == 3 || (pair_env == 1 && g.N > kBN && g.K >= 65536));
    if (wide) return launch<false, true, true>(g, s);
    static const bool e8_ok = [] {
      const char* e = getenv("NNAB_COEF_E8");
      return !(e && e[0] == '0');
    }();
    if (pair && e8_ok && g.coef_re && !g.coef_im) return launch<false, true, false, true>(g, s);
    return pair ? launch<false, true>(g, s) : launch<false, false>(g, s);
  }
  return NNAB_EINVAL;
}

}  // namespace nnab
