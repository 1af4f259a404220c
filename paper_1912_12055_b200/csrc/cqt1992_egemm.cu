// CQT1992v2 as a hop-offset GEMM ("E-GEMM") plus a diagonal sum.
//
// The reference correlates every clip with the long complex bank
// (transforms.py:175-186, 201-208): D[s][row] = sum_k frame_s[k] K[row][k].
// With the clip staged as hop rows (frame s = rows s, s+1, ... of `hop`
// samples, csrc/frames.cu) and k = hop * r + c:
//   D[s][row] = sum_r E[s + r][(row, r)],   E[s][(row, r)] = sum_c rows[s][c] K[row][hop r + c].
// E is a plain GEMM with K = hop (512) whose N columns are the (row, r) pairs
// where row's centred support touches hop block r -- about 1,730 of them for
// the 84-bin bank, against the 709 narrow K blocks (N = 24..168 rows) the
// direct schedule (cqt1992.cu) issues per M tile; the long low-frequency rows
// become many columns instead of many tiny MMAs.
//
// Used for the long low-frequency bins of the default hybrid
// (nnab_cqt1992v2_hybrid_staged; CqtLongEngine(method="hybrid")): bins whose
// support spans >= 8 hops here, the per-K-block schedule (cqt1992.cu) for the
// rest.  On the 1,770-clip batch: schedule alone 3.4 ms, E-GEMM alone 1.6 ms,
// hybrid 1.45 ms (+ 0.4 ms frame staging).
//
// Columns are packed into groups of <= 256 columns / <= 8 bins (16 bank rows),
// longest bins first; each row's columns are whole windows of 16 consecutive
// hop offsets r (zero-weight past its support).  A persistent CTA owns one group
// and a contiguous run of M tiles (128 hop rows each): TMA producer warp,
// single-thread tcgen05.mma issuer (M = 128, N = 256, K = 8, TF32, two TMEM
// accumulators), and 4 epilogue warps.  Epilogue: thread = E row s; for a
// window (row, r0 .. r0+15) lane l gathers E[s_l + k][(row, r0 + k)] from lane
// (l + k) mod 32 by shuffle, so the window folds into two register sums (the
// pairs whose source lane wrapped belong to D row s_l - 32 - r0, the rest to
// s_l - r0) and two read-modify-writes of the warp's private ring of D rows --
// no atomics, no shared-memory staging of E, deterministic for a given tiling.
// D rows that can receive nothing more are summed over the four warp rings,
// turned into magnitude / power / complex and written to the (B, n_bins, T)
// output, coalesced along T.  Each CTA also computes the first tile past its
// run (a 1-in-~150 overlap) so its last D rows are complete; D rows before its
// run belong to the previous CTA.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 32, kThreads = 384;
constexpr int kA = kBM * kBK * 4;  // 16 KB A tile per stage
constexpr int kRows = 16;   // D rows (bank rows: 2 per bin) per group
constexpr int kRing = 256;  // D ring length (slots, power of two); >= 128 + max r
constexpr uint16_t kUnused = 0xFFFF;
constexpr int kWin = 16;  // a row's columns come in windows of 16 consecutive r

constexpr int kChunk = 64;  // run-table granularity (host plan only)
constexpr int kChunks = kBN / kChunk;
constexpr int kRunSlots = kChunk + 1;  // per chunk: count, then up to 64 runs
constexpr int kEpi = 256;  // warps 4-11: TMEM readers and reducers (two per TMEM lane quarter)

struct EParams {
  int64_t B;
  int32_t R, T, n_mtiles, n_bins, out_kind;
  int32_t n_groups, ctas_per_group, r_max;
  float eps;
  const uint16_t* col_table;  // [n_groups][256]: row_local << 8 | r
  const int32_t* group_rows;  // [n_groups][64]: bank row 2*bin + im, -1 unused
  float* out;
  const int32_t* a_exp;  // FP16: per-clip scale exponent of the staged rows
  const int32_t* b_exp;  // FP16: the bank's scale exponent
};

NNAB_DEV uint64_t sdesc(const void* p) {  // K-major, 128-byte swizzle, 8-row atoms
  uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

NNAB_DEV void ep_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }  // epilogue warps 4-11

// Pipeline geometry: single CTAs stage A (16 KB) + all of B (32 KB) x 3; a CTA
// pair (kPair) stages A + half of B (16 + 16 KB) x 4; 3xTF32 (kSplit, pairs)
// stages hi and lo of both (64 KB) x 2.
// kHalf: FP16 operands (staged rows and bank under exact power-of-two scales, kind::f16):
// the same 128-byte K-block rows hold 64 samples instead of 32, so K = hop = 512 is 8
// K blocks; the scales are undone when the D rows are emitted.
template <bool kPair, bool kSplit = false, bool kHalf = false>
struct ECfg {
  static constexpr int STAGES = kSplit ? 2 : kPair ? 4 : 3;
  static constexpr int B_ROWS = kPair ? kBN / 2 : kBN;
  static constexpr int HALF = kA + B_ROWS * 128;  // the hi (or lo) operands: 128-byte rows
  static constexpr int STAGE = HALF * (kSplit ? 2 : 1);
  static constexpr int NACC = kSplit ? 1 : 2;  // split: main + correction fill TMEM
  static constexpr int BK = kHalf ? 64 : 32;   // elements per K block
  static constexpr int NKB = 512 / BK;         // K blocks per hop
};
template <bool kPair, bool kSplit = false, bool kHalf = false>
constexpr size_t egemm_smem() {
  using EC = ECfg<kPair, kSplit, kHalf>;
  return 1024 + (size_t)EC::STAGES * EC::STAGE + (size_t)4 * kRows * kRing * 4 + kBN * 2 + kRows * 4 + 16 * 8;
}

// kPair: a cluster of two CTAs of the same group runs two independent tile runs
// in lockstep with cta_group::2 MMAs (M = 256: each CTA's A tile, the group's
// B columns split between them), ~25 % more MMA throughput per SM; each CTA's
// epilogue and D rings stay its own.
// kSplit (3xTF32, FP32-accurate): E = A_hi B_hi (main accumulator) +
// (A_hi B_lo + A_lo B_hi) (correction accumulator), summed in the epilogue.
template <bool kPair, bool kSplit = false, bool kHalf = false>
__global__ void __launch_bounds__(kThreads, 1)
    cqt1992_egemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                         const __grid_constant__ CUtensorMap tm_a_lo, const __grid_constant__ CUtensorMap tm_b_lo,
                         const EParams p) {
  using EC = ECfg<kPair, kSplit, kHalf>;
  constexpr int kBK = EC::BK;
  static_assert(!kSplit || kPair, "3xTF32 E-GEMM runs as CTA pairs");
  constexpr int NACC = EC::NACC;
  constexpr int kStages = EC::STAGES, kStage = EC::STAGE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* ring = reinterpret_cast<float*>(smem + kStages * kStage);  // [4 warps][kRows][kRing]
  uint16_t* cols = reinterpret_cast<uint16_t*>(ring + 4 * kRows * kRing);  // [kBN], 16-byte aligned
  int32_t* rows = reinterpret_cast<int32_t*>(cols + kBN);
  uint64_t* bars = reinterpret_cast<uint64_t*>(rows + kRows);  // 8-byte aligned: 512 + 256 bytes above
  uint64_t* full = bars;            // [kStages]
  uint64_t* empty = bars + 4;       // [kStages]
  uint64_t* tfull = bars + 8;       // [2]
  uint64_t* tempty = bars + 10;     // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0;
  const int g = blockIdx.x / p.ctas_per_group, gi = blockIdx.x % p.ctas_per_group;  // pairs: consecutive CTAs
  const bool active = g < p.n_groups;
  // this CTA's run of M tiles, plus one extra tile past it.  A pair runs both of
  // its runs in lockstep, so it always walks per + 1 tiles (tiles past the data
  // are zero-filled by TMA and emit nothing).
  const int per = (p.n_mtiles + p.ctas_per_group - 1) / p.ctas_per_group;
  const int m_a = kPair ? gi * per : min(p.n_mtiles, gi * per);
  const int m_b = kPair ? m_a + per : min(p.n_mtiles, m_a + per);
  const int m_end = kPair ? m_b + 1 : min(p.n_mtiles, m_b + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kPair ? 16 : 8);  // one per epilogue warp (pair: of both CTAs)
    }
    fence_barrier_init();
  }
  if (kPair) cluster_sync();
  if (warp == 2) {
    if (kPair) tmem_alloc_pair<512>(tslot);
    else tmem_alloc<512>(tslot);
  }
  for (int i = threadIdx.x; i < 4 * kRows * kRing; i += kThreads) ring[i] = 0.f;
  if (active) {
    for (int i = threadIdx.x; i < kBN; i += kThreads) cols[i] = p.col_table[g * kBN + i];
    for (int i = threadIdx.x; i < kRows; i += kThreads) rows[i] = p.group_rows[g * kRows + i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (active && m_a < m_b) {
    if (warp == 0) {
      // -------------------------------------------------------------- TMA producer
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        int s = 0;
        uint32_t ph = 0;
        for (int m = m_a; m < m_end; ++m)
          for (int kb = 0; kb < EC::NKB; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = smem + s * kStage;
            if (kPair) {  // both CTAs' bytes complete on the leader's barrier
              const uint32_t fb = mapa(&full[s], 0);
              if (rank == 0) mbar_expect_tx(&full[s], 2 * kStage);
              tma_load_2d_pair(st, &tm_a, fb, kb * kBK, m * kBM, keep);
              tma_load_2d_pair(st + kA, &tm_b, fb, kb * kBK, g * kBN + (int)rank * EC::B_ROWS, keep);
              if (kSplit) {
                tma_load_2d_pair(st + EC::HALF, &tm_a_lo, fb, kb * kBK, m * kBM, keep);
                tma_load_2d_pair(st + EC::HALF + kA, &tm_b_lo, fb, kb * kBK, g * kBN + (int)rank * EC::B_ROWS,
                                 keep);
              }
            } else {
              mbar_expect_tx(&full[s], kStage);
              tma_load_2d_hint(st, &tm_a, &full[s], kb * kBK, m * kBM, keep);
              tma_load_2d_hint(st + kA, &tm_b, &full[s], kb * kBK, g * kBN, keep);
            }
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
      }
      __syncwarp();
    } else if (warp == 1) {
      // -------------------------------------------------------------- MMA issuer
      if (rank == 0 && elect_one()) {
        constexpr uint32_t idesc = kHalf ? idesc_f16(kPair ? 2 * kBM : kBM, kBN) : idesc_tf32(kPair ? 2 * kBM : kBM, kBN);
        int s = 0, acc = 0;
        uint32_t ph = 0, aph = 0;
        for (int m = m_a; m < m_end; ++m) {
          mbar_wait(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + acc * kBN;
          for (int kb = 0; kb < EC::NKB; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            uint8_t* st = smem + s * kStage;
            const uint64_t a = sdesc(st), b = sdesc(st + kA);
            const uint64_t a_lo = sdesc(st + EC::HALF), b_lo = sdesc(st + EC::HALF + kA);
            auto mma = [&](uint32_t dd, uint64_t aa, uint64_t bb, uint32_t acc_) {
              if (kHalf) {
                if (kPair) mma_f16_pair(dd, aa, bb, idesc, acc_);
                else mma_f16(dd, aa, bb, idesc, acc_);
              } else {
                if (kPair) mma_tf32_pair(dd, aa, bb, idesc, acc_);
                else mma_tf32(dd, aa, bb, idesc, acc_);
              }
            };
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 MMAs of 32 bytes of K per 128-byte K block
              mma(d, a + 2 * k, b + 2 * k, (kb | k) != 0);
              if (kSplit) {
                mma(d + kBN, a + 2 * k, b_lo + 2 * k, (kb | k) != 0);
                mma(d + kBN, a_lo + 2 * k, b + 2 * k, 1u);
              }
            }
            if (kPair) mma_commit_pair(&empty[s], 0x3);
            else mma_commit(&empty[s]);
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
          if (kPair) mma_commit_pair(&tfull[acc], 0x3);
          else mma_commit(&tfull[acc]);
          if (++acc == NACC) {
            acc = 0;
            aph ^= 1;
          }
        }
      }
      __syncwarp();
    } else if (warp >= 4) {
      // -------------------------------------------------------------- epilogue
      // Thread = E row s (TMEM lane).  Column (row, r) of E[s] belongs to
      // D[s - r][row]: each warp adds its 32 rows' values into its own ring of
      // D rows (ring[q][row][d & 255]); for one column the 32 lanes hit 32
      // consecutive D rows, so every add is a conflict-free shared-memory RMW
      // and no two threads ever touch the same element (no atomics).  Rows that
      // can receive nothing more are summed over the four rings and emitted.
      // Two warps per TMEM lane quarter: part 0 takes the windows of even bank rows (Re),
      // part 1 those of odd rows (Im), so no two warps ever update the same ring row.
      const int q = (warp - 4) & 3, part = (warp - 4) >> 2, et = threadIdx.x - 128;  // et: 0 .. 255
      float* myring = ring + q * (kRows * kRing);
      int acc = 0;
      uint32_t aph = 0;
      const int64_t own = (int64_t)m_a * kBM;  // D rows from here on are this CTA's to emit
      int n_gbins = 0;                          // bins of this group (rows are filled front to back)
      while (n_gbins < kRows / 2 && rows[2 * n_gbins] >= 0) ++n_gbins;
      int n_cols = 0;
      while (n_cols < kBN && cols[n_cols] != kUnused) ++n_cols;
      int64_t done = own - p.r_max;  // ring rows below this are cleared
      for (int m = m_a; m < m_end; ++m) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * kBN;
        const int s_row = m * kBM + q * 32 + lane;  // this thread's E row (global slot)
        // The plan lays each bank row's columns out as whole windows of 16
        // consecutive r (zero-weight padding past the support).  Column k of a
        // window (row, r0 + k): lane l gathers E[s_l + k][k] from lane (l + k) mod
        // 32 -- pairs whose source lane did not wrap all belong to D row s_l - r0,
        // the wrapped ones to s_l - 32 - r0 -- so a window costs 16 shuffles and
        // two read-modify-writes per lane, cells distinct across lanes.
#pragma unroll 1
        for (int c0 = 0; c0 < n_cols; c0 += 16) {
          const uint32_t meta = cols[c0];  // warp-uniform
          if (((meta >> 8) & 1) != (uint32_t)part) continue;
          float v[16];
          tmem_ld16(ta + c0, v);
          if (kSplit) {
            float u[16];
            tmem_ld16(ta + kBN + c0, u);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += u[j];
          } else {
            tmem_ld_wait();
          }
          const int r0 = (int)(meta & 0xFF);
          float* rrow = myring + (meta >> 8) * kRing;
          float h4[4] = {0.f, 0.f, 0.f, 0.f}, l4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 chains: ILP over the adds
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const float x = __shfl_sync(0xffffffffu, v[k], (lane + k) & 31);
            if (lane + k < 32) h4[k & 3] += x;
            else l4[k & 3] += x;
          }
          const float hi = (h4[0] + h4[1]) + (h4[2] + h4[3]), lo = (l4[0] + l4[1]) + (l4[2] + l4[3]);
          rrow[(s_row - r0) & (kRing - 1)] += hi;
          rrow[(s_row - 32 - r0) & (kRing - 1)] += lo;
          __syncwarp();  // the next window's cells overlap other lanes' cells of this one
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kPair) mbar_arrive_cluster(mapa(&tempty[acc], 0));
          else mbar_arrive(&tempty[acc]);
        }
        if (++acc == NACC) {
          acc = 0;
          aph ^= 1;
        }
        ep_sync();
        // D rows < limit can receive nothing more: emit the CTA's own ones, clear the rings
        const int64_t limit = m + 1 == m_end ? (int64_t)m_b * kBM : (int64_t)(m + 1) * kBM - p.r_max;
        const int n_d = (int)(limit - done);
        for (int dd = et; dd < n_d; dd += kEpi) {  // consecutive threads: consecutive t
          const int64_t d = done + dd;
          const int b = (int)(d / p.R), t = (int)(d - (int64_t)b * p.R);
          const bool emit = d >= own && b < p.B && t < p.T;  // else: partial sums of another CTA's rows
          const int slot = (int)(d & (kRing - 1));
          const float osc = (kHalf && emit) ? ldexpf(1.f, -(__ldg(p.a_exp + b) + __ldg(p.b_exp))) : 1.f;
          for (int bl = 0; bl < n_gbins; ++bl) {
            float re = 0.f, im = 0.f;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              float* pre = ring + w * (kRows * kRing) + (2 * bl) * kRing + slot;
              re += pre[0];
              im += pre[kRing];
              pre[0] = 0.f;
              pre[kRing] = 0.f;
            }
            if (!emit) continue;
            re *= osc;
            im *= osc;
            const int64_t o = ((int64_t)b * p.n_bins + (rows[2 * bl] >> 1)) * (int64_t)p.T + t;
            if (p.out_kind == NNAB_OUT_COMPLEX) {
              reinterpret_cast<float2*>(p.out)[o] = make_float2(re, im);
            } else {
              const float pw = fmaf(re, re, im * im);
              p.out[o] = p.out_kind == NNAB_OUT_POWER       ? pw
                         : p.out_kind == NNAB_OUT_SMOOTH_MAG ? fast_sqrt(pw + p.eps)
                                                             : fast_sqrt(pw);
            }
          }
        }
        done = limit;
        ep_sync();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();  // the leader's MMAs write the peer's TMEM until the end
  tc_fence_after();
  if (warp == 2) {
    if (kPair) tmem_dealloc_pair<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

__global__ void pack_egemm_kernel(const float* __restrict__ k_re, const float* __restrict__ k_im, int32_t width,
                                  int32_t hop, const uint16_t* __restrict__ col_table,
                                  const int32_t* __restrict__ group_rows, int32_t n_groups, int32_t split,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = (int64_t)n_groups * kBN * hop;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = e / hop;
    const int c = (int)(e - col * hop);
    const int g = (int)(col / kBN);
    const uint16_t meta = col_table[col];
    float v = 0.f;
    if (meta != kUnused) {
      const int row = group_rows[g * kRows + (meta >> 8)];
      const int64_t k = (int64_t)(meta & 0xFF) * hop + c;
      if (row >= 0 && k < width) v = ((row & 1) ? k_im : k_re)[(int64_t)(row >> 1) * width + k];
    }
    const float h = tf32_rne(v);
    hi[e] = h;
    if (split) lo[e] = tf32_rne(v - h);
  }
}

// Peak |value| over the E-GEMM bank's columns (ordered bits of a non-negative float)
__global__ void egemm_absmax_kernel(const float* __restrict__ k_re, const float* __restrict__ k_im, int32_t width,
                                    int32_t hop, const uint16_t* __restrict__ col_table,
                                    const int32_t* __restrict__ group_rows, int32_t n_groups,
                                    unsigned int* __restrict__ out) {
  const int64_t total = (int64_t)n_groups * kBN * hop;
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / hop;
    const int c = (int)(i - col * hop);
    const uint16_t meta = col_table[col];
    if (meta == kUnused) continue;
    const int row = group_rows[(int)(col / kBN) * kRows + (meta >> 8)];
    const int64_t k = (int64_t)(meta & 0xFF) * hop + c;
    if (row >= 0 && k < width) m = fmaxf(m, fabsf(((row & 1) ? k_im : k_re)[(int64_t)(row >> 1) * width + k]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

// FP16 E-GEMM bank: the same columns scaled by 2^e_h (trailer[1], from the bank peak in trailer[0])
__global__ void pack_egemm_f16_kernel(const float* __restrict__ k_re, const float* __restrict__ k_im, int32_t width,
                                      int32_t hop, const uint16_t* __restrict__ col_table,
                                      const int32_t* __restrict__ group_rows, int32_t n_groups, int32_t split,
                                      __half* __restrict__ hi, __half* __restrict__ lo, int32_t* __restrict__ trailer) {
  const float pk = __uint_as_float(static_cast<unsigned int>(trailer[0]));
  int ex = 0;
  if (pk > 0.f && pk < INFINITY) frexpf(pk, &ex);
  const int e = pk > 0.f ? max(-100, min(100, 15 - ex)) : 0;
  const float sc = ldexpf(1.f, e);
  if (blockIdx.x == 0 && threadIdx.x == 0) trailer[1] = e;
  const int64_t total = (int64_t)n_groups * kBN * hop;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / hop;
    const int c = (int)(i - col * hop);
    const int g = (int)(col / kBN);
    const uint16_t meta = col_table[col];
    float v = 0.f;
    if (meta != kUnused) {
      const int row = group_rows[g * kRows + (meta >> 8)];
      const int64_t k = (int64_t)(meta & 0xFF) * hop + c;
      if (row >= 0 && k < width) v = ((row & 1) ? k_im : k_re)[(int64_t)(row >> 1) * width + k];
    }
    v *= sc;
    const __half h = __float2half_rn(v);
    hi[i] = h;
    if (split) lo[i] = __float2half_rn(v - __half2float(h));
  }
}

}  // namespace

}  // namespace nnab

using namespace nnab;

// Host only.  support[2*bin], support[2*bin+1]: the row's non-zero column range.
// Packs the (row, r) columns of whole bins into groups (<= 256 columns,
// <= 64 rows), longest bins first, columns sorted by (row, r) inside a group.
extern "C" int nnab_cqt_egemm_plan(const int32_t* support, int32_t n_bins, int32_t width, int32_t hop,
                                   int32_t max_groups, uint16_t* col_table, int32_t* group_rows, uint32_t* run_table,
                                   int32_t* n_groups, int32_t* r_max) {
  if (!support || !col_table || !group_rows || !run_table || !n_groups || !r_max || n_bins < 1 || width < 1 ||
      hop < 1)
    return NNAB_EINVAL;
  struct Bin {
    int bin, r0, r1;  // hop blocks [r0, r1]
  };
  std::vector<Bin> bins;
  int rmax = 0;
  for (int b = 0; b < n_bins; ++b) {
    int k0 = support[2 * b], k1 = support[2 * b + 1];
    if (k0 >= k1) {  // all-zero row: keep one column so the bin still gets an output
      k0 = 0;
      k1 = 1;
    }
    Bin x{b, k0 / hop, (k1 - 1) / hop};
    x.r1 = x.r0 + (x.r1 - x.r0 + kWin) / kWin * kWin - 1;  // whole 16-column windows (zero-weight tail)
    if (x.r1 > 254) return NNAB_ENOTSUP;
    rmax = std::max(rmax, x.r1);
    bins.push_back(x);
  }
  if (rmax + kBM > kRing) return NNAB_ENOTSUP;  // the D ring must hold a tile + its reach
  std::stable_sort(bins.begin(), bins.end(), [](const Bin& a, const Bin& b) { return a.r1 - a.r0 > b.r1 - b.r0; });
  std::vector<std::vector<Bin>> groups;
  std::vector<int> used_cols;
  for (const Bin& x : bins) {
    const int need = 2 * (x.r1 - x.r0 + 1);
    if (need > kBN) return NNAB_ENOTSUP;
    size_t gi = 0;
    for (; gi < groups.size(); ++gi)
      if (used_cols[gi] + need <= kBN && (int)groups[gi].size() < kRows / 2) break;
    if (gi == groups.size()) {
      groups.push_back({});
      used_cols.push_back(0);
    }
    groups[gi].push_back(x);
    used_cols[gi] += need;
  }
  if ((int)groups.size() > max_groups) return NNAB_ENOTSUP;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    std::vector<std::pair<int, int>> cl;  // (row_local, r), row-major: the epilogue sums row runs
    for (size_t k = 0; k < groups[gi].size(); ++k) {
      const Bin& x = groups[gi][k];
      group_rows[gi * kRows + 2 * k] = 2 * x.bin;
      group_rows[gi * kRows + 2 * k + 1] = 2 * x.bin + 1;
      for (int ri = 0; ri < 2; ++ri)
        for (int r = x.r0; r <= x.r1; ++r) cl.push_back({(int)(2 * k + ri), r});
    }
    for (size_t k = 2 * groups[gi].size(); k < (size_t)kRows; ++k) group_rows[gi * kRows + k] = -1;
    for (int j = 0; j < kBN; ++j)
      col_table[gi * kBN + j] = j < (int)cl.size() ? (uint16_t)((cl[j].first << 8) | cl[j].second) : kUnused;
    // runs per 64-column chunk: row_local | j0 << 8 | n << 14 | r0 << 21
    for (int c = 0; c < kChunks; ++c) {
      uint32_t* t = run_table + ((size_t)gi * kChunks + c) * kRunSlots;
      int cnt = 0;
      for (int j = c * kChunk; j < (c + 1) * kChunk && j < (int)cl.size();) {
        int e = j + 1;
        while (e < (c + 1) * kChunk && e < (int)cl.size() && cl[e].first == cl[j].first) ++e;
        t[1 + cnt++] = (uint32_t)cl[j].first | (uint32_t)(j - c * kChunk) << 8 | (uint32_t)(e - j) << 14 |
                       (uint32_t)cl[j].second << 21;
        j = e;
      }
      t[0] = (uint32_t)cnt;
    }
  }
  *n_groups = (int32_t)groups.size();
  *r_max = rmax;
  return NNAB_OK;
}

extern "C" size_t nnab_cqt_egemm_bank_bytes(int32_t n_groups, int32_t hop) {
  return (size_t)std::max(0, n_groups) * kBN * std::max(0, hop) * sizeof(float);
}

extern "C" size_t nnab_cqt_egemm_bank_bytes_prec(int32_t n_groups, int32_t hop, int32_t precision) {
  if (!prec_is_f16(precision)) return nnab_cqt_egemm_bank_bytes(n_groups, hop);
  const size_t data = (size_t)std::max(0, n_groups) * kBN * std::max(0, hop) * 2;
  return ((data + 255) & ~size_t(255)) + 256;  // + trailer: [0] peak bits, [1] scale exponent
}

// Device tables (col_table, group_rows as produced by nnab_cqt_egemm_plan).
extern "C" int nnab_pack_cqt_egemm(const float* k_re, const float* k_im, int32_t width, int32_t hop,
                                   const uint16_t* col_table, const int32_t* group_rows, int32_t n_groups,
                                   int32_t precision, float* packed_hi, float* packed_lo, void* stream) {
  if (!k_re || !k_im || !col_table || !group_rows || !packed_hi || n_groups < 1 || width < 1 || hop < 1)
    return NNAB_EINVAL;
  if (!prec_valid(precision)) return NNAB_EINVAL;
  const int split = prec_is_split(precision);
  if (split && !packed_lo) return NNAB_EINVAL;
  const int64_t total = (int64_t)n_groups * kBN * hop;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8192);
  cudaStream_t s = (cudaStream_t)stream;
  if (prec_is_f16(precision)) {
    int32_t* trailer = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(packed_hi) +
                                                  nnab_cqt_egemm_bank_bytes_prec(n_groups, hop, precision) - 256);
    NNAB_CUDA_TRY(cudaMemsetAsync(trailer, 0, 8, s));
    egemm_absmax_kernel<<<blocks, 256, 0, s>>>(k_re, k_im, width, hop, col_table, group_rows, n_groups,
                                               reinterpret_cast<unsigned int*>(trailer));
    NNAB_LAUNCHED();
    pack_egemm_f16_kernel<<<blocks, 256, 0, s>>>(k_re, k_im, width, hop, col_table, group_rows, n_groups, split,
                                                 reinterpret_cast<__half*>(packed_hi),
                                                 reinterpret_cast<__half*>(packed_lo), trailer);
    NNAB_LAUNCHED();
    return NNAB_OK;
  }
  pack_egemm_kernel<<<blocks, 256, 0, s>>>(k_re, k_im, width, hop, col_table, group_rows, n_groups, split,
                                           packed_hi, packed_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

namespace nnab {
int cqt_schedule_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo, int32_t n_bins,
                        const uint32_t* schedule, int32_t n_entries, int32_t precision, int32_t out_kind, float eps,
                        float* out, int32_t out_bins, const void* workspace, size_t workspace_bytes,
                        cudaStream_t s);

// E-GEMM on staged frames (TF32): the group tables' bins are written into an
// output of out_bins bins per clip (group_rows hold global bank rows).
static int cqt_egemm_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo,
                            const uint16_t* col_table, const int32_t* group_rows, int32_t n_groups, int32_t r_max,
                            int32_t out_bins, int32_t out_kind, float eps, float* out, const void* workspace,
                            size_t workspace_bytes, int32_t precision, cudaStream_t stream) {
  if (!prec_valid(precision)) return NNAB_EINVAL;
  const bool split = prec_is_split(precision), half = prec_is_f16(precision);
  FrameGeom g;
  const void *rows_hi, *rows_lo;
  const int32_t* exps;
  int rc = staged_views(f, precision, workspace, workspace_bytes, &g, &rows_hi, &rows_lo, &exps);
  if (rc) return rc;
  if (!packed_hi || (split && !packed_lo) || !col_table || !group_rows || !out || n_groups < 1 || out_bins < 1)
    return NNAB_EINVAL;
  if (r_max < 0 || r_max + kBM > kRing) return NNAB_EINVAL;
  const int bk = half ? 64 : 32;  // elements per 128-byte K block
  if (g.row_len != g.hop || g.hop != 512) return NNAB_ENOTSUP;  // K = hop = 512
  if (out_kind != NNAB_OUT_MAGNITUDE && out_kind != NNAB_OUT_POWER && out_kind != NNAB_OUT_COMPLEX &&
      out_kind != NNAB_OUT_SMOOTH_MAG)
    return NNAB_EINVAL;
  if (g.B == 0) return NNAB_OK;
  const int nsm = num_sms();
  if (n_groups > nsm) return NNAB_ENOTSUP;
  static const bool pair_ok = [] {
    const char* e = getenv("NNAB_EGEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  const bool pair = (pair_ok || split || half) && nsm / n_groups >= 2;
  if ((split || half) && !pair) return NNAB_ENOTSUP;  // split and FP16 modes run as CTA pairs only
  CUtensorMap ta, tb, ta_lo, tb_lo;
  const uint64_t rows_total = (uint64_t)g.B * g.R;
  const int b_box = pair ? kBN / 2 : kBN;
  const int E = half ? 2 : 4;
  rc = make_tmap_2d(&ta, rows_hi, g.row_len, rows_total, (uint64_t)g.row_len * E, bk, kBM, 128, E);
  if (!rc) rc = make_tmap_2d(&tb, packed_hi, g.hop, (uint64_t)n_groups * kBN, (uint64_t)g.hop * E, bk, b_box, 128, E);
  if (!rc && split) {
    rc = make_tmap_2d(&ta_lo, rows_lo, g.row_len, rows_total, (uint64_t)g.row_len * E, bk, kBM, 128, E);
    if (!rc)
      rc = make_tmap_2d(&tb_lo, packed_lo, g.hop, (uint64_t)n_groups * kBN, (uint64_t)g.hop * E, bk, b_box, 128, E);
  }
  if (rc) return rc;
  if (!split) {
    ta_lo = ta;
    tb_lo = tb;
  }
  EParams p{};
  p.B = g.B;
  p.R = g.R;
  p.T = g.T;
  p.n_mtiles = (int32_t)((rows_total + kBM - 1) / kBM);
  p.n_bins = out_bins;
  p.out_kind = out_kind;
  p.n_groups = n_groups;
  p.ctas_per_group = pair ? nsm / n_groups / 2 * 2 : nsm / n_groups;
  p.r_max = r_max;
  p.eps = eps;
  p.col_table = col_table;
  p.group_rows = group_rows;
  p.out = out;
  p.a_exp = exps;
  if (half)
    p.b_exp = reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(packed_hi) +
                                               nnab_cqt_egemm_bank_bytes_prec(n_groups, g.hop, precision) - 256) + 1;
  const int grid = p.ctas_per_group * n_groups;
  if (!pair) {
    const size_t smem = egemm_smem<false>();
    NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt1992_egemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    cqt1992_egemm_kernel<false><<<grid, kThreads, smem, stream>>>(ta, tb, ta_lo, tb_lo, p);
  } else {
    auto kern = half ? (split ? cqt1992_egemm_kernel<true, true, true> : cqt1992_egemm_kernel<true, false, true>)
                     : (split ? cqt1992_egemm_kernel<true, true> : cqt1992_egemm_kernel<true, false>);
    const size_t smem = half ? (split ? egemm_smem<true, true, true>() : egemm_smem<true, false, true>())
                             : (split ? egemm_smem<true, true>() : egemm_smem<true, false>());
    NNAB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    NNAB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, ta_lo, tb_lo, p));
  }
  NNAB_LAUNCHED();
  return NNAB_OK;
}
}  // namespace nnab

// E-GEMM forward on frames staged by nnab_stage_frames (TF32 only).  run_table
// is reserved (the plan still emits it; the kernel reads col_table only).
extern "C" int nnab_cqt1992v2_egemm_staged(const nnab_frames* f, const float* packed_hi, const uint16_t* col_table,
                                           const int32_t* group_rows, const uint32_t* run_table,
                                           int32_t n_groups, int32_t r_max,
                                           int32_t n_bins, int32_t out_kind, float eps, float* out,
                                           const void* workspace, size_t workspace_bytes, void* stream) {
  (void)run_table;
  if (n_bins < 1) return NNAB_EINVAL;
  return cqt_egemm_staged(f, packed_hi, nullptr, col_table, group_rows, n_groups, r_max, n_bins, out_kind, eps, out,
                          workspace, workspace_bytes, NNAB_PREC_TF32, (cudaStream_t)stream);
}

// CQT1992v2 hybrid on staged frames (TF32): bins [0, n_long) -- the long,
// low-frequency kernels -- on the E-GEMM (tables from nnab_cqt_egemm_plan over
// those bins), bins [n_long, n_bins) on the per-K-block schedule (bank and
// schedule of those rows at the full width, so both share the staged frames).
extern "C" int nnab_cqt1992v2_hybrid_staged(const nnab_frames* f, const float* eg_bank, const float* eg_bank_lo,
                                            const uint16_t* col_table, const int32_t* group_rows, int32_t n_groups,
                                            int32_t r_max, const float* sched_bank, const float* sched_bank_lo,
                                            const uint32_t* schedule, int32_t n_entries, int32_t n_long,
                                            int32_t n_bins, int32_t precision, int32_t out_kind, float eps,
                                            float* out, const void* workspace, size_t workspace_bytes, void* stream) {
  if (n_long < 0 || n_long > n_bins || n_bins < 1 || !out) return NNAB_EINVAL;
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_long > 0) {
    rc = cqt_egemm_staged(f, eg_bank, eg_bank_lo, col_table, group_rows, n_groups, r_max, n_bins, out_kind, eps, out,
                          workspace, workspace_bytes, precision, s);
    if (rc) return rc;
  }
  if (n_long < n_bins) {
    float* o = out + (int64_t)n_long * g.T * (out_kind == NNAB_OUT_COMPLEX ? 2 : 1);
    rc = cqt_schedule_staged(f, sched_bank, sched_bank_lo, n_bins - n_long, schedule, n_entries, precision, out_kind,
                             eps, o, n_bins, workspace, workspace_bytes, s);
  }
  return rc;
}

extern "C" int nnab_cqt1992v2_hybrid_forward(const nnab_frames* f, const float* x, const float* eg_bank,
                                             const float* eg_bank_lo, const uint16_t* col_table,
                                             const int32_t* group_rows, int32_t n_groups, int32_t r_max,
                                             const float* sched_bank, const float* sched_bank_lo,
                                             const uint32_t* schedule, int32_t n_entries, int32_t n_long,
                                             int32_t n_bins, int32_t precision, int32_t out_kind, float eps,
                                             float* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!x) return NNAB_EINVAL;
  int rc = nnab_stage_frames(f, x, precision, workspace, workspace_bytes, stream);
  if (rc) return rc;
  return nnab_cqt1992v2_hybrid_staged(f, eg_bank, eg_bank_lo, col_table, group_rows, n_groups, r_max, sched_bank,
                                      sched_bank_lo, schedule, n_entries, n_long, n_bins, precision, out_kind, eps,
                                      out, workspace, workspace_bytes, stream);
}
