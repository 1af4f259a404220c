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
// Status (round 1): correct (tests/test_gpu_cqt.py) and its GEMM alone runs the
// 1,770-clip batch in 0.95 ms, but the diagonal-sum epilogue (~30k cycles per
// tile, mostly TMEM->smem staging and the short-bin groups' many runs) does not
// yet keep up with the MMAs (11k cycles per tile), so the engine's default stays
// the per-K-block schedule (CqtLongEngine(method="schedule")).  Next: E-GEMM for
// the long bins only (few long runs), the schedule for the short ones.
//
// Columns are packed into groups of <= 256 columns / <= 64 rows (whole bins,
// re and im together), sorted by (row, r) inside a group.  A persistent CTA owns
// one group and a contiguous run of M tiles (128 hop rows each): TMA producer
// warp, single-thread tcgen05.mma issuer (M = 128, N = 256, K = 8, TF32), and
// 4 epilogue warps that stage each E tile through shared memory 32 columns at a
// time and fold it into a ring of D rows (D[row][d & 255]); each D element has
// one owner thread per pass, so the sum needs no atomics and is deterministic.  D rows
// that can receive nothing more are turned into magnitude / power / complex
// and written to the (B, n_bins, T) output, coalesced along T.  Each CTA also
// computes the first tile past its run (a 1-in-~150 overlap) so its last D rows
// are complete; D rows before its run belong to the previous CTA.
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 32, kThreads = 256;
constexpr int kStages = 3;
constexpr int kA = kBM * kBK * 4, kB = kBN * kBK * 4, kStage = kA + kB;  // 16 + 32 KB
constexpr int kRows = 64;   // D rows (bank rows: 2 per bin) per group
constexpr int kChunk = 64;  // E columns staged in shared memory per reduction pass
constexpr int kEB = kBM;  // staged E row stride (floats): writes and diagonal reads are both lane-consecutive
constexpr int kRing = 192;  // D ring length (slots); >= 128 + max r
constexpr uint16_t kUnused = 0xFFFF;

constexpr int kChunks = kBN / kChunk;
constexpr int kRunSlots = kChunk + 1;  // per chunk: count, then up to 64 runs
constexpr int kEpi = 192;  // warps 2-7 reduce; warps 4-7 also read TMEM

struct EParams {
  int64_t B;
  int32_t R, T, n_mtiles, n_bins, out_kind;
  int32_t n_groups, ctas_per_group, r_max;
  float eps;
  const uint16_t* col_table;  // [n_groups][256]: row_local << 8 | r
  const uint32_t* run_table;  // [n_groups][kChunks][kRunSlots]: count, runs (see nnab_cqt_egemm_plan)
  const int32_t* group_rows;  // [n_groups][64]: bank row 2*bin + im, -1 unused
  float* out;
};

NNAB_DEV uint64_t sdesc(const void* p) {  // K-major, 128-byte swizzle, 8-row atoms
  uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

NNAB_DEV void ep_sync() { asm volatile("bar.sync 1, 192;" ::: "memory"); }  // epilogue warps 2-7
// ring slot of D row d (d >= -64): rows are offset by one ring length to stay non-negative
NNAB_DEV int ring_slot(int64_t d) { return (int)((uint32_t)(d + kRing) % (uint32_t)kRing); }

__global__ void __launch_bounds__(kThreads, 1)
    cqt1992_egemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                         const EParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* ring = reinterpret_cast<float*>(smem + kStages * kStage);  // [kRows][kRing]
  float* ebuf = ring + kRows * kRing;                                // [kChunk][kEB]
  uint32_t* runs = reinterpret_cast<uint32_t*>(ebuf + kChunk * kEB);  // [kChunks][kRunSlots]
  uint16_t* cols = reinterpret_cast<uint16_t*>(runs + kChunks * kRunSlots);
  int32_t* rows = reinterpret_cast<int32_t*>(cols + kBN);
  uint64_t* bars = reinterpret_cast<uint64_t*>(rows + kRows);  // 8-byte aligned: 512 + 256 bytes above
  uint64_t* full = bars;            // [kStages]
  uint64_t* empty = bars + 4;       // [kStages]
  uint64_t* tfull = bars + 8;       // [2]
  uint64_t* tempty = bars + 10;     // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x / p.ctas_per_group, gi = blockIdx.x % p.ctas_per_group;
  const bool active = g < p.n_groups;
  // this CTA's run of M tiles, plus one extra tile past it
  const int per = (p.n_mtiles + p.ctas_per_group - 1) / p.ctas_per_group;
  const int m_a = min(p.n_mtiles, gi * per), m_b = min(p.n_mtiles, m_a + per);
  const int m_end = min(p.n_mtiles, m_b + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  for (int i = threadIdx.x; i < kRows * kRing; i += kThreads) ring[i] = 0.f;
  if (active) {
    for (int i = threadIdx.x; i < kBN; i += kThreads) cols[i] = p.col_table[g * kBN + i];
    for (int i = threadIdx.x; i < kChunks * kRunSlots; i += kThreads) runs[i] = p.run_table[g * kChunks * kRunSlots + i];
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
          for (int kb = 0; kb < 16; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = smem + s * kStage;
            mbar_expect_tx(&full[s], kStage);
            tma_load_2d_hint(st, &tm_a, &full[s], kb * kBK, m * kBM, keep);
            tma_load_2d_hint(st + kA, &tm_b, &full[s], kb * kBK, g * kBN, keep);
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
      }
      __syncwarp();
    } else if (warp == 1) {
      // -------------------------------------------------------------- MMA issuer
      if (elect_one()) {
        constexpr uint32_t idesc = idesc_tf32(kBM, kBN);
        int s = 0, acc = 0;
        uint32_t ph = 0, aph = 0;
        for (int m = m_a; m < m_end; ++m) {
          mbar_wait(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + acc * kBN;
          for (int kb = 0; kb < 16; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            uint8_t* st = smem + s * kStage;
            const uint64_t a = sdesc(st), b = sdesc(st + kA);
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) mma_tf32(d, a + 2 * k, b + 2 * k, idesc, (kb | k) != 0);
            mma_commit(&empty[s]);
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
          mma_commit(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            aph ^= 1;
          }
        }
      }
      __syncwarp();
    } else if (warp >= 2) {
      // -------------------------------------------------------------- epilogue
      const bool tm = warp >= 4;  // TMEM readers (lane quarter warp - 4)
      const int q = warp & 3, row_in_tile = q * 32 + lane;
      int acc = 0;
      uint32_t aph = 0;
      const int64_t own = (int64_t)m_a * kBM;  // D rows from here on are this CTA's to emit
      int n_gbins = 0;                          // bins of this group (rows are filled front to back)
      while (n_gbins < kRows / 2 && rows[2 * n_gbins] >= 0) ++n_gbins;
      int64_t done = own - p.r_max;             // ring rows below this are cleared
      for (int m = m_a; m < m_end; ++m) {
        if (tm) {
          mbar_wait(&tfull[acc], aph);
          tc_fence_after();
        }
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * kBN;
        // D[row][d] += sum over the row's columns (row, r) of E[d + r][(row, r)]: E goes
        // through shared memory one 32-column chunk at a time, then thread et sums, for
        // d_local = et and et + 128 (d = 128 m - r_max + d_local), the chunk's columns
        // row by row (columns are sorted by (row, r)) and adds each row's sum into the
        // ring once -- every D element has a single owner thread, no atomics or races.
        const int et = threadIdx.x - 64;  // 0 .. 191
        const int span = kBM + p.r_max;   // D rows this tile reaches (<= kEpi: one per thread)
#pragma unroll 1
        for (int c0 = 0; c0 < kBN; c0 += kChunk) {
          if (cols[c0] == kUnused) break;  // the rest of the table is empty
          if (tm) {
#pragma unroll
            for (int h = 0; h < kChunk; h += 32) {
              float v[32];
              tmem_ld32(ta + c0 + h, v);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) ebuf[(h + j) * kEB + row_in_tile] = v[j];
            }
          }
          ep_sync();
          // run = consecutive columns of one D row with consecutive r: the row's sum for
          // D row d is a diagonal of the staged chunk (stride kEB + 1), summed with 4
          // independent accumulators over the in-tile range of E rows
          const uint32_t* cr = runs + (c0 / kChunk) * kRunSlots;
          const int n_runs = (int)cr[0];
#pragma unroll 1
          for (int dl = et; dl < span; dl += kEpi) {
            const int slot = ring_slot((int64_t)m * kBM - p.r_max + dl);
#pragma unroll 1
            for (int k = 0; k < n_runs; ++k) {
              const uint32_t run = cr[1 + k];
              const int rl = (int)(run & 0xFF), j0 = (int)((run >> 8) & 0x3F), n = (int)((run >> 14) & 0x7F),
                        r0 = (int)(run >> 21);
              const int sl0 = dl - p.r_max + r0;  // E row of the run's first column
              const int i0 = max(0, -sl0), i1 = min(n, kBM - sl0);
              if (i0 >= i1) continue;
              const float* e = ebuf + j0 * kEB + sl0;
              float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
              int i = i0;
              for (; i + 4 <= i1; i += 4) {
                a0 += e[i * (kEB + 1)];
                a1 += e[(i + 1) * (kEB + 1)];
                a2 += e[(i + 2) * (kEB + 1)];
                a3 += e[(i + 3) * (kEB + 1)];
              }
              for (; i < i1; ++i) a0 += e[i * (kEB + 1)];
              ring[rl * kRing + slot] += (a0 + a1) + (a2 + a3);
            }
          }
          ep_sync();
        }
        if (tm) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
        ep_sync();
        // D rows < limit can receive nothing more: emit the CTA's own ones, clear the ring
        const int64_t limit = m + 1 == m_end ? (int64_t)m_b * kBM : (int64_t)(m + 1) * kBM - p.r_max;
        const int n_d = (int)(limit - done);
        for (int dd = et; dd < n_d; dd += kEpi) {  // consecutive threads: consecutive t
          const int64_t d = done + dd;
          const int b = (int)(d / p.R), t = (int)(d - (int64_t)b * p.R);
          const bool emit = d >= own && b < p.B && t < p.T;  // else: partial sums of another CTA's rows
          const int slot = ring_slot(d);
          for (int bl = 0; bl < n_gbins; ++bl) {
            float* pre = &ring[(2 * bl) * kRing + slot];
            const float re = pre[0], im = pre[kRing];
            pre[0] = 0.f;
            pre[kRing] = 0.f;
            if (!emit) continue;
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
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
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
    const Bin x{b, k0 / hop, (k1 - 1) / hop};
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

// Device tables (col_table, group_rows as produced by nnab_cqt_egemm_plan).
extern "C" int nnab_pack_cqt_egemm(const float* k_re, const float* k_im, int32_t width, int32_t hop,
                                   const uint16_t* col_table, const int32_t* group_rows, int32_t n_groups,
                                   int32_t precision, float* packed_hi, float* packed_lo, void* stream) {
  if (!k_re || !k_im || !col_table || !group_rows || !packed_hi || n_groups < 1 || width < 1 || hop < 1)
    return NNAB_EINVAL;
  const int split = precision == NNAB_PREC_3XTF32;
  if (split && !packed_lo) return NNAB_EINVAL;
  const int64_t total = (int64_t)n_groups * kBN * hop;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8192);
  pack_egemm_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(k_re, k_im, width, hop, col_table, group_rows,
                                                              n_groups, split, packed_hi, packed_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

// E-GEMM forward on frames staged by nnab_stage_frames (TF32 only).
extern "C" int nnab_cqt1992v2_egemm_staged(const nnab_frames* f, const float* packed_hi, const uint16_t* col_table,
                                           const int32_t* group_rows, const uint32_t* run_table,
                                           int32_t n_groups, int32_t r_max,
                                           int32_t n_bins, int32_t out_kind, float eps, float* out,
                                           const void* workspace, size_t workspace_bytes, void* stream) {
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  if (!packed_hi || !col_table || !group_rows || !run_table || !out || n_groups < 1 || n_bins < 1) return NNAB_EINVAL;
  if (g.row_len != g.hop || g.hop % kBK != 0 || g.hop / kBK != 16) return NNAB_ENOTSUP;  // K = hop = 512
  if (out_kind != NNAB_OUT_MAGNITUDE && out_kind != NNAB_OUT_POWER && out_kind != NNAB_OUT_COMPLEX &&
      out_kind != NNAB_OUT_SMOOTH_MAG)
    return NNAB_EINVAL;
  if (g.B == 0) return NNAB_OK;
  if (!workspace || workspace_bytes < nnab_stft_workspace_bytes(f, NNAB_PREC_TF32)) return NNAB_EINVAL;
  const int nsm = num_sms();
  if (n_groups > nsm) return NNAB_ENOTSUP;
  CUtensorMap ta, tb;
  const uint64_t rows_total = (uint64_t)g.B * g.R;
  rc = make_tmap_2d(&ta, workspace, g.row_len, rows_total, (uint64_t)g.row_len * 4, kBK, kBM, 128);
  if (!rc) rc = make_tmap_2d(&tb, packed_hi, g.hop, (uint64_t)n_groups * kBN, (uint64_t)g.hop * 4, kBK, kBN, 128);
  if (rc) return rc;
  EParams p{};
  p.B = g.B;
  p.R = g.R;
  p.T = g.T;
  p.n_mtiles = (int32_t)((rows_total + kBM - 1) / kBM);
  p.n_bins = n_bins;
  p.out_kind = out_kind;
  p.n_groups = n_groups;
  p.ctas_per_group = nsm / n_groups;
  p.r_max = r_max;
  p.eps = eps;
  p.col_table = col_table;
  p.group_rows = group_rows;
  p.run_table = run_table;
  p.out = out;
  const size_t smem = 1024 + (size_t)kStages * kStage + (size_t)kRows * kRing * 4 + (size_t)kChunk * kEB * 4 +
                      kChunks * kRunSlots * 4 + kBN * 2 + kRows * 4 + 16 * 8;
  NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt1992_egemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cqt1992_egemm_kernel<<<p.ctas_per_group * n_groups, kThreads, smem, (cudaStream_t)stream>>>(ta, tb, p);
  NNAB_LAUNCHED();
  return NNAB_OK;
}
