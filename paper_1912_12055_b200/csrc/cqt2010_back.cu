// CQT2010v2 back end: the octave chain (halvings, cqt2010_chain.cu) and the per-octave
// complex convs (the batched conv, cqt2010_tc.cu) of a group of clips in ONE persistent
// kernel (transforms.py:300-313, signal.py:232-247), so each octave's conv reads the level
// the chain has just written while it is in L2, and the two pipelines fill each other's
// latency bubbles.  One CTA per SM, a group of ceil(B / SMs) clips per CTA.
//
//   warp 0     halving TMA producer (K-block ring, 256-sample level rows)
//   warp 1     halving MMA issue + TMEM allocation (512 columns)
//   warp 2     conv TMA producer (im2col tiles of 128 frames, the conv kernel's layouts)
//   warp 3     conv MMA issue (frames as M, bank as N = 32)
//   warps 4-7  halving epilogue: level a + 1 rows, then its reflect margins, zero tail and
//              the conv's shifted copies; arrives lvl_ready[a + 1]
//   warps 8-15 conv epilogue: two warpgroups on alternate tiles
//
// Each CTA walks SETS of kNG clip groups with their levels interleaved (group A level a,
// group B level a, group C level a, group A level a + 1, ...), so one group's level
// transition (drain, margins, barrier) hides behind the others' tiles.  Level a's conv and halving both need
// level a of that group complete (lvl_ready[group][a]; level 0 comes from the front
// kernel); the halving producer waits for the conv producer to finish the previous set,
// so no level barrier runs two phases ahead of a waiter.
#include <algorithm>
#include <cmath>

#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kML = 128;
constexpr int kMaxLv = 12;
constexpr int kThreads = 16 * 32;
constexpr int kERows = 352;        // E rows r = -224 .. 127 (halving B windows)
#ifndef NNAB_BACK_HST
#define NNAB_BACK_HST 4
#endif
#ifndef NNAB_BACK_CST
#define NNAB_BACK_CST 4
#endif
constexpr int kHStages = NNAB_BACK_HST;  // halving K-block ring (16 KB stages; 3 / 5 / 6 with 4 / 3 / 2 conv
                                         // stages: the same time, 0.316-0.324 ms)
constexpr uint32_t kKB = 16384;
constexpr int kCStages = NNAB_BACK_CST;  // conv tile ring (24 KB stages)
constexpr uint32_t kCA = 12 * 2048;
constexpr int KC = 96, NCONV = 32, kFiltLog2 = 6;
constexpr int kCMaps = 8;
constexpr uint32_t kRows8 = 128 + KC / 8 - 1;
constexpr int kMaxG = 8;     // clips per group (the margin buffers)
#ifndef NNAB_BACK_NG
#define NNAB_BACK_NG 3  // 2: 0.316-0.317 ms, 3: 0.314-0.315, 4: 0.326, 6: 0.364
#endif
constexpr int kNG = NNAB_BACK_NG;  // clip groups per CTA, levels interleaved between them
constexpr int kMLeft = 160;  // margin sources kept in shared memory: outputs [0, 160) ...
constexpr int kMRight = 192; // ... and [rb, rb + 192), rb = (n - 160) rounded down to 32

struct BackParams {
  CUtensorMap hmap[kMaxLv];        // halving input: level a as rows of 256 samples
  CUtensorMap cmap[kCMaps];        // conv: per (octave, copy) [wide box, narrow box] (rs >= 64) or one
  int32_t n_oct, B, G;
  int32_t n[kMaxLv], stride[kMaxLv], R[kMaxLv], h[kMaxLv], copies[kMaxLv], U[kMaxLv], rs[kMaxLv], cmap0[kMaxLv];
  int64_t copy_stride[kMaxLv];
  __half* lv[kMaxLv];
  const __half* crows[kMaxLv];     // rs = 8: level base + the frame offset (ML - pad_al)
  float taps[255];
  int32_t T, n_bins, first_bin, bpo, n_filt, out_kind;
  const int32_t* exps;
  const uint4* filt_img;
  float* out;
  unsigned long long* prof;  // debug: per-role wait cycles, or null
};

NNAB_DEV uint64_t swz_desc(uint32_t addr, uint32_t row_bytes) {  // K-major, 32/64/128-byte swizzle
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(((8 * row_bytes) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(row_bytes == 128 ? 2 : row_bytes == 64 ? 4 : 6) << 61;
  return d;
}
NNAB_DEV uint64_t nsw_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void __launch_bounds__(kThreads, 1) cqt2010_back_kernel(const __grid_constant__ BackParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* HA = base;                             // kHStages x kKB
  uint8_t* E = HA + kHStages * kKB;               // kERows x 128 B (128-byte swizzle)
  uint8_t* CA = E + kERows * 128;                 // kCStages x kCA (1024-aligned: 45,056 + 65,536)
  uint8_t* filt = CA + kCStages * kCA;            // conv bank: 12 chunks x 32 rows x 16 B
  uint64_t* bars = reinterpret_cast<uint64_t*>(filt + KC / 8 * 512);
  uint64_t* h_full = bars;                        // [kHStages] tx
  uint64_t* h_empty = h_full + kHStages;          // [kHStages] commit
  uint64_t* hd_full = h_empty + kHStages;         // [2] commit
  uint64_t* hd_empty = hd_full + 2;               // [2] 4 warps
  uint64_t* c_full = hd_empty + 2;                // [kCStages] tx
  uint64_t* c_mma = c_full + kCStages;            // [kCStages] commit
  uint64_t* c_tfree = c_mma + kCStages;           // [kCStages] 4 warps
  uint64_t* lvl_ready = c_tfree + kCStages;       // [kNG][kMaxLv] per group of the set, 128 halving-epilogue threads
  uint64_t* cgrp_done = lvl_ready + kNG * kMaxLv; // conv producer finished a group set
  uint32_t* tslot = reinterpret_cast<uint32_t*>(cgrp_done + 1);
  int32_t* exps_s = reinterpret_cast<int32_t*>(tslot + 4);  // B ints
  __half* mbuf = reinterpret_cast<__half*>((reinterpret_cast<uintptr_t>(exps_s + p.B) + 15) & ~uintptr_t(15));  // [kMaxG][kMLeft + kMRight]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kHStages; ++i) {
      mbar_init(&h_full[i], 1);
      mbar_init(&h_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&hd_full[i], 1);
      mbar_init(&hd_empty[i], 4);
    }
    for (int i = 0; i < kCStages; ++i) {
      mbar_init(&c_full[i], 1);
      mbar_init(&c_mma[i], 1);
      mbar_init(&c_tfree[i], 4);
    }
    for (int i = 0; i < kNG * kMaxLv; ++i) mbar_init(&lvl_ready[i], 128);
    mbar_init(cgrp_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  __shared__ float taps_s[256];
  for (int j = tid; j < 256; j += kThreads) taps_s[j] = j < 255 ? p.taps[j] : 0.f;
  for (int j = tid; j < KC / 8 * 32; j += kThreads) reinterpret_cast<uint4*>(filt)[j] = __ldg(p.filt_img + j);
  for (int j = tid; j < p.B; j += kThreads) exps_s[j] = __ldg(p.exps + j);
  __syncthreads();
  for (int i = tid; i < kERows * 8; i += kThreads) {  // E[r][k'] = h[k' - 2 r - 1], one 16-byte chunk per step
    const int w = i >> 3, c = i & 7, r = w - 224;
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = 8 * c + e - 2 * r - 1;
      v[e] = __float2half_rn((j >= 0 && j < 255) ? taps_s[j] : 0.f);
    }
    *reinterpret_cast<uint4*>(E + w * 128 + ((c ^ (w & 7)) << 4)) = *reinterpret_cast<const uint4*>(v);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  unsigned long long pw[4] = {0, 0, 0, 0};
  const long long tb = clock64();
  auto W = [&](uint64_t* bar, uint32_t par, int slot) {
    const long long t0 = clock64();
    if (warp >= 4) mbar_wait(bar, par);  // epilogues spin: no wake-up latency on their critical path
    else mbar_wait_sleep(bar, par);
    pw[slot] += (unsigned long long)(clock64() - t0);
  };
  const uint32_t tmem_c = tmem + 256;  // conv accumulators: kCStages x 32 columns
  const int n_groups = (p.B + p.G - 1) / p.G;
  const int nl = p.n_oct;
  auto htiles = [&](int a, int gc) { return (gc * p.R[a] + 127) / 128; };
  auto ctiles = [&](int a, int gc) { return p.copies[a] * ((gc * p.U[a] + 127) / 128); };

  if (warp == 0) {
    // ------------------------------------------------------------ halving producer
    if (elect_one()) {
      uint32_t kq = 0;
      int gi = 0;
      for (int pr = blockIdx.x; kNG * pr < n_groups; pr += gridDim.x, ++gi) {
        if (gi > 0) W(cgrp_done, (gi - 1) & 1, 0);  // keeps lvl_ready at most one pair ahead
        for (int a = 0; a + 1 < nl; ++a)
        for (int hm = 0; hm < kNG && kNG * pr + hm < n_groups; ++hm) {
          const int b0 = (kNG * pr + hm) * p.G, gc = min(p.G, p.B - b0);
          if (a > 0) W(&lvl_ready[hm * kMaxLv + a], gi & 1, 1);
          const int R = p.R[a], nt = htiles(a, gc);
          for (int t = 0; t < nt; ++t) {
            const int row0 = b0 * R + 128 * t;
            for (int kb = 0; kb < 8; ++kb, ++kq) {
              const uint32_t s = kq % kHStages, r = kq / kHStages;
              if (r > 0) W(&h_empty[s], (r - 1) & 1, 2);
              mbar_expect_tx(&h_full[s], kKB);
              tma_load_2d(HA + s * kKB, &p.hmap[a], &h_full[s], 64 * (kb & 3), row0 + (kb >> 2));
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ halving MMA issue
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_f16(128, 128);
      const uint32_t e0 = smem_u32(E);
      uint32_t kq = 0, sq = 0;
      for (int pr = blockIdx.x; kNG * pr < n_groups; pr += gridDim.x) {
        for (int a = 0; a + 1 < nl; ++a)
        for (int hm = 0; hm < kNG && kNG * pr + hm < n_groups; ++hm) {
          const int gc = min(p.G, p.B - (kNG * pr + hm) * p.G);
          const int nt = htiles(a, gc);
          for (int t = 0; t < nt; ++t, ++sq) {
            const uint32_t d = sq & 1;
            if (sq >= 2) W(&hd_empty[d], ((sq >> 1) - 1) & 1, 0);
            for (int kb = 0; kb < 8; ++kb, ++kq) {
              const uint32_t s = kq % kHStages, r = kq / kHStages;
              W(&h_full[s], r & 1, 1);
              tc_fence_after();
              const uint32_t a0 = smem_u32(HA + s * kKB);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_f16(tmem + 128u * d, sdesc_kmajor_sw128_addr(a0 + 32u * k),
                        sdesc_kmajor_sw128_addr(e0 + (uint32_t)(224 - 32 * kb) * 128u + 32u * k), idesc,
                        (kb | k) != 0);
              mma_commit(&h_empty[s]);
            }
            mma_commit(&hd_full[d]);
          }
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ conv producer
    if (elect_one()) {
      uint32_t i = 0;
      int gi = 0;
      for (int pr = blockIdx.x; kNG * pr < n_groups; pr += gridDim.x, ++gi) {
        for (int a = 0; a < nl; ++a)
        for (int hm = 0; hm < kNG && kNG * pr + hm < n_groups; ++hm) {
          const int b0 = (kNG * pr + hm) * p.G, gc = min(p.G, p.B - b0);
          if (a > 0) W(&lvl_ready[hm * kMaxLv + a], gi & 1, 0);
          const int rs = p.rs[a], U = p.U[a], tpc = (gc * U + 127) / 128;
          for (int v = 0; v < p.copies[a]; ++v) {
            for (int t = 0; t < tpc; ++t, ++i) {
              const int s = (int)(i % kCStages);
              const uint32_t r = i / kCStages;
              if (r > 0) W(&c_mma[s], (r - 1) & 1, 1);  // the stage's MMAs have read it
              uint8_t* As = CA + s * kCA;
              const int y = b0 * U + 128 * t;
              if (rs == 8) {
                mbar_expect_tx(&c_full[s], kRows8 * 16);
                bulk_load(As, p.crows[a] + v * p.copy_stride[a] + (int64_t)8 * y, kRows8 * 16, &c_full[s]);
              } else {
                mbar_expect_tx(&c_full[s], kCA);
                const CUtensorMap* map = &p.cmap[p.cmap0[a] + v * (rs >= 64 ? 2 : 1)];
                if (rs >= 64) {
                  tma_load_2d(As, map, &c_full[s], 0, y);
                  tma_load_2d(As + 16384, map + 1, &c_full[s], 64 % rs, y + 64 / rs);
                } else if (rs == 32) {
                  for (int j = 0; j < 3; ++j) tma_load_2d(As + 8192 * j, map, &c_full[s], 0, y + j);
                } else {
                  for (int j = 0; j < 6; ++j) tma_load_2d(As + 4096 * j, map, &c_full[s], 0, y + j);
                }
              }
            }
          }
        }
        mbar_arrive(cgrp_done);
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ conv MMA issue
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_f16(128, NCONV);
      const uint32_t b0s = smem_u32(filt);
      uint32_t i = 0;
      for (int pr = blockIdx.x; kNG * pr < n_groups; pr += gridDim.x) {
        for (int a = 0; a < nl; ++a)
        for (int hm = 0; hm < kNG && kNG * pr + hm < n_groups; ++hm) {
          const int gc = min(p.G, p.B - (kNG * pr + hm) * p.G);
          const int rs = p.rs[a], nt = ctiles(a, gc);
          for (int t = 0; t < nt; ++t, ++i) {
            const int s = (int)(i % kCStages);
            const uint32_t r = i / kCStages;
            W(&c_full[s], r & 1, 0);
            if (r > 0) W(&c_tfree[s], (r - 1) & 1, 1);
            tc_fence_after();
            const uint32_t a0 = smem_u32(CA + s * kCA);
#pragma unroll
            for (int k = 0; k < KC / 16; ++k) {
              uint64_t ad;
              if (rs >= 64) ad = k < 4 ? swz_desc(a0 + 32u * k, 128) : swz_desc(a0 + 16384u + 32u * (k - 4), 64);
              else if (rs == 32) ad = swz_desc(a0 + 8192u * (k >> 1) + 32u * (k & 1), 64);
              else if (rs == 16) ad = swz_desc(a0 + 4096u * k, 32);
              else ad = nsw_desc(a0 + 32u * k, 16, 128);
              mma_f16(tmem_c + 32 * s, ad, nsw_desc(b0s + (uint32_t)k * 1024u, 512, 128), idesc, k > 0);
            }
            mma_commit(&c_mma[s]);
          }
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ halving epilogue + level edges
    const int q = warp & 3, et = tid - 128;
    uint32_t sq = 0;
    for (int pr = blockIdx.x; kNG * pr < n_groups; pr += gridDim.x) {
      for (int a = 0; a + 1 < nl; ++a)
      for (int hm = 0; hm < kNG && kNG * pr + hm < n_groups; ++hm) {
        const int b0 = (kNG * pr + hm) * p.G, gc = min(p.G, p.B - b0);
        const int R = p.R[a], nt = htiles(a, gc);
        const int n_out = p.n[a + 1], nb = (n_out + 127) / 128;
        __half* dst = p.lv[a + 1];
        const int dstride = p.stride[a + 1];
        for (int t = 0; t < nt; ++t, ++sq) {
          const uint32_t d = sq & 1;
          const int g = 128 * t + q * 32 + lane;
          const int bl = g / R, n = g - bl * R;
          const bool live = bl < gc && n < nb;
          W(&hd_full[d], (sq >> 1) & 1, 0);
          tc_fence_after();
          __half* drow = dst + (int64_t)(b0 + bl) * dstride + kML + 128 * n;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 128u * d + 32u * c, v);
            tmem_ld_wait();
            const int i0 = 128 * n + 32 * c;
            if (!live || i0 >= n_out) continue;
            if (i0 + 32 <= n_out) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                __align__(16) __half2 w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) w[e] = __floats2half2_rn(v[8 * u + 2 * e], v[8 * u + 2 * e + 1]);
                *reinterpret_cast<uint4*>(drow + 32 * c + 8 * u) = *reinterpret_cast<const uint4*>(w);
              }
            } else {
              for (int e = 0; e < 32; ++e)
                if (i0 + e < n_out) drow[32 * c + e] = __float2half_rn(v[e]);
            }
            // the outputs the reflect margins mirror, kept in shared memory for the margin pass
            const int rb = (n_out - kMLeft) & ~31;
            if (i0 < kMLeft || i0 >= rb) {
              __half* mb = mbuf + bl * (kMLeft + kMRight) + (i0 < kMLeft ? i0 : kMLeft + i0 - rb);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                __align__(16) __half2 w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) w[e] = __floats2half2_rn(v[8 * u + 2 * e], v[8 * u + 2 * e + 1]);
                *reinterpret_cast<uint4*>(mb + 8 * u) = *reinterpret_cast<const uint4*>(w);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&hd_empty[d]);
        }
        // level a + 1: reflect margins (np.pad "reflect", signal.py:245) from the shared-memory copy
        // of the outputs they mirror, zero tail; then the conv's shifted copies (hop < 8)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        {
          const int rb = (n_out - kMLeft) & ~31;
          for (int j = et; j < gc * 2 * kML; j += 128) {
            const int bl = j / (2 * kML), r = j - bl * 2 * kML;
            const int i = r < kML ? r + 1 : n_out - 1 - kML + (r - kML);
            const __half val = mbuf[bl * (kMLeft + kMRight) + (r < kML ? i : kMLeft + i - rb)];
            dst[(int64_t)(b0 + bl) * dstride + (r < kML ? kML - i : kML + 2 * (n_out - 1) - i)] = val;
          }
          const int z0 = n_out + 2 * kML, nz = dstride - z0;
          for (int j = et; j < gc * nz; j += 128) {
            const int bl = j / nz;
            dst[(int64_t)(b0 + bl) * dstride + z0 + (j - bl * nz)] = __float2half_rn(0.f);
          }
        }
        // the margin pass's mbuf reads finish before any warp writes the next group's tile
        // outputs into mbuf (the copies pass below has the same barrier)
        if (p.copies[a + 1] <= 1) asm volatile("bar.sync 1, 128;" ::: "memory");
        if (p.copies[a + 1] > 1) {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int h = p.h[a + 1], n8 = dstride / 8, nc = p.copies[a + 1] - 1;
          const int n_items = gc * nc * n8;
          for (int j0 = et; j0 < n_items; j0 += 4 * 128) {
            uint4 w0[4], w1[4];
            int dsto[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = j0 + 128 * u;
              dsto[u] = -1;
              if (j >= n_items) continue;
              const int bl = j / (nc * n8), rem = j - bl * nc * n8, v = 1 + rem / n8, k8 = rem - (v - 1) * n8;
              const __half* row = dst + (int64_t)(b0 + bl) * dstride;
              const int i0 = 8 * k8 + v * h, al = i0 & ~7;
              const uint4 z = make_uint4(0, 0, 0, 0);
              w0[u] = al < dstride ? *reinterpret_cast<const uint4*>(row + al) : z;
              w1[u] = (al + 8 < dstride && (i0 & 7)) ? *reinterpret_cast<const uint4*>(row + al + 8) : z;
              dsto[u] = ((i0 & 7) >> 1) | (v << 3) | (k8 << 8);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (dsto[u] < 0) continue;
              const int j = j0 + 128 * u, bl = j / (nc * n8);
              const int q2 = dsto[u] & 7, v = (dsto[u] >> 3) & 31, k8 = dsto[u] >> 8;
              const uint32_t wd[8] = {w0[u].x, w0[u].y, w0[u].z, w0[u].w, w1[u].x, w1[u].y, w1[u].z, w1[u].w};
              uint4 o;
              o.x = q2 == 0 ? wd[0] : q2 == 1 ? wd[1] : q2 == 2 ? wd[2] : wd[3];
              o.y = q2 == 0 ? wd[1] : q2 == 1 ? wd[2] : q2 == 2 ? wd[3] : wd[4];
              o.z = q2 == 0 ? wd[2] : q2 == 1 ? wd[3] : q2 == 2 ? wd[4] : wd[5];
              o.w = q2 == 0 ? wd[3] : q2 == 1 ? wd[4] : q2 == 2 ? wd[5] : wd[6];
              *reinterpret_cast<uint4*>(dst + v * p.copy_stride[a + 1] + (int64_t)(b0 + bl) * dstride + 8 * k8) = o;
            }
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads these stores next
        mbar_arrive(&lvl_ready[hm * kMaxLv + a + 1]);
      }
    }
  } else {
    // ------------------------------------------------------------ conv epilogue: two warpgroups
    const int q = warp & 3, eg = (warp - 8) >> 2;
    const int j_hi = min(p.n_filt, NCONV / 2);
    uint32_t i = 0;
    for (int pr = blockIdx.x; kNG * pr < n_groups; pr += gridDim.x) {
      for (int a = 0; a < nl; ++a)
      for (int hm = 0; hm < kNG && kNG * pr + hm < n_groups; ++hm) {
        const int b0 = (kNG * pr + hm) * p.G, gc = min(p.G, p.B - b0);
        const int U = p.U[a], C = p.copies[a], tpc = (gc * U + 127) / 128;
        const int lskip = max(0, a * p.bpo - p.first_bin), lrow0 = p.first_bin - a * p.bpo;
        for (int v = 0; v < C; ++v) {
          for (int t = 0; t < tpc; ++t, ++i) {
            if ((int)(i & 1) != eg) continue;
            const int s = (int)(i % kCStages);
            const uint32_t r = i / kCStages;
            const int g = 128 * t + q * 32 + lane;  // frame row within the group's level rows
            const int bl = g / U;
            const int tt = C * (g - bl * U) + v;
            const bool live = bl < gc && tt < p.T;
            const int ex = live ? exps_s[b0 + bl] : 0;
            W(&c_mma[s], r & 1, 0);
            tc_fence_after();
            float acc[32];
            tmem_ld32(tmem_c + ((uint32_t)(q * 32) << 16) + 32 * s, acc);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&c_tfree[s]);
            if (!live) continue;
            const int eo = ex - kFiltLog2;
            const float os = (eo > -126 && eo < 128) ? __int_as_float((eo + 127) << 23) : ldexpf(1.f, eo);
            const int64_t obase = ((int64_t)(b0 + bl) * p.n_bins + lrow0) * p.T + tt;
            if (p.out_kind == NNAB_OUT_COMPLEX) {
              float2* o2 = reinterpret_cast<float2*>(p.out) + obase;
#pragma unroll
              for (int j = 0; j < NCONV / 2; ++j)
                if (j >= lskip && j < j_hi) o2[j * p.T] = make_float2(acc[2 * j] * os, acc[2 * j + 1] * os);
            } else {
              float* o = p.out + obase;
              const bool pw = p.out_kind == NNAB_OUT_POWER;
#pragma unroll
              for (int j = 0; j < NCONV / 2; ++j) {
                if (j < lskip || j >= j_hi) continue;
                const float re = acc[2 * j] * os, im = acc[2 * j + 1] * os, q2 = fmaf(re, re, im * im);
                o[j * p.T] = pw ? q2 : fast_sqrt(q2);
              }
            }
          }
        }
      }
    }
  }
  if (p.prof) {  // [role * 4 + slot]: roles 0 h-producer, 1 h-MMA, 2 c-producer, 3 c-MMA, 4 h-epi, 5 c-epi; [24] elapsed
    const int role = warp < 4 ? warp : warp < 8 ? 4 : 5;
    const bool lead = (warp < 4) || tid == 128 || tid == 256;
    if (lead)
      for (int i = 0; i < 4; ++i)
        if (pw[i]) atomicAdd(p.prof + 4 * role + i, pw[i]);
    if (tid == 128) atomicAdd(p.prof + 24, (unsigned long long)(clock64() - tb));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

__device__ unsigned long long g_back_prof[32];
bool g_back_prof_on = false;

}  // namespace

int launch_cqt2010_back(const CqtBackArgs& g, cudaStream_t st) {
  const int n_oct = g.n_oct;
  const int64_t B = g.B;
  if (g.n_taps != 255 || n_oct < 2 || n_oct > kMaxLv || B > (1 << 24) || 4 * B > 16384) return NNAB_ENOTSUP;
  BackParams* pp = new BackParams{};
  BackParams& p = *pp;
  p.n_oct = n_oct;
  p.B = (int32_t)B;
  p.G = (int32_t)((B + kNG * num_sms() - 1) / (kNG * num_sms()));  // kNG groups per CTA
  for (int j = 0; j < 255; ++j) p.taps[j] = g.taps[j];
  p.T = g.T;
  p.n_bins = g.n_bins;
  p.first_bin = g.first_bin;
  p.bpo = g.bpo;
  p.n_filt = g.n_filt;
  p.out_kind = g.out_kind;
  p.exps = g.exps;
  p.filt_img = g.filt_img;
  p.out = g.out;
  p.prof = nullptr;
  if (g_back_prof_on) {
    void* ptr = nullptr;
    cudaGetSymbolAddress(&ptr, g_back_prof);
    p.prof = reinterpret_cast<unsigned long long*>(ptr);
  }
  int rc = NNAB_OK, nm = 0;
  for (int a = 0; a < n_oct && !rc; ++a) {
    p.lv[a] = g.lv[a];
    p.n[a] = g.n[a];
    p.stride[a] = g.stride[a];
    p.R[a] = g.stride[a] / 256;
    p.h[a] = g.h[a];
    p.copies[a] = g.copies[a];
    p.U[a] = g.U[a];
    p.rs[a] = g.rs[a];
    p.copy_stride[a] = B * (int64_t)g.stride[a];
    const __half* cbase = g.lv[a] + (kML - g.pad_al);
    p.crows[a] = cbase;
    p.cmap0[a] = nm;
    const int rs = g.rs[a];
    if (g.stride[a] % 256 || (a + 1 < n_oct && 256 * ((g.n[a + 1] + 127) / 128 + 1) > g.stride[a]) ||
        B * (int64_t)p.R[a] >= INT32_MAX || (rs != 8 && rs != 16 && rs != 32 && rs < 64) ||
        (int64_t)g.copies[a] * g.U[a] < g.T) {
      rc = NNAB_ENOTSUP;
      break;
    }
    if (a + 1 < n_oct) rc = make_tmap_2d(&p.hmap[a], g.lv[a], 256, (uint64_t)(B * p.R[a]), 512, 64, 128, 128, 2);
    if (rc || rs == 8) continue;
    for (int v = 0; v < g.copies[a] && !rc; ++v) {
      const __half* cb = cbase + (int64_t)v * p.copy_stride[a];
      const int nbox = rs >= 64 ? 2 : 1;
      if (nm + nbox > kCMaps) { rc = NNAB_ENOTSUP; break; }
      const uint32_t w0 = rs >= 64 ? 64 : (uint32_t)rs;
      rc = make_tmap_2d(&p.cmap[nm++], cb, (uint64_t)rs, (uint64_t)(B * g.U[a]), (uint64_t)rs * 2, w0, 128,
                        (int)w0 * 2, 2);
      if (!rc && nbox == 2)
        rc = make_tmap_2d(&p.cmap[nm++], cb, (uint64_t)rs, (uint64_t)(B * g.U[a]), (uint64_t)rs * 2, 32, 128, 64, 2);
    }
  }
  const size_t smem = 1024 + kHStages * kKB + kERows * 128 + kCStages * kCA + KC / 8 * 512 +
                      (2 * kHStages + 4 + 3 * kCStages + kNG * kMaxLv + 1) * 8 + 16 + 4 * (size_t)((B + 7) & ~7) +
                      2 * kMaxG * (kMLeft + kMRight) + 16;
  if (p.G > kMaxG) rc = NNAB_ENOTSUP;
  if (!rc && smem > 227 * 1024) rc = NNAB_ENOTSUP;
  if (!rc) {
    cudaError_t e = cudaFuncSetAttribute(cqt2010_back_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) {
      const int pairs = (int)(((B + p.G - 1) / p.G + kNG - 1) / kNG);  // group sets
      cqt2010_back_kernel<<<std::min(pairs, num_sms()), kThreads, smem, st>>>(p);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "cqt2010_back_kernel");
    else note_launch();
  }
  delete pp;
  return rc;
}

}  // namespace nnab

// Debug: per-role wait cycles of the CQT2010v2 back-end kernel (on != 0 clears and enables;
// on == 0 copies [32] out).
extern "C" int nnab_debug_cqt2010_back_profile(int on, unsigned long long* out) {
  using nnab::cuda_fail;
  if (on) {
    nnab::g_back_prof_on = true;
    unsigned long long z[32] = {};
    NNAB_CUDA_TRY(cudaMemcpyToSymbol(nnab::g_back_prof, z, sizeof(z)));
    return NNAB_OK;
  }
  nnab::g_back_prof_on = false;
  if (out) NNAB_CUDA_TRY(cudaMemcpyFromSymbol(out, nnab::g_back_prof, 32 * sizeof(unsigned long long)));
  return NNAB_OK;
}
