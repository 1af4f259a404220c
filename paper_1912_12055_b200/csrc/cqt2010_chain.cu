// CQT2010v2 octave chain: the halvings octave 0 -> 1 -> ... -> n_oct - 1
// (transforms.py:303-305, signal.py:232-247) of a group of clips per CTA, TMA-fed
// tensor-core FIRs over the level buffers (which stay in L2 between levels).
//
// A halving as one dense GEMM (no operand build): level a's buffer row of clip b is
// [ML reflect margin | signal | ML margin | zeros], viewed as rows of 256 samples, so
//   y[128 n + r] = sum_j h[j] s_ext[2 (128 n + r) + j - 127]
//                = sum_{k < 512} buf[256 n + k] h[k - 2 r - 1]       (buf[i] = s_ext[i - ML])
// i.e. D[block n][r] = A[n][k] B[r][k] with A = two consecutive 256-sample rows (one TMA
// box of 64 x 128 per 64-sample K block, 128-byte swizzle) and B[r][k] = h[k - 2 r - 1]:
// for K block kb, B_kb[r][k'] = E[r - 32 kb][k'] with E[r][k'] = h[k' - 2 r - 1], so all
// eight K blocks are row windows of one 352 x 64 shared-memory matrix (45 KB).  32 MMAs
// (M = N = 128, K = 16) per tile of 128 blocks; rows of all the group's clips are one
// uniform row array (clip stride R_a rows), rows that are not a block of the group are
// computed and dropped.
//
// Per level: warp 0 issues the TMA loads (K-block ring), warp 1 the MMAs (2 TMEM
// accumulators), warps 4-7 the epilogue (thread = block: 128 outputs -> level a + 1 in
// FP16, 16-byte stores).  At the level's end the epilogue warps write the new level's
// reflect margins, zero tail and (hop < 8) the conv's shifted copies, then the CTA syncs
// and the next level's TMA reads what it wrote (generic -> async proxy fence).
#include <algorithm>
#include <cmath>

#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kML = 128;
constexpr int kMaxLv = 12;
constexpr int kThreads = 8 * 32;
constexpr int kERows = 352;                 // E rows r = -224 .. 127
constexpr int kStages = 4;                  // K-block ring (16 KB stages: 128 rows x 64 samples); 2 CTAs / SM
constexpr uint32_t kKB = 16384;

struct ChainParams {
  CUtensorMap map[kMaxLv];                  // level a as rows of 256 samples (halving input)
  int32_t n_oct, B, G;                      // clips, clips per group
  int32_t n[kMaxLv], stride[kMaxLv], R[kMaxLv], h[kMaxLv], copies[kMaxLv];
  int64_t copy_stride[kMaxLv];
  __half* lv[kMaxLv];
  float taps[255];
  unsigned long long* prof;  // debug: per level [3a]: tiles done (epilogue), [3a+1]: margins done, [3a+2]: level end
};

__global__ void __launch_bounds__(kThreads, 2) cqt2010_chain_kernel(const __grid_constant__ ChainParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = base;                       // [kStages] x kKB
  uint8_t* E = base + kStages * kKB;       // kERows x 128 B, 128-byte swizzle
  uint64_t* bars = reinterpret_cast<uint64_t*>(E + kERows * 128);
  uint64_t* a_full = bars;                 // [kStages] TMA tx
  uint64_t* a_empty = a_full + kStages;    // [kStages] commit
  uint64_t* d_full = a_empty + kStages;    // [2] commit
  uint64_t* d_empty = d_full + 2;          // [2] 4 epilogue warps
  uint32_t* tslot = reinterpret_cast<uint32_t*>(d_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  // E[r][k'] = h[k' - 2 r - 1] (r = row - 224), FP16, K-major with the 128-byte swizzle
  // (16-byte chunk c of row w at chunk c ^ (w & 7))
  __shared__ float taps_s[256];
  for (int j = tid; j < 256; j += kThreads) taps_s[j] = j < 255 ? p.taps[j] : 0.f;
  __syncthreads();
  for (int i = tid; i < kERows * 8; i += kThreads) {  // one 16-byte chunk per step
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
  const int n_groups = (p.B + p.G - 1) / p.G;
  uint32_t seq = 0;  // tile sequence over groups and levels (ring / accumulator phases)
  long long tl = clock64();

  for (int grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const int b0 = grp * p.G, gc = min(p.G, p.B - b0);
    for (int a = 0; a + 1 < p.n_oct; ++a) {
      const int R = p.R[a];
      const int n_out = p.n[a + 1], nb = (n_out + 127) / 128;
      const int rows = gc * R, n_tiles = (rows + 127) / 128;
      if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
          const CUtensorMap* map = &p.map[a];
          for (int t = 0; t < n_tiles; ++t) {
            const int row0 = b0 * R + 128 * t;
            for (int kb = 0; kb < 8; ++kb) {
              const uint32_t kq = 8 * (seq + t) + kb, s = kq % kStages, r = kq / kStages;
              if (r > 0) mbar_wait_sleep(&a_empty[s], (r - 1) & 1);
              mbar_expect_tx(&a_full[s], kKB);
              tma_load_2d(A + s * kKB, map, &a_full[s], 64 * (kb & 3), row0 + (kb >> 2));
            }
          }
        }
      } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issue
        if (elect_one()) {
          constexpr uint32_t idesc = idesc_f16(128, 128);
          const uint32_t e0 = smem_u32(E);
          for (int t = 0; t < n_tiles; ++t) {
            const uint32_t sq = seq + t, d = sq & 1;
            if (sq >= 2) mbar_wait_sleep(&d_empty[d], ((sq >> 1) - 1) & 1);
            for (int kb = 0; kb < 8; ++kb) {
              const uint32_t kq = 8 * sq + kb, s = kq % kStages, r = kq / kStages;
              mbar_wait_sleep(&a_full[s], r & 1);
              tc_fence_after();
              const uint32_t a0 = smem_u32(A + s * kKB);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_f16(tmem + 128u * d, sdesc_kmajor_sw128_addr(a0 + 32u * k),
                        sdesc_kmajor_sw128_addr(e0 + (uint32_t)(224 - 32 * kb) * 128u + 32u * k), idesc,
                        (kb | k) != 0);
              mma_commit(&a_empty[s]);
            }
            mma_commit(&d_full[d]);
          }
        }
      } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3, et = tid - 128;
        __half* dst = p.lv[a + 1];
        const int dstride = p.stride[a + 1];
        for (int t = 0; t < n_tiles; ++t) {
          const uint32_t sq = seq + t, s = sq & 1;
          const int g = 128 * t + q * 32 + lane;  // row within the group
          const int bl = g / R, n = g - bl * R;
          const bool live = bl < gc && n < nb;
          mbar_wait_sleep(&d_full[s], (sq >> 1) & 1);
          tc_fence_after();
          __half* drow = dst + (int64_t)(b0 + bl) * dstride + kML + 128 * n;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 128u * s + 32u * c, v);
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
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[s]);
        }
        // level a + 1: reflect margins (np.pad "reflect", signal.py:245) and zero tail, then the
        // conv's shifted copies (hop < 8); items over all the group's clips, loads batched
        // ahead of the stores (plain loads: this CTA's own stores)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (p.prof && et == 0) { const long long n = clock64(); atomicAdd(p.prof + 3 * a, (unsigned long long)(n - tl)); tl = n; }
        {
          const int n_items = gc * 2 * kML;
          for (int j0 = et; j0 < n_items; j0 += 8 * 128) {
            __half v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int j = j0 + 128 * u;
              if (j >= n_items) break;
              const int bl = j / (2 * kML), r = j - bl * 2 * kML;
              const int i = r < kML ? r + 1 : n_out - 1 - kML + (r - kML);
              v[u] = dst[(int64_t)(b0 + bl) * dstride + kML + i];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int j = j0 + 128 * u;
              if (j >= n_items) break;
              const int bl = j / (2 * kML), r = j - bl * 2 * kML;
              const int i = r < kML ? r + 1 : n_out - 1 - kML + (r - kML);
              dst[(int64_t)(b0 + bl) * dstride + (r < kML ? kML - i : kML + 2 * (n_out - 1) - i)] = v[u];
            }
          }
          const int z0 = n_out + 2 * kML, nz = dstride - z0;  // zero tail
          for (int j = et; j < gc * nz; j += 128) {
            const int bl = j / nz;
            dst[(int64_t)(b0 + bl) * dstride + z0 + (j - bl * nz)] = __float2half_rn(0.f);
          }
        }
        if (p.copies[a + 1] > 1) {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int h = p.h[a + 1], n8 = dstride / 8, nc = p.copies[a + 1] - 1;
          const int n_items = gc * nc * n8;  // 8-sample units of the copies
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
        asm volatile("fence.proxy.async.global;" ::: "memory");  // the next level's TMA reads these stores
        if (p.prof && et == 0) { const long long n = clock64(); atomicAdd(p.prof + 3 * a + 1, (unsigned long long)(n - tl)); tl = n; }
      }
      seq += (uint32_t)n_tiles;
      __syncthreads();
      if (p.prof && tid == 128) { const long long n = clock64(); atomicAdd(p.prof + 3 * a + 2, (unsigned long long)(n - tl)); tl = n; }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

__device__ unsigned long long g_chain_prof[40];
bool g_chain_prof_on = false;
unsigned long long* cqt2010_chain_prof() {
  if (!g_chain_prof_on) return nullptr;
  void* ptr = nullptr;
  cudaGetSymbolAddress(&ptr, g_chain_prof);
  return reinterpret_cast<unsigned long long*>(ptr);
}

}  // namespace

// Debug: per-level phase cycles of the octave chain (on != 0 clears and enables; on == 0
// copies [40] out): level a at 3 a: tiles, 3 a + 1: margins / copies, 3 a + 2: barrier.
extern "C" int nnab_debug_cqt2010_chain_profile(int on, unsigned long long* out) {
  if (on) {
    g_chain_prof_on = true;
    unsigned long long z[40] = {};
    NNAB_CUDA_TRY(cudaMemcpyToSymbol(g_chain_prof, z, sizeof(z)));
    return NNAB_OK;
  }
  g_chain_prof_on = false;
  if (out) NNAB_CUDA_TRY(cudaMemcpyFromSymbol(out, g_chain_prof, 40 * sizeof(unsigned long long)));
  return NNAB_OK;
}

// levels: base pointers, strides (multiples of 256), lengths, hops and conv copies of every
// octave; level 0 (with its margins) is already written.  NNAB_ENOTSUP outside the envelope.
int launch_cqt2010_chain(int64_t B, int n_oct, __half* const* lv, const int32_t* stride, const int32_t* n,
                         const int32_t* h, const int32_t* copies, const float* taps, int n_taps, cudaStream_t st) {
  if (n_taps != 255 || n_oct < 2 || n_oct > kMaxLv || B > (1 << 24)) return NNAB_ENOTSUP;
  ChainParams* cp = new ChainParams{};
  ChainParams& p = *cp;
  p.n_oct = n_oct;
  p.B = (int32_t)B;
  p.G = (int32_t)((B + 2 * num_sms() - 1) / (2 * num_sms()));  // two CTAs per SM
  for (int j = 0; j < 255; ++j) p.taps[j] = taps[j];
  p.prof = cqt2010_chain_prof();
  int rc = NNAB_OK;
  for (int a = 0; a < n_oct && !rc; ++a) {
    p.lv[a] = lv[a];
    p.n[a] = n[a];
    p.stride[a] = stride[a];
    p.R[a] = stride[a] / 256;
    p.h[a] = h[a];
    p.copies[a] = copies[a];
    p.copy_stride[a] = B * (int64_t)stride[a];
    if (stride[a] % 256 || (a + 1 < n_oct && 256 * ((n[a + 1] + 127) / 128 + 1) > stride[a]) ||
        B * (int64_t)p.R[a] >= INT32_MAX)
      rc = NNAB_ENOTSUP;
    else if (a + 1 < n_oct)
      rc = make_tmap_2d(&p.map[a], lv[a], 256, (uint64_t)(B * p.R[a]), 512, 64, 128, 128, 2);
  }
  const size_t smem = 1024 + kStages * kKB + kERows * 128 + 256;
  if (!rc) {
    cudaError_t e = cudaFuncSetAttribute(cqt2010_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) {
      const int groups = (int)((B + p.G - 1) / p.G);
      cqt2010_chain_kernel<<<std::min(groups, 2 * num_sms()), kThreads, smem, st>>>(p);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "cqt2010_chain_kernel");
    else note_launch();
  }
  delete cp;
  return rc;
}

}  // namespace nnab
