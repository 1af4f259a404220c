// Frame staging and bank packing.
//
// The reference materialises every frame (`sliding_window_view(x, M)[::stride]`
// then `ascontiguousarray`, signal.py:181) after padding the clip
// (`np.pad(..., "reflect")`, signal.py:151 via transforms.py:106-107).  Here the
// padded clip is instead laid out ONCE as "hop rows": row r of clip b holds
// padded_b[r*hop, r*hop + hop).  Frame t is then rows t .. t+width/hop-1, so a
// GEMM A-tile for 128 consecutive frames and a 32-sample K block is one
// rectangular TMA box (rows g0+k/hop .., columns k%hop ..): the frames are never
// materialised, and the reflect/zero padding is resolved here with the exact
// np.pad index map (gradients.py:18-25).  When hop does not divide into 32-sample
// K blocks (or hop > width) the rows are whole frames (row_len = width rounded up).
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {

int frame_geometry(const nnab_frames* f, FrameGeom* g, int kalign) {
  if (!f || !g) return NNAB_EINVAL;
  if (f->batch < 0 || f->length < 1 || f->width < 1 || f->hop < 1 || f->pad < 0) return NNAB_EINVAL;
  if (f->pad_mode != NNAB_PAD_REFLECT && f->pad_mode != NNAB_PAD_ZERO) return NNAB_EINVAL;
  if (f->pad_mode == NNAB_PAD_REFLECT && f->pad > 0 && f->pad >= f->length) return NNAB_EINVAL;  // signal.py:147
  g->B = f->batch;
  g->L = f->length;
  g->width = f->width;
  g->hop = f->hop;
  g->pad = f->pad;
  g->pad_mode = f->pad_mode;
  g->padded_len = f->length + 2ll * f->pad;
  if (f->width > g->padded_len) return NNAB_EINVAL;  // signal.py:176-177
  int64_t T = (g->padded_len - f->width) / f->hop + 1;
  if (T > (1ll << 30)) return NNAB_ENOTSUP;
  g->T = (int32_t)T;
  g->k_pad = (f->width + kalign - 1) / kalign * kalign;
  if (f->hop % kalign == 0 && f->hop <= g->k_pad) {
    g->row_len = f->hop;
    g->R = g->T + (g->k_pad + f->hop - 1) / f->hop - 1;
  } else {
    g->row_len = g->k_pad;
    g->R = g->T;
  }
  return NNAB_OK;
}

// The 4 padded samples i0 .. i0+3 of clip b (np.pad index map, signal.py:151;
// 0 beyond the padded clip): interior groups of 4 samples are one aligned
// 16-byte load (or two aligned loads and a funnel when clip starts are off
// 16-byte boundaries), reflected groups a reversed funnel, the rest scalar.
NNAB_DEV void gather4(const float* __restrict__ x, int64_t b, int64_t L, int32_t pad, int32_t mode,
                      int64_t padded_len, bool aligned_clips, bool x_aligned, int64_t i0, float* v) {
  const float* xb = x + b * L;
  const int64_t j0 = i0 - pad;    // source sample
  const int64_t ga = b * L + j0;  // absolute source index
  if (aligned_clips && j0 >= 0 && j0 + 3 < L && i0 + 3 < padded_len) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(xb + j0));
    v[0] = w.x;
    v[1] = w.y;
    v[2] = w.z;
    v[3] = w.w;
  } else if (x_aligned && j0 >= 0 && j0 - (ga & 3) + 7 < L && i0 + 3 < padded_len) {
    // interior of a clip whose rows start off a 16-byte boundary (e.g. the CQT
    // pad of 11,341): two aligned loads and a funnel by the misalignment
    const float4* a4 = reinterpret_cast<const float4*>(x + (ga & ~int64_t(3)));
    const float4 w0 = __ldg(a4), w1 = __ldg(a4 + 1);
    const float e[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const int m = (int)(ga & 3);
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = m == 0 ? e[u] : m == 1 ? e[u + 1] : m == 2 ? e[u + 2] : e[u + 3];
  } else if (x_aligned && mode == NNAB_PAD_REFLECT && i0 + 3 < padded_len &&
             ((j0 + 3 < 0 && -j0 < L) || (j0 >= L && 2 * (L - 1) - j0 - 3 >= 0))) {
    // a reflected group (np.pad "reflect": one mirror image, left or right):
    // its 4 sources are one descending run -- the same funnel, reversed
    const int64_t a_lo = j0 < 0 ? -j0 - 3 : 2 * (L - 1) - j0 - 3;
    const int64_t gl = b * L + a_lo;
    if (a_lo - (gl & 3) + 7 < L) {
      const float4* a4 = reinterpret_cast<const float4*>(x + (gl & ~int64_t(3)));
      const float4 w0 = __ldg(a4), w1 = __ldg(a4 + 1);
      const float e[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
      const int m = (int)(gl & 3);
#pragma unroll
      for (int u = 0; u < 4; ++u) v[3 - u] = m == 0 ? e[u] : m == 1 ? e[u + 1] : m == 2 ? e[u + 2] : e[u + 3];
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[3 - u] = __ldg(xb + a_lo + u);
    }
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u;
      float sv = 0.f;
      if (i < padded_len) {
        int64_t j = i - pad;
        if (mode == NNAB_PAD_REFLECT) {
          if (j < 0) j = -j;
          if (j >= L) j = 2 * (L - 1) - j;
          sv = __ldg(xb + j);
        } else if (j >= 0 && j < L) {
          sv = __ldg(xb + j);
        }
      }
      v[u] = sv;
    }
  }
}

// rows[(b*R + r)*row_len + c] = padded_b[r*hop + c]  (0 beyond the padded clip),
// TF32-rounded (split=0) or split into tf32 hi + tf32 lo residual (split=1).
// One CTA walks whole rows (no 64-bit divisions per element).
__global__ void __launch_bounds__(256) stage_rows_kernel(const float* __restrict__ x, int64_t B, int64_t L,
                                                         int32_t pad, int32_t mode, int32_t hop, int32_t row_len,
                                                         int32_t R, int64_t padded_len, int split,
                                                         float* __restrict__ hi, float* __restrict__ lo) {
  const int32_t q_per_row = row_len / 4;
  const int64_t rows = B * (int64_t)R;
  const bool aligned_clips = (L % 4) == 0 && (pad % 4) == 0 && (hop % 4) == 0;
  const bool x_aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int per = q_per_row < (int)blockDim.x ? q_per_row : (int)blockDim.x;  // threads per row
  const int rpb = blockDim.x / per;                                           // rows per block step
  const int sub = threadIdx.x / per, lane = threadIdx.x - sub * per;
  if (sub >= rpb) return;
  for (int64_t grow = (int64_t)blockIdx.x * rpb + sub; grow < rows; grow += (int64_t)gridDim.x * rpb) {
    const int64_t b = grow / R;
    const int64_t r = grow - b * R;
    float4* hrow = reinterpret_cast<float4*>(hi) + grow * q_per_row;
    float4* lrow = reinterpret_cast<float4*>(lo) + grow * q_per_row;
    for (int32_t q = lane; q < q_per_row; q += per) {
      float v[4];
      gather4(x, b, L, pad, mode, padded_len, aligned_clips, x_aligned, r * hop + 4 * q, v);
      float4 h, l;
      h.x = tf32_rne(v[0]);
      h.y = tf32_rne(v[1]);
      h.z = tf32_rne(v[2]);
      h.w = tf32_rne(v[3]);
      hrow[q] = h;
      if (split) {
        l.x = tf32_rne(v[0] - h.x);
        l.y = tf32_rne(v[1] - h.y);
        l.z = tf32_rne(v[2] - h.z);
        l.w = tf32_rne(v[3] - h.w);
        lrow[q] = l;
      }
    }
  }
}

// FP16 operands: 2^scale_exp(peak) so the clip's peak lands in [2^14, 2^15)
// (FP16's 11-bit significand = TF32's, with the 5-bit exponent kept in range by
// the exact power-of-two scale).  0 for a silent clip; clamped so 2^e is finite.
NNAB_DEV int f16_scale_exp(float peak) {
  int ex = 0;
  if (peak > 0.f && peak < INFINITY) frexpf(peak, &ex);  // peak = m 2^ex, m in [0.5, 1)
  return peak > 0.f ? max(-100, min(100, 15 - ex)) : 0;
}

// One CTA per clip (persistent over clips): pass 1 finds the clip's peak, pass 2
// (the clip now in L2) writes its hop rows scaled by 2^e as FP16 (split: hi =
// RN(v), lo = RN(v - hi), 22 significant bits), and exps[b] = e.
__global__ void __launch_bounds__(1024, 1) stage_rows_f16_kernel(const float* __restrict__ x, int64_t B, int64_t L,
                                                              int32_t pad, int32_t mode, int32_t hop, int32_t row_len,
                                                              int32_t R, int64_t padded_len, int split,
                                                              __half* __restrict__ hi, __half* __restrict__ lo,
                                                              int32_t* __restrict__ exps) {
  __shared__ float red[32];
  const bool aligned_clips = (L % 4) == 0 && (pad % 4) == 0 && (hop % 4) == 0;
  const bool x_aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int32_t q_per_row = row_len / 4;
  const int64_t groups = (int64_t)R * q_per_row;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const float* xb = x + b * L;
    float mx = 0.f;
    if (x_aligned && ((b * L) & 3) == 0) {
      const int64_t n4 = L / 4;
      const float4* x4 = reinterpret_cast<const float4*>(xb);
      const int64_t step = blockDim.x;
      int64_t i = threadIdx.x;
      for (; i + 3 * step < n4; i += 4 * step) {  // 4 loads in flight per thread (64 KB per SM)
        float4 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = __ldg(x4 + i + u * step);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(w[u].x), fabsf(w[u].y)), fmaxf(fabsf(w[u].z), fabsf(w[u].w))));
      }
      for (; i < n4; i += step) {
        const float4 w = __ldg(x4 + i);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(w.x), fabsf(w.y)), fmaxf(fabsf(w.z), fabsf(w.w))));
      }
      for (int64_t i = 4 * n4 + threadIdx.x; i < L; i += blockDim.x) mx = fmaxf(mx, fabsf(__ldg(xb + i)));
    } else {
      for (int64_t i = threadIdx.x; i < L; i += blockDim.x) mx = fmaxf(mx, fabsf(__ldg(xb + i)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
      float m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (threadIdx.x == 0) red[0] = m;
    }
    __syncthreads();
    const int e = f16_scale_exp(red[0]);
    __syncthreads();  // red[] reused by the next clip
    if (threadIdx.x == 0) exps[b] = e;
    const float sc = ldexpf(1.f, e);
    uint2* hrow = reinterpret_cast<uint2*>(hi) + b * groups;
    uint2* lrow = reinterpret_cast<uint2*>(lo) + b * groups;
    // pass 2 from L2: kU independent groups per thread in flight before any store
    constexpr int kU = 4;
    for (int64_t g0 = threadIdx.x; g0 < groups; g0 += (int64_t)kU * blockDim.x) {
      float v[kU][4];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t gq = g0 + (int64_t)u * blockDim.x;
        if (gq < groups) {
          const int64_t r = gq / q_per_row;
          const int32_t q = (int32_t)(gq - r * q_per_row);
          gather4(x, b, L, pad, mode, padded_len, aligned_clips, x_aligned, r * hop + 4 * q, v[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t gq = g0 + (int64_t)u * blockDim.x;
        if (gq >= groups) break;
        __half2 h01 = __floats2half2_rn(v[u][0] * sc, v[u][1] * sc), h23 = __floats2half2_rn(v[u][2] * sc, v[u][3] * sc);
        uint2 hv;
        hv.x = *reinterpret_cast<uint32_t*>(&h01);
        hv.y = *reinterpret_cast<uint32_t*>(&h23);
        hrow[gq] = hv;
        if (split) {
          const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
          __half2 l01 = __floats2half2_rn(v[u][0] * sc - f01.x, v[u][1] * sc - f01.y);
          __half2 l23 = __floats2half2_rn(v[u][2] * sc - f23.x, v[u][3] * sc - f23.y);
          uint2 lv;
          lv.x = *reinterpret_cast<uint32_t*>(&l01);
          lv.y = *reinterpret_cast<uint32_t*>(&l23);
          lrow[gq] = lv;
        }
      }
    }
  }
}

// FP16 staging that reads each clip from HBM once: a cluster of two CTAs (two SMs) per
// clip, each holding half of it in shared memory (bulk copies); the clip's peak is the max
// of the two halves' (exchanged through distributed shared memory); each CTA then writes
// half of the clip's hop rows, reading its sources from its own half or, near the split
// and for reflected samples, from the peer's (ld.shared::cluster).  Hop-row layouts with
// halves up to kPairHalf samples; else the two-pass kernel above.
constexpr int kPairHalf = 54 * 1024;  // floats per CTA (216 KB)

NNAB_DEV float ld_cluster_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

__global__ void __launch_bounds__(1024, 1) stage_rows_f16_pair_kernel(
    const float* __restrict__ x, int64_t B, int64_t L, int32_t pad, int32_t mode, int32_t hop, int32_t R,
    int64_t padded_len, int split, __half* __restrict__ hi, __half* __restrict__ lo, int32_t* __restrict__ exps) {
  extern __shared__ __align__(128) float sx[];  // this CTA's half of the clip
  __shared__ float red[32];
  __shared__ float half_max[2];                  // [clip parity]: this CTA's peak, read by the peer
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int64_t L2 = (L / 2) & ~int64_t(3);
  const int64_t h0 = rank ? L2 : 0, h1 = rank ? L : L2, hn = h1 - h0;
  const uint32_t peer_sx = mapa(sx, peer);
  const bool bulk = (L % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t q_total = (int64_t)R * hop;                 // staged elements per clip (row_len = hop)
  const int64_t qh = ((q_total / 2) & ~int64_t(3));          // CTA 0 writes [0, qh), CTA 1 [qh, q_total)
  const int64_t q0 = rank ? qh : 0, q1 = rank ? q_total : qh;
  uint32_t phase = 0;
  int it = 0;
  for (int64_t b = cluster_id_x(); b < B; b += nclusters_x(), ++it) {
    const float* xb = x + b * L;
    // ---- load this CTA's half
    if (bulk) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, (uint32_t)(hn * 4));
        for (int64_t o = 0; o < hn * 4; o += 32768) {
          const uint32_t n = (uint32_t)(hn * 4 - o < 32768 ? hn * 4 - o : 32768);
          bulk_load(reinterpret_cast<char*>(sx) + o, reinterpret_cast<const char*>(xb + h0) + o, n, &bar);
        }
      }
      mbar_wait(&bar, phase);
      phase ^= 1;
    } else {
      for (int64_t i = threadIdx.x; i < hn; i += blockDim.x) sx[i] = __ldg(xb + h0 + i);
      __syncthreads();
    }
    // ---- the clip's peak: this half's, then the max with the peer's
    float mx = 0.f;
    for (int64_t i = threadIdx.x; i < hn; i += blockDim.x) mx = fmaxf(mx, fabsf(sx[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
      float m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (threadIdx.x == 0) half_max[it & 1] = m;
    }
    cluster_sync();  // both halves loaded and both peaks published
    const float pk = fmaxf(half_max[it & 1], ld_cluster_f32(mapa(&half_max[it & 1], peer)));
    const int e = f16_scale_exp(pk);
    if (rank == 0 && threadIdx.x == 0) exps[b] = e;
    const float sc = ldexpf(1.f, e);
    // ---- write staged elements [q0, q1): padded position q -> source sample j
    auto src = [&](int64_t j) -> float {
      if (j >= h0 && j < h1) return sx[j - h0];
      return ld_cluster_f32(peer_sx + (uint32_t)((j - (rank ? 0 : L2)) * 4));
    };
    uint2* hrow = reinterpret_cast<uint2*>(hi + b * q_total);
    uint2* lrow = reinterpret_cast<uint2*>(lo + b * q_total);
    const int li0 = (int)h0, li1 = (int)h1, lpad = pad, lL = (int)L, lpl = (int)padded_len;
    for (int g4 = (int)(q0 / 4) + threadIdx.x; g4 < (int)(q1 / 4); g4 += blockDim.x) {
      float v[4];
      const int j0 = 4 * g4 - lpad;  // source of the group's first element (interior)
      if (j0 >= li0 && j0 + 3 < li1 && 4 * g4 + 3 < lpl) {  // interior of this half: smem only
        const int a = j0 - li0;
        if ((a & 3) == 0) {
          const float4 w = *reinterpret_cast<const float4*>(sx + a);
          v[0] = w.x;
          v[1] = w.y;
          v[2] = w.z;
          v[3] = w.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = sx[a + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] *= sc;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = 4 * g4 + u;
          float sv = 0.f;
          if (q < lpl) {
            int j = q - lpad;
            if (mode == NNAB_PAD_REFLECT) {
              if (j < 0) j = -j;
              if (j >= lL) j = 2 * (lL - 1) - j;
              sv = src(j);
            } else if (j >= 0 && j < lL) {
              sv = src(j);
            }
          }
          v[u] = sv * sc;
        }
      }
      __half2 h01 = __floats2half2_rn(v[0], v[1]), h23 = __floats2half2_rn(v[2], v[3]);
      uint2 hv;
      hv.x = *reinterpret_cast<uint32_t*>(&h01);
      hv.y = *reinterpret_cast<uint32_t*>(&h23);
      hrow[g4] = hv;
      if (split) {
        const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
        __half2 l01 = __floats2half2_rn(v[0] - f01.x, v[1] - f01.y);
        __half2 l23 = __floats2half2_rn(v[2] - f23.x, v[3] - f23.y);
        uint2 lv;
        lv.x = *reinterpret_cast<uint32_t*>(&l01);
        lv.y = *reinterpret_cast<uint32_t*>(&l23);
        lrow[g4] = lv;
      }
    }
    cluster_sync();  // the peer is done reading this half before the next clip overwrites it
  }
}

int stage_frames(const FrameGeom& g, const float* x, float* rows_hi, float* rows_lo, int split, cudaStream_t s) {
  const int64_t rows = g.B * (int64_t)g.R;
  if (rows == 0) return NNAB_OK;
  const int blocks = (int)std::min<int64_t>(rows, (int64_t)num_sms() * 16);
  stage_rows_kernel<<<blocks, 256, 0, s>>>(x, g.B, g.L, g.pad, g.pad_mode, g.hop, g.row_len, g.R, g.padded_len,
                                          split, rows_hi, rows_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

int stage_frames_f16(const FrameGeom& g, const float* x, void* rows_hi, void* rows_lo, int32_t* exps, int split,
                     cudaStream_t s) {
  if (g.B == 0) return NNAB_OK;
  if (g.row_len == g.hop && (g.L - ((g.L / 2) & ~int64_t(3))) <= kPairHalf && num_sms() >= 2 &&
      (int64_t)g.R * g.hop % 8 == 0) {
    // read once: clip halves in the shared memory of a two-CTA cluster
    const int64_t half = g.L - ((g.L / 2) & ~int64_t(3));
    const size_t smem = (size_t)half * 4;
    auto kern = stage_rows_f16_pair_kernel;
    NNAB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(g.B, num_sms() / 2)));
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    NNAB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, x, g.B, g.L, g.pad, g.pad_mode, g.hop, g.R, g.padded_len, split,
                                     reinterpret_cast<__half*>(rows_hi), reinterpret_cast<__half*>(rows_lo), exps));
    NNAB_LAUNCHED();
    return NNAB_OK;
  }
  // one clip per CTA at a time, one CTA per SM: 148 clips (47 MB) in flight, so pass 2
  // re-reads each clip from L2 (two CTAs per SM thrashed L2: 960 MB of DRAM reads, ncu)
  const int blocks = (int)std::min<int64_t>(g.B, (int64_t)num_sms());
  stage_rows_f16_kernel<<<blocks, 1024, 0, s>>>(x, g.B, g.L, g.pad, g.pad_mode, g.hop, g.row_len, g.R, g.padded_len,
                                               split, reinterpret_cast<__half*>(rows_hi),
                                               reinterpret_cast<__half*>(rows_lo), exps);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

// Bank operand layout: tile n = rows [2hb n, 2hb (n + 1)): hb cosine rows of bins hb n.. then
// the hb matching sine rows (hb = dft_half: 128, or the bin count rounded up to 8 for a one-tile
// bank, whose GEMM then runs N = 2 hb); K zero-padded to k_pad.
__global__ void pack_dft_bank_kernel(const float* __restrict__ h_re, const float* __restrict__ h_im, int32_t n_bins,
                                     int32_t n_fft, int32_t k_pad, int32_t n_tiles, int32_t fold, int32_t split,
                                     int32_t hb, float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = (int64_t)n_tiles * 2 * hb * k_pad;
  const int32_t n_body = fold ? n_bins - 1 : n_bins;  // bins held in the regular slots
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / k_pad;
    const int32_t k = (int32_t)(e - row * k_pad);
    const int32_t tile = (int32_t)(row / (2 * hb)), col = (int32_t)(row % (2 * hb));
    const bool is_sin = col >= hb;
    const int32_t bin = tile * hb + (is_sin ? col - hb : col);
    float v = 0.f;
    if (k < n_fft) {
      if (fold && tile == 0 && col == hb) {
        v = h_re[(int64_t)(n_bins - 1) * n_fft + k];  // Nyquist cosine in bin 0's (zero) sine slot
      } else if (bin < n_body) {
        v = (is_sin ? h_im : h_re)[(int64_t)bin * n_fft + k];
      }
    }
    const float h = tf32_rne(v);
    hi[e] = h;
    if (split) lo[e] = tf32_rne(v - h);
  }
}

// FP16 bank: |h| peak over both banks (as ordered bits of a non-negative float)
__global__ void bank_absmax_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                                   unsigned int* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fmaxf(fabsf(__ldg(a + i)), fabsf(__ldg(b + i))));
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

// The same tile layout as pack_dft_bank_kernel in FP16, scaled by 2^e_h (peak in
// [2^14, 2^15)); trailer[1] = e_h for the GEMM epilogue.
__global__ void pack_dft_bank_f16_kernel(const float* __restrict__ h_re, const float* __restrict__ h_im,
                                         int32_t n_bins, int32_t n_fft, int32_t k_pad, int32_t n_tiles, int32_t fold,
                                         int32_t split, int32_t hb, __half* __restrict__ hi,
                                         __half* __restrict__ lo, int32_t* __restrict__ trailer) {
  const int e = f16_scale_exp(__uint_as_float(static_cast<unsigned int>(trailer[0])));
  const float sc = ldexpf(1.f, e);
  if (blockIdx.x == 0 && threadIdx.x == 0) trailer[1] = e;
  const int64_t total = (int64_t)n_tiles * 2 * hb * k_pad;
  const int32_t n_body = fold ? n_bins - 1 : n_bins;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / k_pad;
    const int32_t k = (int32_t)(i - row * k_pad);
    const int32_t tile = (int32_t)(row / (2 * hb)), col = (int32_t)(row % (2 * hb));
    const bool is_sin = col >= hb;
    const int32_t bin = tile * hb + (is_sin ? col - hb : col);
    float v = 0.f;
    if (k < n_fft) {
      if (fold && tile == 0 && col == hb) v = h_re[(int64_t)(n_bins - 1) * n_fft + k];
      else if (bin < n_body) v = (is_sin ? h_im : h_re)[(int64_t)bin * n_fft + k];
    }
    v *= sc;
    const __half h = __float2half_rn(v);
    hi[i] = h;
    if (split) lo[i] = __float2half_rn(v - __half2float(h));
  }
}

int launch_bank_absmax(const float* a, const float* b, int64_t n, unsigned int* out, cudaStream_t s) {
  if (n <= 0) return NNAB_OK;
  bank_absmax_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(a, b, n, out);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

}  // namespace nnab

using namespace nnab;

// cosine (= sine) rows per DFT-layout tile: 128, or for a one-tile bank of <= 120 bins (not
// folded) the bin count rounded up to 8 -- its GEMMs then run N = 2 hb instead of 256
int nnab::dft_half(int32_t n_bins, int32_t fold_nyquist) {
  static const bool narrow = [] {
    const char* e = getenv("NNAB_DFT_NARROW");
    return !(e && e[0] == '0');
  }();
  return (narrow && !fold_nyquist && n_bins >= 1 && n_bins <= 120) ? (n_bins + 7) / 8 * 8 : 128;
}

extern "C" int nnab_dft_bank_tiles(int32_t n_bins, int32_t fold_nyquist) {
  if (n_bins < 1) return 0;
  const int body = fold_nyquist ? n_bins - 1 : n_bins;
  return std::max(1, (body + 127) / 128);
}

extern "C" size_t nnab_dft_bank_bytes(int32_t n_bins, int32_t n_fft, int32_t fold_nyquist) {
  const int64_t k_pad = (n_fft + 31) / 32 * 32;
  return (size_t)nnab_dft_bank_tiles(n_bins, fold_nyquist) * 2 * dft_half(n_bins, fold_nyquist) * k_pad *
         sizeof(float);
}

extern "C" size_t nnab_dft_bank_bytes_prec(int32_t n_bins, int32_t n_fft, int32_t fold_nyquist, int32_t precision) {
  if (!prec_is_f16(precision)) return nnab_dft_bank_bytes(n_bins, n_fft, fold_nyquist);
  const int64_t k_pad = (n_fft + 63) / 64 * 64;
  const size_t data = (size_t)nnab_dft_bank_tiles(n_bins, fold_nyquist) * 2 * dft_half(n_bins, fold_nyquist) * k_pad * 2;
  return ((data + 255) & ~size_t(255)) + 256;  // + trailer: [0] peak bits, [1] scale exponent
}

extern "C" int nnab_pack_dft_bank(const float* h_re, const float* h_im, int32_t n_bins, int32_t n_fft,
                                  int32_t fold_nyquist, int32_t precision, float* packed_hi, float* packed_lo,
                                  void* stream) {
  if (!h_re || !h_im || !packed_hi || n_bins < 1 || n_fft < 1) return NNAB_EINVAL;
  if (fold_nyquist && n_bins < 2) return NNAB_EINVAL;
  if (precision < NNAB_PREC_TF32 || precision > NNAB_PREC_3XF16) return NNAB_EINVAL;
  const int split = prec_is_split(precision);
  if (split && !packed_lo) return NNAB_EINVAL;
  const int32_t tiles = nnab_dft_bank_tiles(n_bins, fold_nyquist);
  cudaStream_t s = (cudaStream_t)stream;
  if (prec_is_f16(precision)) {
    const int32_t k_pad = (n_fft + 63) / 64 * 64;
    const int32_t hb = dft_half(n_bins, fold_nyquist);
    const int64_t total = (int64_t)tiles * 2 * hb * k_pad;
    int32_t* trailer = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(packed_hi) +
                                                  nnab_dft_bank_bytes_prec(n_bins, n_fft, fold_nyquist, precision) -
                                                  256);
    NNAB_CUDA_TRY(cudaMemsetAsync(trailer, 0, 8, s));
    const int64_t n = (int64_t)n_bins * n_fft;
    bank_absmax_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(
        h_re, h_im, n, reinterpret_cast<unsigned int*>(trailer));
    NNAB_LAUNCHED();
    pack_dft_bank_f16_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, s>>>(
        h_re, h_im, n_bins, n_fft, k_pad, tiles, fold_nyquist, split, hb, reinterpret_cast<__half*>(packed_hi),
        reinterpret_cast<__half*>(packed_lo), trailer);
    NNAB_LAUNCHED();
    return NNAB_OK;
  }
  const int32_t k_pad = (n_fft + 31) / 32 * 32;
  const int32_t hb = dft_half(n_bins, fold_nyquist);
  const int64_t total = (int64_t)tiles * 2 * hb * k_pad;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
  pack_dft_bank_kernel<<<blocks, 256, 0, s>>>(h_re, h_im, n_bins, n_fft, k_pad, tiles, fold_nyquist, split, hb,
                                              packed_hi, packed_lo);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

extern "C" int nnab_frames_geometry(const nnab_frames* f, int32_t* n_frames, int32_t* row_len, int32_t* rows) {
  FrameGeom g;
  int rc = frame_geometry(f, &g);
  if (rc) return rc;
  if (n_frames) *n_frames = g.T;
  if (row_len) *row_len = g.row_len;
  if (rows) *rows = g.R;
  return NNAB_OK;
}
