// CQT2010v2 on the tensor cores: the whole octave recursion of one clip in one
// CTA (one per SM, persistent over clips), every intermediate signal in shared
// memory, so HBM sees the clip once and the output once
// (transforms.py:290-313, signal.py:232-247).
//
// Operands are FP16 with an exact per-clip power-of-two scale 2^-e (e from the
// clip's peak), i.e. the same 11-bit significand as TF32 at twice the tcgen05
// rate (kind::f16, K = 16); accumulation is FP32 and the scale is undone exactly
// in the conv epilogue.  The peak comes from a dedicated scan warp that streams
// the NEXT clip through a bulk-copy ring while the other warps work on the
// current one (so the clip is in L2 when stage 1 reads it).
//
// Half-band FIR as a banded Toeplitz MMA.  downsample2 keeps
//   y[i] = sum_d h[d] x_ext[2i + d],  d = -127..127 (reflect-extended x)
// and the cutoff-0.5 windowed sinc is half-band: every even d != 0 is <= 6.6e-17,
// so  y[i] = h0 * x[2i] + sum_{j<128} g_j * xo[i + j],  g_j = h[2j - 127],
// xo[m] = x_ext[2m - 127] (the odd phase).  A block of 128 outputs is
// Y[r] = sum_s T[r][s] W[s], T[r][s] = g_{s-r} (128 x 256 Toeplitz band), W = 256
// consecutive odd-phase samples; windows of consecutive blocks overlap by 128.
//   A = "planes": the odd phase stored once as rows of 128 samples, plane q
//       holding the 16-byte chunk q of every row (rows 16 B apart); block n's
//       window is rows n, n+1, i.e. a 16-byte start offset (LBO = plane stride);
//       M = 128 blocks per MMA.
//   B = T with its rows reversed: T'[r'][s] = g[s + r' - 127] depends on s + r'
//       only, so the band lives in a 6 KB "diagonal" array (chunk j = 8 taps
//       g[j-127 ..]) that a no-swizzle K-major descriptor with LBO = SBO = 128 B
//       walks; N = 128 output offsets.
//   D[block][r'] in TMEM: each lane holds 128 consecutive outputs of one block,
//       so the epilogue writes 16-byte vectors.
// Each epilogue writes its signal straight into the next stage's layouts (odd
// phase -> planes, even phase / contiguous copy with reflect margins -> centre
// taps and conv frames); a small edge pass adds the reflect images.
// Per-octave centred complex conv (<= 16 bins x <= 96 taps, hop h >> alpha):
// frames as N (im2col B tile, <= 256 frames), the filter bank as A (M = 128
// rows, re/im of bin j at row 32 (j % 4) + 2 (j / 4) + {0, 1} so every TMEM lane
// quarter carries bins), D = 128 x frames.
#include <algorithm>
#include <cmath>

#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kCompute = 256;             // warps 0-7: MMA issue (thread 0), builds, epilogues
constexpr int kThreads = kCompute + 64;   // warp 8: scan of the next clip; warp 9: MMA issue
constexpr int kTile1 = 128;               // stage-1 blocks per MMA tile (= M)
constexpr int ML = 128;                   // reflect margins of the contiguous signal copies (fp16)
constexpr int KC = 96;                    // conv taps (K), padded
constexpr int kFiltLog2 = 6;              // conv bank scaled by 2^6 before the FP16 rounding
constexpr int kMaxOct = 12;
constexpr int TOEP_CHUNKS = 8 * 31 + 128;  // 376 diagonal chunks of 8 taps
constexpr uint32_t kConvCol = 256;          // TMEM columns of the conv accumulators (2 x 32)
constexpr int NCONV = 32;                   // conv N: re/im rows of <= 16 bins
constexpr uint32_t kRing = 16384;           // scan ring slot (bytes), 2 slots

struct TcParams {
  const float* x;
  int64_t B, L;
  int32_t L1, L0, n1_tiles;
  int32_t n_oct, kernel_hop, first_bin, bpo, n_bins, n_filt, width, T, out_kind;
  int32_t pad, pad_al, rows2;          // conv pad, pad rounded to 8, rows of the (compact) second frame tile
  int32_t oct_len[kMaxOct];            // signal length of octave alpha
  int32_t oct_blocks[kMaxOct];         // 128-output blocks of the halving producing octave alpha
  int32_t plane_rows[kMaxOct];         // rows of octave alpha's odd-phase planes (feed halving alpha+1)
  int32_t s_off[kMaxOct];              // smem offset of octave alpha's contiguous copy (with ML margins)
  int32_t o_off[kMaxOct];              // smem offset of octave alpha's planes
  float h0;                            // centre tap
  float g[128];                        // odd taps g_j = h[2j - 127]
  const float* k_re;                   // top-octave bank (n_filt, width), device
  const float* k_im;
  float* out;
  // front-only mode (lv0 != null): after stage 2 the octave-0 signal (scaled FP16 with its
  // ML-sample reflect margins) goes to lv0[b * lv0_stride ..] and the clip's scale
  // exponent to lv_exp[b]; the octave levels then run as batched kernels
  __half* lv0;
  int32_t* lv_exp;
  int32_t lv0_stride;
  // lv_mode 2 ("no-conv"): the kernel also runs the halvings and writes every octave to
  // lv[a] (stride lv_stride[a]); the convs of all octaves then run as one batched launch
  int32_t lv_mode;
  __half* lv[kMaxOct];
  int32_t lv_stride[kMaxOct];
  // shared-memory carve-up (bytes from the 1 KB-aligned base)
  int32_t off_toep, off_filt, off_ring, off_x, off_xe, off_y, off_ye, off_col, off_stage, off_bars;
  int32_t pl_x, pl_y, y_rows;          // plane strides (bytes); stage-2 plane rows
  unsigned long long* prof;            // optional per-phase cycle counters (nnab_debug_cqt2010_profile)
};

// Phase clock of thread 0 (only when p.prof is set); accumulators in shared memory.
struct Prof {
  long long t = 0;
  unsigned long long* acc = nullptr;  // [16]
  NNAB_DEV void mark(const TcParams& p, int i) {
    if (p.prof && threadIdx.x == 0) {
      const long long n = clock64();
      acc[i] += (unsigned long long)(n - t);
      t = n;
    }
  }
};

NNAB_DEV void csync() { asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory"); }  // compute warps only

NNAB_DEV uint64_t nsw_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {  // no-swizzle K-major
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// byte offset of odd-phase sample m inside a plane set of stride pl
NNAB_DEV uint32_t plane_off(int m, uint32_t pl) {
  return (uint32_t)((m & 127) >> 3) * pl + (uint32_t)(m >> 7) * 16u + (uint32_t)(m & 7) * 2u;
}

NNAB_DEV __half h16(float v) { return __float2half_rn(v); }

// Contiguous FP16 signal arrays in shared memory are read and written by lanes
// 128 samples apart (lane = block); the 16-byte chunk index inside each 256-byte
// row is XORed with the row index so those accesses spread over all banks.
// Aligned runs of <= 8 samples stay contiguous; arrays are whole 128-sample rows.
NNAB_DEV int sw(int i) { return i ^ (((i >> 7) & 15) << 3); }
NNAB_DEV uint4 ld8(const __half* a, int i) { return *reinterpret_cast<const uint4*>(a + sw(i)); }
NNAB_DEV void st8(__half* a, int i, uint4 v) { *reinterpret_cast<uint4*>(a + sw(i)) = v; }

struct Ctx {
  const TcParams& p;
  uint8_t* base;
  uint32_t tmem;
  uint64_t* bar;  // MMA completion
  uint32_t phase;
  Prof pf;
  NNAB_DEV void wait_mma() {
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
  }
};

// Toeplitz FIR of 128 consecutive blocks (plane rows row0 ..) into TMEM column
// d_col; thread 0 only, the caller commits.  Rows past a signal's end only feed
// discarded blocks (they may hold anything; the descriptors stay in smem).
NNAB_DEV void issue_fir(Ctx& c, uint32_t planes, uint32_t pl, int row0, uint32_t d_col) {
  tc_fence_after();
  constexpr uint32_t idesc = idesc_f16(128, 128);
  const uint32_t toep = smem_u32(c.base + c.p.off_toep);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint64_t a = nsw_desc(planes + (uint32_t)(2 * (k & 7)) * pl + (uint32_t)(row0 + (k >> 3)) * 16u, pl, 128);
    const uint64_t b = nsw_desc(toep + 256u * k, 128, 128);
    mma_f16(c.tmem + d_col, a, b, idesc, k > 0);
  }
}

// Epilogue of a FIR tile: lane = block n = blk0 + TMEM lane, column r' = 127 - r.
// Warp w reads lane quarter w & 3 and column half w >> 2 in four chunks of 16
// columns = 16 consecutive outputs i0 .. i0+15 (i0 = 128 n + rbase).
// cen16(i0, c) loads their centre-tap samples, out16(i0, y) stores them
// (vectorised); cen1 / out1 handle the last, partial chunk of a signal.  Blocks
// below blk_lo (already written by an overlapping tile) are skipped.
template <class Cen16, class Cen1, class Out16, class Out1>
NNAB_DEV void fir_epilogue(Ctx& c, int blk0, int blk_lo, int n_out, uint32_t d_col, float h0, Cen16 cen16, Cen1 cen1,
                           Out16 out16, Out1 out1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  const int n = blk0 + q * 32 + lane;
  const uint32_t ta = c.tmem + ((uint32_t)(q * 32) << 16) + d_col + half * 64;
#pragma unroll 1
  for (int k = 0; k < 4; ++k) {
    const int rbase = 112 - 64 * half - 16 * k;  // columns half*64 + 16k .. +15 hold r = rbase+15 .. rbase
    const int i0 = n * 128 + rbase;
    float v[16], y[16];
    tmem_ld16(ta + 16 * k, v);
    const bool live = n >= blk_lo && i0 < n_out;
    const bool full = i0 + 16 <= n_out;
    if (live) {
      if (full) {
        cen16(i0, y);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) y[e] = i0 + e < n_out ? cen1(i0 + e) : 0.f;
      }
    }
    tmem_ld_wait();
    if (live) {
#pragma unroll
      for (int e = 0; e < 16; ++e) y[e] = fmaf(h0, y[e], v[15 - e]);
      if (full) {
        out16(i0, y);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (i0 + e < n_out) out1(i0 + e, y[e]);
      }
    }
  }
}

// 8 consecutive odd-phase samples m0 .. m0+7 (m0 % 8 == 0) -> one plane chunk
NNAB_DEV void store_planes8(uint8_t* planes, uint32_t pl, int rows, int m0, const __half2* h) {
  if ((m0 >> 7) < rows)
    *reinterpret_cast<uint4*>(planes + (uint32_t)((m0 & 127) >> 3) * pl + (uint32_t)(m0 >> 7) * 16u) =
        *reinterpret_cast<const uint4*>(h);
}
NNAB_DEV void store_plane1(uint8_t* planes, uint32_t pl, int rows, int m, __half v) {
  if (m >= 0 && (m >> 7) < rows) *reinterpret_cast<__half*>(planes + plane_off(m, pl)) = v;
}
// outputs y[0..15] of i0 .. i0+15 (i0 % 16 == 0): odd ones (planes at
// m = (i + 127) / 2 = i0 / 2 + 64 + u), even ones, all of them (contiguous copy)
NNAB_DEV void pack_odd(const float* y, __half2* o) {
#pragma unroll
  for (int u = 0; u < 4; ++u) o[u] = __floats2half2_rn(y[4 * u + 1], y[4 * u + 3]);
}
NNAB_DEV void pack_even(const float* y, __half2* o) {
#pragma unroll
  for (int u = 0; u < 4; ++u) o[u] = __floats2half2_rn(y[4 * u], y[4 * u + 2]);
}
NNAB_DEV void pack_all(const float* y, __half2* o) {
#pragma unroll
  for (int u = 0; u < 8; ++u) o[u] = __floats2half2_rn(y[2 * u], y[2 * u + 1]);
}
NNAB_DEV void unpack8(uint4 w, float* f) {
  const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float2 t = __half22float2(h2[u]);
    f[2 * u] = t.x;
    f[2 * u + 1] = t.y;
  }
}

// Edge pass of a signal of length n held as a contiguous copy s (with ML margins)
// and, optionally, odd-phase planes: the reflect images (np.pad "reflect",
// signal.py:245) from the stored samples.  One image per thread.
NNAB_DEV void edge_pass(__half* s, uint8_t* planes, uint32_t pl, int rows, int n) {
  for (int e = threadIdx.x; e < 2 * ML; e += kCompute) {
    const int i = e < ML ? e + 1 : n - 1 - ML + (e - ML);  // left: 1..ML, right: n-1-ML .. n-2
    const int dst = e < ML ? -i : 2 * (n - 1) - i;         // ext position of the image
    const __half v = s[sw(ML + i)];
    s[sw(ML + dst)] = v;
    if (planes && (dst & 1)) store_plane1(planes, pl, rows, (dst + 127) >> 1, v);
  }
}

// Stage-1 operands of blocks [n0, n0 + nb): odd-phase planes (rows 0 .. nb) and
// the even phase (centre taps, xe[u] = x[2 (128 n0 + u)]), scaled, FP16.
// The tile's clip range x_ext[256 n0 - 128 .. 256 (n0 + nb + 1) - 128) is read
// with coalesced float4 loads (lane = consecutive 16 bytes): float4 g holds odd
// samples m = 128 n0 + 2g, +1 (one 4-byte store into the planes, whose stride is
// padded off 128 B so the eight chunks a warp touches hit different banks) and
// even samples u = 2g - 64, +1 (one 4-byte store into xe).
NNAB_DEV void build_x(Ctx& c, const float* xb, float scale, int n0, int nb, bool vec) {
  const TcParams& p = c.p;
  uint8_t* planes = c.base + p.off_x;
  __half* xe = reinterpret_cast<__half*>(c.base + p.off_xe);
  const int64_t L = p.L;
  const int64_t j_start = 256 * (int64_t)n0 - 128;
  const int n4 = (nb + 1) * 64;  // float4 groups
  constexpr int kPer = 8;        // groups in flight per thread
  for (int g0 = threadIdx.x; g0 < n4; g0 += kPer * kCompute) {
    float4 f[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int g = g0 + u * kCompute;
      const int64_t j = j_start + 4 * (int64_t)g;
      if (g >= n4) {
        f[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else if (vec && j >= 0 && j + 4 <= L) {
        f[u] = __ldg(reinterpret_cast<const float4*>(xb + j));
      } else {
        float e[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int64_t jj = j + k;
          if (jj < 0) jj = -jj;
          if (jj >= L) jj = 2 * (L - 1) - jj;
          e[k] = (jj >= 0 && jj < L) ? __ldg(xb + jj) : 0.f;  // beyond one reflection: never a kept output
        }
        f[u] = make_float4(e[0], e[1], e[2], e[3]);
      }
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int g = g0 + u * kCompute;
      if (g >= n4) continue;
      const int m = 2 * g;  // odd-phase index relative to 128 n0
      *reinterpret_cast<__half2*>(planes + (uint32_t)((m & 127) >> 3) * p.pl_x + (uint32_t)(m >> 7) * 16u +
                                  (uint32_t)(m & 7) * 2u) = __floats2half2_rn(f[u].y * scale, f[u].w * scale);
      const int ue = 2 * g - 64;
      if (ue >= 0 && ue < nb * 128) *reinterpret_cast<__half2*>(xe + sw(ue)) = __floats2half2_rn(f[u].x * scale, f[u].z * scale);
    }
  }
}

// im2col A tiles of octave alpha's conv, frames t0 .. t0 + 255 x 96 taps (FP16,
// no-swizzle K-major): tile 0 (128 frames) has chunk cc (8 taps) at cc * 2048 and
// frame t at t * 16; tile 1 is compact (rows2 rows, chunk stride rows2 * 16) --
// its MMA also reads rows past rows2, which only feed discarded frames.  Column m
// holds signal sample t*h - pad_al + m (the bank is shifted by pad_al - pad).
NNAB_DEV uint4 frame_chunk(const TcParams& p, const __half* sig, int h, int tt, int cc) {
  if (tt >= p.T) return make_uint4(0, 0, 0, 0);
  const int s0 = ML + tt * h - p.pad_al + cc * 8;
  if ((h & 7) == 0) return ld8(sig, s0);
  __align__(16) __half hv[8];
  if ((h & 3) == 0) {
    *reinterpret_cast<uint2*>(hv) = *reinterpret_cast<const uint2*>(sig + sw(s0));
    *reinterpret_cast<uint2*>(hv + 4) = *reinterpret_cast<const uint2*>(sig + sw(s0 + 4));
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) hv[k] = sig[sw(s0 + k)];
  }
  return *reinterpret_cast<uint4*>(hv);
}
NNAB_DEV void build_frames(Ctx& c, const __half* sig, int h, int t0, int ntile) {
  // thread = frame t0 + tid (tile 0: tid < 128, tile 1: the first rows2 frames after);
  // its 12 chunk loads are issued before any store
  const TcParams& p = c.p;
  const int t = threadIdx.x;
  uint8_t* dst;
  uint32_t cstride;
  if (t < 128) {
    dst = c.base + p.off_col + t * 16;
    cstride = 2048;
  } else {
    if (ntile < 2 || t - 128 >= p.rows2) return;
    dst = c.base + p.off_col + 128 * KC * 2 + (t - 128) * 16;
    cstride = (uint32_t)p.rows2 * 16u;
  }
  const int tt = t0 + t;
  if (h < 8 && (h & 1) == 0 && tt < p.T) {
    // short hops (the top octaves): the frame's 96 taps start 2*sh halves past an
    // 8-aligned position -- 13 aligned 16-byte loads, each chunk four 32-bit words
    // of two neighbours picked by two select levels, instead of 8 (h = 2) or 2
    // (h = 4) narrow swizzled loads per chunk
    const int s_base = ML + tt * h - p.pad_al;
    const int a0 = s_base & ~7, sh = (s_base & 7) >> 1;
    uint4 q0 = ld8(sig, a0);
#pragma unroll
    for (int cc = 0; cc < KC / 8; ++cc) {
      const uint4 q1 = ld8(sig, a0 + 8 * (cc + 1));
      const uint32_t e[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      uint32_t f[5];
#pragma unroll
      for (int j = 0; j < 5; ++j) f[j] = (sh & 2) ? e[j + 2] : e[j];
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = (sh & 1) ? f[j + 1] : f[j];
      *reinterpret_cast<uint4*>(dst + cc * cstride) = make_uint4(o[0], o[1], o[2], o[3]);
      q0 = q1;
    }
    return;
  }
  uint4 v[KC / 8];
#pragma unroll
  for (int cc = 0; cc < KC / 8; ++cc) v[cc] = frame_chunk(p, sig, h, tt, cc);
#pragma unroll
  for (int cc = 0; cc < KC / 8; ++cc) *reinterpret_cast<uint4*>(dst + cc * cstride) = v[cc];
}

NNAB_DEV void issue_conv(Ctx& c, int ntile) {
  tc_fence_after();
  constexpr uint32_t idesc = idesc_f16(128, NCONV);
  const uint32_t a0 = smem_u32(c.base + c.p.off_col), b0 = smem_u32(c.base + c.p.off_filt);
  for (int u = 0; u < ntile; ++u) {
    const uint32_t au = a0 + (u ? 128 * KC * 2 : 0), lbo = u ? (uint32_t)c.p.rows2 * 16u : 2048u;
#pragma unroll
    for (int k = 0; k < KC / 16; ++k)
      mma_f16(c.tmem + kConvCol + 32 * u, nsw_desc(au + 2 * k * lbo, lbo, 128), nsw_desc(b0 + 2 * k * 512, 512, 128),
              idesc, k > 0);
  }
}

// conv epilogue: warp w reads lane quarter w & 3 of tile w >> 2: thread = frame,
// columns 2j, 2j+1 = re, im of bin j; stores coalesced along T.
NNAB_DEV void conv_epilogue(Ctx& c, int alpha, int64_t b, int t0, int ntile, float out_scale, float* stage) {
  const TcParams& p = c.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, u = warp >> 2;
  if (u >= ntile) return;
  const int skip = max(0, alpha * p.bpo - p.first_bin);
  const int row0 = p.first_bin - alpha * p.bpo;
  const int t = t0 + u * 128 + q * 32 + lane;
  float v[32];
  tmem_ld32(c.tmem + ((uint32_t)(q * 32) << 16) + kConvCol + 32 * u, v);
  tmem_ld_wait();
  if (t >= p.T) return;
#pragma unroll
  for (int j = 0; j < NCONV / 2; ++j) {
    if (j < skip || j >= p.n_filt) continue;
    const float re = v[2 * j] * out_scale, im = v[2 * j + 1] * out_scale;
    if (stage) {  // the octave's rows are one aligned block of the output: staged, bulk-stored
      stage[(j - skip) * p.T + t] = p.out_kind == NNAB_OUT_POWER ? fmaf(re, re, im * im)
                                                                 : fast_sqrt(fmaf(re, re, im * im));
      continue;
    }
    const int64_t o = (b * p.n_bins + row0 + j) * (int64_t)p.T + t;
    if (p.out_kind == NNAB_OUT_COMPLEX) {
      reinterpret_cast<float2*>(p.out)[o] = make_float2(re, im);
    } else if (p.out_kind == NNAB_OUT_POWER) {
      p.out[o] = fmaf(re, re, im * im);
    } else {
      p.out[o] = fast_sqrt(fmaf(re, re, im * im));
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) cqt2010_tc_kernel(const __grid_constant__ TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // bars[0] FIR MMAs done, [1..2] scan ring, [3] scale published, [4] scan may start the next clip,
  // [5] conv MMAs done, [6] FIR operands ready, [7] conv operands ready
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + p.off_bars);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
  volatile int* scale_exp = reinterpret_cast<volatile int*>(bars + 9);
  __shared__ unsigned long long prof_acc[16];
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool vec = (p.L % 4) == 0;

  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tslot);
  if (tid < 16) prof_acc[tid] = 0;
  // zero the signal regions once: windows of real blocks read rows past a signal's
  // end at zero Toeplitz weight, and 0 * NaN would poison them (everything written
  // later is finite)
  for (int i = tid; i < (p.off_bars - p.off_x) / 16; i += kThreads)
    reinterpret_cast<uint4*>(base + p.off_x)[i] = make_uint4(0, 0, 0, 0);
  // diagonal Toeplitz chunks: chunk j = g[j - 127 + e], e < 8
  for (int j = tid; j < TOEP_CHUNKS; j += kThreads) {
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int gi = j - 127 + e;
      v[e] = h16((gi >= 0 && gi < 128) ? p.g[gi] : 0.f);
    }
    *reinterpret_cast<uint4*>(base + p.off_toep + 16 * j) = *reinterpret_cast<uint4*>(v);
  }
  // conv bank B (N = 32 rows x 96 taps): row 2j = Re bin j, 2j+1 = Im; chunk cc at cc * 512,
  // row at 16 B; column m holds tap m - shift
  const int shift = p.pad_al - p.pad;
  for (int e = tid; e < NCONV * KC; e += kThreads) {
    const int n = e / KC, m = e % KC, j = n >> 1, tap = m - shift;
    float v = 0.f;
    if (j < p.n_filt && tap >= 0 && tap < p.width)
      v = ldexpf(((n & 1) ? p.k_im : p.k_re)[(int64_t)j * p.width + tap], kFiltLog2);
    *reinterpret_cast<__half*>(base + p.off_filt + (m >> 3) * 512 + n * 16 + (m & 7) * 2) = h16(v);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == kCompute / 32) {
    // ------------------------------------------------ scan warp: peak of each clip of this CTA
    const int lane = tid & 31;
    const uint64_t keep = policy_evict_last();
    uint32_t seq = 0;  // ring uses (slot = seq & 1, parity = seq >> 1)
    int k = 0;
    for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++k) {
      if (k > 0) mbar_wait(&bars[4], (k - 1) & 1);  // the previous clip finished stage 1
      const float* xb = p.x + b * p.L;
      float mx = 0.f;
      if (vec) {
        const uint32_t bytes = (uint32_t)(p.L * 4);
        const int nch = (int)((bytes + kRing - 1) / kRing);
        auto issue = [&](int ch) {
          const uint32_t sz = min((uint32_t)kRing, bytes - (uint32_t)ch * kRing);
          const uint32_t s = (seq + ch) & 1;
          mbar_expect_tx(&bars[1 + s], sz);
          // keep the clip in L2 for stage 1, which reads it again after this scan
          bulk_load_hint(base + p.off_ring + s * kRing, reinterpret_cast<const char*>(xb) + (size_t)ch * kRing, sz,
                         &bars[1 + s], keep);
        };
        if (lane == 0)
          for (int ch = 0; ch < 2 && ch < nch; ++ch) issue(ch);
        for (int ch = 0; ch < nch; ++ch) {
          const uint32_t s = seq + ch;
          mbar_wait(&bars[1 + (s & 1)], (s >> 1) & 1);
          const uint32_t sz = min((uint32_t)kRing, bytes - (uint32_t)ch * kRing);
          const float4* b4 = reinterpret_cast<const float4*>(base + p.off_ring + (s & 1) * kRing);
          for (int i = lane; i < (int)(sz / 16); i += 32) {
            const float4 a = b4[i];
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
          }
          __syncwarp();
          if (lane == 0 && ch + 2 < nch) issue(ch + 2);
        }
        seq += (uint32_t)nch;
      } else {
        for (int64_t i = lane; i < p.L; i += 32) mx = fmaxf(mx, fabsf(__ldg(xb + i)));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) {
        int ex = 0;
        if (mx > 0.f && mx < INFINITY) frexpf(mx, &ex);
        *scale_exp = ex;
        mbar_arrive(&bars[3]);
      }
      __syncwarp();
    }
  } else if (warp == kCompute / 32 + 1) {
    // ------------------------------------------------ MMA issue warp: the compute warps' schedule,
    // each step waiting for its operands to be ready (the issue of a tcgen05.mma chain
    // blocks its thread for ~100 cycles per instruction, which no compute warp pays now)
    if (elect_one()) {
      Ctx c{p, base, *tslot, &bars[0], 0, {}};
      uint32_t go_fir = 0, go_conv = 0;
      auto wait_fir = [&]() { mbar_wait(&bars[6], go_fir); go_fir ^= 1; };
      auto wait_conv = [&]() { mbar_wait(&bars[7], go_conv); go_conv ^= 1; };
      const uint32_t xp_s = smem_u32(base + p.off_x), yp_s = smem_u32(base + p.off_y);
      for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
        for (int t = 0; t < p.n1_tiles; ++t) {
          wait_fir();
          issue_fir(c, xp_s, p.pl_x, 0, 0);
          mma_commit(&bars[0]);
        }
        wait_fir();
        issue_fir(c, yp_s, p.pl_y, 0, 0);
        if (p.oct_blocks[0] > 128) issue_fir(c, yp_s, p.pl_y, p.oct_blocks[0] - 128, 128);
        mma_commit(&bars[0]);
        if (p.lv0) {  // the octave levels (mode 1) or just the convs (mode 2) run as batched kernels
          if (p.lv_mode == 2)
            for (int a = 0; a + 1 < p.n_oct; ++a) {
              wait_fir();
              issue_fir(c, smem_u32(base + p.o_off[a]), (uint32_t)p.plane_rows[a] * 16u, 0, 0);
              mma_commit(&bars[0]);
            }
          continue;
        }
        for (int a = 0; a < p.n_oct; ++a) {
          if (a + 1 < p.n_oct) {
            wait_fir();
            issue_fir(c, smem_u32(base + p.o_off[a]), (uint32_t)p.plane_rows[a] * 16u, 0, 0);
            mma_commit(&bars[0]);
          }
          for (int t0 = 0; t0 < p.T; t0 += 256) {
            wait_conv();
            issue_conv(c, min(2, (p.T - t0 + 127) / 128));
            mma_commit(&bars[5]);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ compute warps
    Ctx c{p, base, *tslot, &bars[0], 0, {}};
    c.pf.acc = prof_acc;
    if (p.prof && tid == 0) c.pf.t = clock64();
    uint8_t* xp = base + p.off_x;
    uint8_t* yp = base + p.off_y;
    __half* xe = reinterpret_cast<__half*>(base + p.off_xe);
    __half* ye = reinterpret_cast<__half*>(base + p.off_ye);
    const uint32_t xp_s = smem_u32(xp), yp_s = smem_u32(yp);
    uint64_t* conv_bar = &bars[5];
    uint32_t conv_phase = 0;
    int k = 0;
    for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++k) {
      const float* xb = p.x + b * p.L;
      mbar_wait(&bars[3], k & 1);
      const int ex = *scale_exp;
      const float scale = ldexpf(1.f, -ex), out_scale = ldexpf(1.f, ex - kFiltLog2);
      c.pf.mark(p, 12);

      // -------------------------------------------- stage 1: x -> y1 (odd -> planes, even -> ye)
      const int L1 = p.L1;
      for (int t = 0; t < p.n1_tiles; ++t) {
        const int nb = min(kTile1, (L1 - t * kTile1 * 128 + 127) / 128);
        build_x(c, xb, scale, t * kTile1, nb, vec);
        fence_proxy_async_smem();
        csync();
        c.pf.mark(p, 0);
        if (tid == 0) mbar_arrive(&bars[6]);  // operands ready: the issue warp runs the FIR
        c.wait_mma();
        c.pf.mark(p, 1);
        const int u_base = t * kTile1 * 128;
        fir_epilogue(
            c, t * kTile1, 0, L1, 0, p.h0,
            [&](int i0, float* cv) {
              unpack8(ld8(xe, i0 - u_base), cv);
              unpack8(ld8(xe, i0 - u_base + 8), cv + 8);
            },
            [&](int i) { return __half2float(xe[sw(i - u_base)]); },
            [&](int i0, const float* y) {
              __align__(16) __half2 od[4], ev[4];
              pack_odd(y, od);
              pack_even(y, ev);
              store_planes8(yp, p.pl_y, p.y_rows, i0 / 2 + 64, od);
              st8(ye, i0 / 2, *reinterpret_cast<const uint4*>(ev));
            },
            [&](int i, float y) {
              if (i & 1) store_plane1(yp, p.pl_y, p.y_rows, (i + 127) >> 1, h16(y));
              else ye[sw(i >> 1)] = h16(y);
            });
        tc_fence_before();
        csync();
        c.pf.mark(p, 2);
      }
      if (tid == 0) mbar_arrive(&bars[4]);  // x of this clip is no longer needed: scan the next one
      // reflect images of y1's odd phase (left: -i, right: 2(L1-1) - i, i odd)
      for (int e = tid; e < 128; e += kCompute) {
        const int i = e < 64 ? 2 * e + 1 : ((L1 - 128) | 1) + 2 * (e - 64);
        const int dst = e < 64 ? -i : 2 * (L1 - 1) - i;
        if (i <= L1 - 2)
          store_plane1(yp, p.pl_y, p.y_rows, (dst + 127) >> 1,
                       *reinterpret_cast<const __half*>(yp + plane_off((i + 127) >> 1, p.pl_y)));
      }
      fence_proxy_async_smem();
      csync();

      // epilogue functors of a halving whose output goes to a contiguous copy + planes
      auto out16_of = [&](__half* dst, uint8_t* planes, uint32_t pl, int rows) {
        return [=](int i0, const float* y) {
          __align__(16) __half2 al[8];
          pack_all(y, al);
          st8(dst, ML + i0, reinterpret_cast<const uint4*>(al)[0]);
          st8(dst, ML + i0 + 8, reinterpret_cast<const uint4*>(al)[1]);
          if (planes) {
            __align__(16) __half2 od[4];
            pack_odd(y, od);
            store_planes8(planes, pl, rows, i0 / 2 + 64, od);
          }
        };
      };
      auto out1_of = [&](__half* dst, uint8_t* planes, uint32_t pl, int rows) {
        return [=](int i, float y) {
          const __half v = h16(y);
          dst[sw(ML + i)] = v;
          if (planes && (i & 1)) store_plane1(planes, pl, rows, (i + 127) >> 1, v);
        };
      };
      auto sig = [&](int a) { return reinterpret_cast<__half*>(base + p.s_off[a]); };
      auto planes_of = [&](int a) { return a + 1 < p.n_oct ? base + p.o_off[a] : nullptr; };

      // -------------------------------------------- stage 2: y1 -> octave 0
      {
        const int n2 = p.oct_len[0], nb2 = p.oct_blocks[0];
        const int row_b = nb2 > 128 ? nb2 - 128 : 0;  // second tile: the last 128 blocks
        if (tid == 0) mbar_arrive(&bars[6]);
        c.wait_mma();
        c.pf.mark(p, 4);
        uint8_t* o0 = planes_of(0);
        const uint32_t pl0 = (uint32_t)p.plane_rows[0] * 16u;
        auto cen16 = [&](int i0, float* cv) {
          unpack8(ld8(ye, i0), cv);
          unpack8(ld8(ye, i0 + 8), cv + 8);
        };
        auto cen1 = [&](int i) { return __half2float(ye[sw(i)]); };
        fir_epilogue(c, 0, 0, n2, 0, p.h0, cen16, cen1, out16_of(sig(0), o0, pl0, p.plane_rows[0]),
                     out1_of(sig(0), o0, pl0, p.plane_rows[0]));
        if (nb2 > 128)
          fir_epilogue(c, row_b, 128, n2, 128, p.h0, cen16, cen1, out16_of(sig(0), o0, pl0, p.plane_rows[0]),
                       out1_of(sig(0), o0, pl0, p.plane_rows[0]));
        csync();
        edge_pass(sig(0), o0, pl0, p.plane_rows[0], n2);
        fence_proxy_async_smem();
        tc_fence_before();
        csync();
        c.pf.mark(p, 5);
      }
      if (p.lv0) {
        // front-only: octave 0 with its reflect margins (positions [0, n0 + 2 ML)) to the
        // level buffer, zero past them; the next clip's stage 1 reuses this region
        const int n_valid = p.oct_len[0] + 2 * ML;
        __half* dst = p.lv0 + b * (int64_t)p.lv0_stride;
        const __half* src = sig(0);
        for (int k8 = tid; k8 < p.lv0_stride / 8; k8 += kCompute) {
          uint4 v = ld8(src, 8 * k8);
          if (8 * k8 + 8 > n_valid) {
            __half* hv = reinterpret_cast<__half*>(&v);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (8 * k8 + e >= n_valid) hv[e] = __float2half(0.f);
          }
          *reinterpret_cast<uint4*>(dst + 8 * k8) = v;
        }
        if (tid == 0) p.lv_exp[b] = ex;
        csync();
        if (p.lv_mode != 2) continue;
        // no-conv mode: the halvings, each octave to its level buffer
        for (int a = 0; a + 1 < p.n_oct; ++a) {
          if (tid == 0) mbar_arrive(&bars[6]);  // octave a's planes are ready: the issue warp runs the FIR
          c.wait_mma();
          const __half* sp = sig(a);
          __half* sd = sig(a + 1);
          uint8_t* po = planes_of(a + 1);
          const uint32_t pl_out = (uint32_t)p.plane_rows[a + 1] * 16u;
          const int n_out = p.oct_len[a + 1];
          fir_epilogue(
              c, 0, 0, n_out, 0, p.h0,
              [&](int i0, float* cv) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  const uint4 w = ld8(sp, ML + 2 * i0 + 8 * kk);
                  const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
                  for (int u = 0; u < 4; ++u) cv[4 * kk + u] = __low2float(h2[u]);
                }
              },
              [&](int i) { return __half2float(sp[sw(ML + 2 * i)]); }, out16_of(sd, po, pl_out, p.plane_rows[a + 1]),
              out1_of(sd, po, pl_out, p.plane_rows[a + 1]));
          tc_fence_before();
          csync();
          edge_pass(sd, po, pl_out, p.plane_rows[a + 1], n_out);
          fence_proxy_async_smem();
          csync();
          const int nv = n_out + 2 * ML;
          __half* dst = p.lv[a + 1] + b * (int64_t)p.lv_stride[a + 1];
          for (int k8 = tid; k8 < p.lv_stride[a + 1] / 8; k8 += kCompute) {
            uint4 v = ld8(sd, 8 * k8);
            if (8 * k8 + 8 > nv) {
              __half* hv = reinterpret_cast<__half*>(&v);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (8 * k8 + e >= nv) hv[e] = __float2half(0.f);
            }
            *reinterpret_cast<uint4*>(dst + 8 * k8) = v;
          }
        }
        csync();
        continue;
      }

      // -------------------------------------------- octaves, software-pipelined: the halving
      // alpha+1 MMA runs under the im2col of alpha, the conv alpha MMA under the
      // halving alpha+1 epilogue
      for (int a = 0; a < p.n_oct; ++a) {
        const int h = p.kernel_hop >> a;
        const bool halve = a + 1 < p.n_oct;
        if (halve && tid == 0) mbar_arrive(&bars[6]);
        for (int t0 = 0; t0 < p.T; t0 += 256) {
          const int ntile = min(2, (p.T - t0 + 127) / 128);
          c.pf.mark(p, 3);
          build_frames(c, sig(a), h, t0, ntile);
          c.pf.mark(p, 6);
          fence_proxy_async_smem();
          if (tid == 0) bulk_wait_read();  // the previous octave's output stage may be rewritten after this sync
          c.pf.mark(p, 13);
          csync();
          c.pf.mark(p, 9);
          if (tid == 0) mbar_arrive(&bars[7]);
          if (halve && t0 == 0) {
            c.wait_mma();
            c.pf.mark(p, 7);
            const __half* sp = sig(a);
            __half* sd = sig(a + 1);
            uint8_t* po = planes_of(a + 1);
            const uint32_t pl_out = (uint32_t)p.plane_rows[a + 1] * 16u;
            const int n_out = p.oct_len[a + 1];
            fir_epilogue(
                c, 0, 0, n_out, 0, p.h0,
                [&](int i0, float* cv) {
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) {
                    const uint4 w = ld8(sp, ML + 2 * i0 + 8 * kk);
                    const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
                    for (int u = 0; u < 4; ++u) cv[4 * kk + u] = __low2float(h2[u]);
                  }
                },
                [&](int i) { return __half2float(sp[sw(ML + 2 * i)]); }, out16_of(sd, po, pl_out, p.plane_rows[a + 1]),
                out1_of(sd, po, pl_out, p.plane_rows[a + 1]));
            csync();
            edge_pass(sd, po, pl_out, p.plane_rows[a + 1], n_out);
            fence_proxy_async_smem();
            c.pf.mark(p, 8);
          }
          mbar_wait(conv_bar, conv_phase);
          conv_phase ^= 1;
          tc_fence_after();
          c.pf.mark(p, 10);
          // the octave's rows (row0 + skip ..) are contiguous in the (B, n_bins, T) output;
          // when that block is 16-byte aligned it is staged in the (consumed) im2col
          // tile and written with one bulk copy
          const int skip = max(0, a * p.bpo - p.first_bin);
          const int64_t o0 = (b * p.n_bins + p.first_bin - a * p.bpo + skip) * (int64_t)p.T;
          const uint32_t bytes = (uint32_t)((p.n_filt - skip) * p.T * 4);
          const bool staged = p.out_kind != NNAB_OUT_COMPLEX && p.T <= 256 && (o0 & 3) == 0 && (bytes & 15) == 0;
          float* stage = staged ? reinterpret_cast<float*>(base + p.off_stage) : nullptr;
          conv_epilogue(c, a, b, t0, ntile, out_scale, stage);
          c.pf.mark(p, 11);
          tc_fence_before();
          if (staged) fence_proxy_async_smem();
          csync();
          c.pf.mark(p, 14);
          if (staged && tid == 0) bulk_store(p.out + o0, stage, bytes);  // drained before the next octave's epilogue
        }
      }
      c.pf.mark(p, 15);
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // output bulk stores performed
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(*tslot);
  if (p.prof && tid == 0)
    for (int i = 0; i < 16; ++i) atomicAdd(p.prof + i, prof_acc[i]);
}

// ------------------------------------------------------------------ batched octave levels
// After the front (the fused kernel in front-only mode: stages 1-2 per clip, octave 0
// to the level buffer), every octave level runs as two launches over ALL clips:
// CONV (the 12-bin complex conv of octave alpha, frames as M) and HALVE (octave alpha ->
// alpha + 1, blocks of 128 outputs as M, the same Toeplitz band as the fused kernel).
// Tiles span clips, so no CTA walks one clip's serial chain: small shared memory, several
// CTAs per SM, and the latency of one tile's build / MMA / epilogue hides behind the others'.
// Level buffers: [B][stride] FP16 in the clip's power-of-two scale, sample i at ML + i,
// np.pad "reflect" images of ML samples on both sides (written by the producer).
struct LvParams {
  int64_t B;
  const __half* src;
  int32_t src_stride, n_src;  // halves per clip row; signal length
  __half* dst;
  int32_t dst_stride, n_dst;
  int32_t nb;                 // HALVE: blocks of 128 outputs per clip
  float h0;
  float g[128];
  const int32_t* exps;        // per-clip scale exponent (values are s * 2^-e)
  int32_t h, T, pad, pad_al, skip, row0, n_filt, n_bins, out_kind, width;
  const float* k_re;
  const float* k_im;
  float* out;
  const uint4* toep_img;  // the diagonal Toeplitz chunks (TOEP_CHUNKS x 16 B), built once per call
  const uint4* filt_img;  // the conv bank operand (KC / 8 x 512 B), built once per call
  unsigned long long* prof;  // debug: per-phase globaltimer ns sums (block 0's thread 0), or null
  // CONV over all octaves in one launch: level a's buffer, row stride, length
  const __half* lv[kMaxOct];
  int32_t lv_stride[kMaxOct], lv_n[kMaxOct];
  int32_t n_lv, kernel_hop, first_bin, bpo;
};

NNAB_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kLvThreads = 256;
constexpr int kHalveA = 32 * 128 * 16;   // A tile: 32 K-chunks x 128 rows x 16 B = 64 KB
constexpr int kConvA = (KC / 8) * 128 * 16;  // im2col: 12 chunks x 128 frames x 16 B = 24 KB

// 8 FP16 samples at (possibly unaligned) position i of a level row, 0 outside [0, lim).
// The slow path is out of line: inlined, the compiler predicated it into every call.
__device__ __noinline__ uint4 lv_load8_slow(const __half* row, int i, int lim);
NNAB_DEV uint4 lv_load8(const __half* row, int i, int lim) {
  if (i >= 0 && i + 8 <= lim && (i & 7) == 0) return __ldg(reinterpret_cast<const uint4*>(row + i));
  return lv_load8_slow(row, i, lim);
}
// 8 samples at an EVEN misalignment (the deep octaves' frames at hop 2 / 4): two aligned
// loads and a word select (explicit selects: no local-memory array)
NNAB_DEV uint4 lv_load8_even(const __half* row, int i, int lim) {
  const int a = i & ~7;
  if ((i & 1) || a < 0 || a + 16 > lim) return lv_load8(row, i, lim);
  const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(row + a)), w1 = __ldg(reinterpret_cast<const uint4*>(row + a + 8));
  const int sh = (i & 7) >> 1;
  uint4 o;
  o.x = sh == 0 ? w0.x : sh == 1 ? w0.y : sh == 2 ? w0.z : w0.w;
  o.y = sh == 0 ? w0.y : sh == 1 ? w0.z : sh == 2 ? w0.w : w1.x;
  o.z = sh == 0 ? w0.z : sh == 1 ? w0.w : sh == 2 ? w1.x : w1.y;
  o.w = sh == 0 ? w0.w : sh == 1 ? w1.x : sh == 2 ? w1.y : w1.z;
  return o;
}
__device__ __noinline__ uint4 lv_load8_slow(const __half* row, int i, int lim) {
  __align__(16) __half v[8];
  const unsigned short* r16 = reinterpret_cast<const unsigned short*>(row);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int k = i + e;
    unsigned short u = (k >= 0 && k < lim) ? __ldg(r16 + k) : (unsigned short)0;
    v[e] = __ushort_as_half(u);
  }
  return *reinterpret_cast<uint4*>(v);
}

// The shared-memory operand images every level CTA copies in: Toeplitz diagonal chunks
// (chunk j = g[j - 127 + e]) and the conv bank (row 2j = Re bin j, 2j+1 = Im, scaled 2^6,
// column m = tap m - (pad_al - pad)).  One CTA, once per call.
__global__ void cqt2010_prep_kernel(const __grid_constant__ LvParams p, uint4* toep_img, uint4* filt_img) {
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int j = t0; j < TOEP_CHUNKS; j += nt) {
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int gi = j - 127 + e;
      v[e] = h16((gi >= 0 && gi < 128) ? p.g[gi] : 0.f);
    }
    toep_img[j] = *reinterpret_cast<uint4*>(v);
  }
  const int shift = p.pad_al - p.pad;
  __half* f = reinterpret_cast<__half*>(filt_img);
  for (int e = t0; e < NCONV * KC; e += nt) {
    const int n = e / KC, m = e % KC, j = n >> 1, tap = m - shift;
    float v = 0.f;
    if (j < p.n_filt && tap >= 0 && tap < p.width)
      v = ldexpf(((n & 1) ? p.k_im : p.k_re)[(int64_t)j * p.width + tap], kFiltLog2);
    f[(m >> 3) * 256 + n * 8 + (m & 7)] = h16(v);
  }
}

// HALVE: octave alpha -> alpha + 1 for all clips.  Rows: clip b owns nb + 1 rows of 128
// odd-phase samples (row r = src_ext[2 (128 r + u) - 127], u < 128); block (b, blk) = 128
// outputs whose Toeplitz window is rows blk, blk + 1, so an M = 128 tile of rows reads 129
// plane rows (the existing FIR's "planes": 16-byte chunk q of every row in plane q) and a
// clip's extra row only feeds a discarded D row.  The build reads each row's 256 source
// samples with coalesced 16-byte loads (16 threads per row) and keeps both phases: odd ->
// planes, even -> the centre-tap rows (16-byte units XOR-swizzled by row).
constexpr int kHPl = 131 * 16;  // plane stride: 129 rows + pad, an odd number of 16-byte units

__global__ void __launch_bounds__(kLvThreads) cqt2010_halve_kernel(const __grid_constant__ LvParams p) {
  const unsigned long long t_start = gtime();
  unsigned long long t_mark = t_start;
  auto mark = [&](int i) {
    if (p.prof && threadIdx.x == 0) {
      const unsigned long long n = gtime();
      atomicAdd(p.prof + i, n - t_mark);
      t_mark = n;
    }
  };
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* planes = base;                     // 16 planes x kHPl
  uint8_t* even = base + 16 * kHPl;           // 129 rows x 256 B (centre taps)
  uint8_t* toep = even + 129 * 256;
  uint64_t* bar = reinterpret_cast<uint64_t*>(toep + ((TOEP_CHUNKS * 16 + 127) & ~127));
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(tslot);
  for (int j = tid; j < TOEP_CHUNKS; j += kLvThreads) reinterpret_cast<uint4*>(toep)[j] = __ldg(p.toep_img + j);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  mark(0);
  const int R = p.nb + 1;  // rows per clip
  const int64_t n_rows = p.B * R;
  const int64_t n_tiles = (n_rows + 127) / 128;
  const int src_lim = p.n_src + 2 * ML;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    // build 129 rows x 16 chunks; thread -> (row, chunk q), 16 threads per row; all of a
    // thread's loads (9 jobs x 32 B) are in flight before the first store
    constexpr int kJobs = (129 * 16 + kLvThreads - 1) / kLvThreads;
    uint4 wa[kJobs], wb[kJobs];
#pragma unroll
    for (int jj = 0; jj < kJobs; ++jj) {
      const int job = tid + jj * kLvThreads;
      const int rr = job >> 4, qq = job & 15;
      const int64_t g = tile * 128 + rr;
      wa[jj] = wb[jj] = make_uint4(0, 0, 0, 0);
      if (job < 129 * 16 && g < n_rows) {
        const int64_t b = g / R;
        const int r = (int)(g - b * R);
        const __half* row = p.src + b * p.src_stride;
        const int i0 = ML - 128 + 256 * r + 16 * qq;  // samples i0 .. i0 + 15: odd-phase u = 8 qq + e at i0 + 1 + 2e
        wa[jj] = lv_load8(row, i0, src_lim);
        wb[jj] = lv_load8(row, i0 + 8, src_lim);
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJobs; ++jj) {
      const int job = tid + jj * kLvThreads;
      if (job >= 129 * 16) break;
      const int rr = job >> 4, qq = job & 15;
      const uint4 w0 = wa[jj], w1 = wb[jj];
      uint4 o, e;
      o.x = __byte_perm(w0.x, w0.y, 0x7632);
      o.y = __byte_perm(w0.z, w0.w, 0x7632);
      o.z = __byte_perm(w1.x, w1.y, 0x7632);
      o.w = __byte_perm(w1.z, w1.w, 0x7632);
      e.x = __byte_perm(w0.x, w0.y, 0x5410);
      e.y = __byte_perm(w0.z, w0.w, 0x5410);
      e.z = __byte_perm(w1.x, w1.y, 0x5410);
      e.w = __byte_perm(w1.z, w1.w, 0x5410);
      *reinterpret_cast<uint4*>(planes + qq * kHPl + rr * 16) = o;
      // even samples of row rr: src[ML - 128 + 256 rr' + 2 (8 qq + e)] = src[2 i] for i = 128 r - 64 + 8 qq + e
      *reinterpret_cast<uint4*>(even + rr * 256 + ((qq ^ (rr & 15)) << 4)) = e;
    }
    fence_proxy_async_smem();
    __syncthreads();
    mark(1);
    if (tid == 0) {
      tc_fence_after();
      constexpr uint32_t idesc = idesc_f16(128, 128);
      const uint32_t a0 = smem_u32(planes), t0 = smem_u32(toep);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        mma_f16(tmem, nsw_desc(a0 + (uint32_t)(2 * (k & 7)) * kHPl + (uint32_t)(k >> 3) * 16u, kHPl, 128),
                nsw_desc(t0 + 256u * k, 128, 128), idesc, k > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    mark(2);
    // epilogue: TMEM lane = tile row m = block (b, blk), column r' = 127 - r; warp w reads lane
    // quarter w & 3 and column half w >> 2 in 4 chunks of 16 columns = 16 consecutive outputs
    const int q = warp & 3, half = warp >> 2;
    const int m = q * 32 + lane;
    const int64_t g = tile * 128 + m;
    const int64_t b = g < n_rows ? g / R : 0;
    const int blk = g < n_rows ? (int)(g - b * R) : 0;
    const bool live = g < n_rows && blk < p.nb;  // the clip's extra row is not a block
    __half* drow = p.dst + b * p.dst_stride;
    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + half * 64;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int rbase = 112 - 64 * half - 16 * k;
      const int i0 = blk * 128 + rbase;
      float v[16];
      tmem_ld16(ta + 16 * k, v);
      tmem_ld_wait();
      if (!live || i0 >= p.n_dst) continue;
      // centre taps src[2 i], i = i0 .. i0 + 15: the even samples 128 blk - 64 + ... of rows m
      // (i < 128 blk + 64) and m + 1 (the rest)
      float y[16];
      {
        const int u = rbase + 64;  // even index within rows m, m + 1 (128 per row)
        const int rr = m + (u >> 7), uu = u & 127;
        const uint8_t* er = even + rr * 256;
        const uint4 a = *reinterpret_cast<const uint4*>(er + ((((uu >> 3)) ^ (rr & 15)) << 4));
        const uint4 c = *reinterpret_cast<const uint4*>(er + ((((uu >> 3) + 1) ^ (rr & 15)) << 4));
        float t[8];
        unpack8(a, t);
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = t[e];
        unpack8(c, t);
#pragma unroll
        for (int e = 0; e < 8; ++e) y[8 + e] = t[e];
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) y[e] = fmaf(p.h0, y[e], v[15 - e]);
      if (i0 + 16 <= p.n_dst) {
        __align__(16) __half2 al[8];
        pack_all(y, al);
        *reinterpret_cast<uint4*>(drow + ML + i0) = reinterpret_cast<const uint4*>(al)[0];
        *reinterpret_cast<uint4*>(drow + ML + i0 + 8) = reinterpret_cast<const uint4*>(al)[1];
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (i0 + e < p.n_dst) drow[ML + i0 + e] = h16(y[e]);
      }
      // np.pad "reflect" images of the new level (signal.py:151): left -i, right 2(n-1) - i
      if (i0 <= ML || i0 + 16 >= p.n_dst - 1 - ML) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int i = i0 + e;
          if (i >= p.n_dst) break;
          if (i >= 1 && i <= ML) drow[ML - i] = h16(y[e]);
          if (i >= p.n_dst - 1 - ML && i <= p.n_dst - 2) drow[ML + 2 * (p.n_dst - 1) - i] = h16(y[e]);
        }
      }
      if (i0 < p.n_dst && i0 + 16 >= p.n_dst) {  // the row's tail past the right image: finite zeros
        for (int j = p.n_dst + 2 * ML; j < p.dst_stride; ++j) drow[j] = __float2half(0.f);
      }
    }
    tc_fence_before();
    __syncthreads();
    mark(3);
  }
  if (warp == 0) tmem_dealloc<128>(tmem);
  mark(4);
  if (p.prof && threadIdx.x == 0) atomicAdd(p.prof + 5, 1ull);
}

// CONV: the complex conv of every octave and clip in one persistent launch, frames as M,
// the top-octave bank as N = 32 (re/im rows of <= 16 bins), K = 96 taps.  Level a's
// buffer is laid out as rows of rs = max(h, 8) samples (clip stride U rows, so the rows
// of all clips form one uniform array): frame (b, u) starts at row g = b U + u and its
// K window is (row g + k / rs, col k mod rs).  The im2col tile is therefore a handful of
// bulk copies, no thread touches it:
//   rs >= 64: taps 0-63 one TMA box (64 cols x 128 rows, 128-byte swizzle), taps 64-95
//             one box (32 cols, 64-byte swizzle) at row + 64 / rs
//   rs = 32:  three boxes of 32 cols (64-byte swizzle) at rows g, g + 1, g + 2
//   rs = 16:  six boxes of 16 cols (32-byte swizzle)
//   rs = 8:   the rows are the contiguous signal: one 1-D bulk copy of 139 rows, read by
//             a no-swizzle descriptor with LBO 16 B / SBO 128 B (frame g + 1 = 16 B on)
// Hops below 8 (the deepest octaves) read C = 8 / h copies of the level shifted by v h
// samples, frame t = C u + v.  Rows past a clip's T frames are computed and discarded.
// Warp roles (persistent, one CTA per SM, ring of kConvStages tiles / accumulators):
//   warp 0    producer (one elected thread)
//   warp 1    MMA issue (one elected thread) + TMEM allocation
//   warps 4-19 epilogue, four warpgroups taking tiles in turn: thread = frame (TMEM lane
//             quarter), magnitude / power / complex of the bins, stores coalesced along T
constexpr int kConvStages = 8;
constexpr int kConvEpi = 4;  // epilogue warpgroups
constexpr int kConvThreads = (4 + 4 * kConvEpi) * 32;
constexpr int kConvMaps = 16;
constexpr uint32_t kRows8 = 128 + KC / 8 - 1;  // rs = 8: rows a 128-frame tile reads

struct ConvParams {
  CUtensorMap map[kConvMaps];       // per (octave, copy): [wide box, narrow box] (rs >= 64) or one
  int64_t B;
  int32_t n_oct, T, n_bins, first_bin, bpo, n_filt, out_kind;
  int32_t copies[kMaxOct], U[kMaxOct], map0[kMaxOct], rs[kMaxOct];
  int64_t tiles_per_copy[kMaxOct], tile0[kMaxOct + 1];  // tile0[i]: first tile of the i-th octave in walk order
  int32_t ord[kMaxOct];  // walk order: deepest octave first (the chain wrote those last: still in L2)
  const __half* rows[kMaxOct];      // rs = 8: level base (+ the frame offset), copy stride below
  int64_t copy_stride[kMaxOct];
  const int32_t* exps;
  const uint4* filt_img;
  float* out;
  unsigned long long* prof;  // debug: [0] producer wait, [1] MMA full wait, [2] MMA tfree wait, [3] epilogue wait, [4] elapsed
};

NNAB_DEV uint64_t swz_desc(uint32_t addr, uint32_t row_bytes) {  // K-major, 32/64/128-byte swizzle
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(((8 * row_bytes) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(row_bytes == 128 ? 2 : row_bytes == 64 ? 4 : 6) << 61;
  return d;
}

__global__ void __launch_bounds__(kConvThreads, 1) cqt2010_conv_kernel(const __grid_constant__ ConvParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = base;                                   // kConvStages x kConvA
  uint8_t* filt = base + kConvStages * kConvA;
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(filt + KC / 8 * 512);  // [S] operands landed (TMA tx)
  uint64_t* bar_mma = bar_full + kConvStages;                             // [S] MMAs done (commit)
  uint64_t* bar_tfree = bar_mma + kConvStages;                            // [S] accumulator read (4 warps)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar_tfree + kConvStages);
  int32_t* exps_s = reinterpret_cast<int32_t*>(tslot + 4);  // the clips' scale exponents (B ints)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kConvStages; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_mma[s], 1);
      mbar_init(&bar_tfree[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<32 * kConvStages>(tslot);
  for (int j = tid; j < KC / 8 * 32; j += kConvThreads) reinterpret_cast<uint4*>(filt)[j] = __ldg(p.filt_img + j);
  for (int j = tid; j < p.B; j += kConvThreads) exps_s[j] = __ldg(p.exps + j);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  unsigned long long pw = 0, pw2 = 0;
  const long long tb = clock64();
  auto tw = [&](uint64_t* bar, uint32_t par, unsigned long long& acc) {
    const long long t0 = clock64();
    mbar_wait_sleep(bar, par);
    acc += (unsigned long long)(clock64() - t0);
  };
  const int64_t n_tiles = p.tile0[p.n_oct];
  const int64_t n_local = n_tiles > blockIdx.x ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  // tile -> (octave, copy, first row); i only grows, so the octave is tracked incrementally
  struct Loc {
    int a = 0, ia = 0;
    NNAB_DEV void at(const ConvParams& p, int64_t i, int& v, int& row0) {
      const int k = (int)(blockIdx.x + i * gridDim.x);
      while (ia + 1 < p.n_oct && k >= (int)p.tile0[ia + 1]) ++ia;
      a = p.ord[ia];
      const int kl = k - (int)p.tile0[ia], tpc = (int)p.tiles_per_copy[a];
      v = kl / tpc;
      row0 = (kl - v * tpc) * 128;
    }
  };
  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      Loc loc;
      for (int m = 0; m < kConvMaps; ++m)
        if (m < p.map0[p.n_oct - 1] + 2) tma_prefetch(&p.map[m]);
      for (int64_t i = 0; i < n_local; ++i) {
        const int s = (int)(i % kConvStages);
        const uint32_t r = (uint32_t)(i / kConvStages);
        int v, row0;
        loc.at(p, i, v, row0);
        const int a = loc.a, rs = p.rs[a];
        if (r > 0) tw(&bar_mma[s], (r - 1) & 1, pw);  // the stage's previous MMAs have read it
        uint8_t* As = A + s * kConvA;
        const int y = (int)row0;
        if (rs == 8) {
          mbar_expect_tx(&bar_full[s], kRows8 * 16);
          bulk_load(As, p.rows[a] + v * p.copy_stride[a] + (int64_t)8 * row0, kRows8 * 16, &bar_full[s]);
        } else {
          mbar_expect_tx(&bar_full[s], (uint32_t)kConvA);
          const CUtensorMap* map = &p.map[p.map0[a] + v * (rs >= 64 ? 2 : 1)];
          if (rs >= 64) {
            tma_load_2d(As, map, &bar_full[s], 0, y);
            tma_load_2d(As + 16384, map + 1, &bar_full[s], 64 % rs, y + 64 / rs);
          } else if (rs == 32) {
            for (int j = 0; j < 3; ++j) tma_load_2d(As + 8192 * j, map, &bar_full[s], 0, y + j);
          } else {
            for (int j = 0; j < 6; ++j) tma_load_2d(As + 4096 * j, map, &bar_full[s], 0, y + j);
          }
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ---------------------------------------------------------------- MMA issue: two issuing
    // threads on alternate tiles (the per-thread tcgen05 issue latency, not the tensor pipe,
    // bounds these narrow MMAs)
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_f16(128, NCONV);
      const uint32_t b0 = smem_u32(filt);
      Loc loc;
      for (int64_t i = warp - 1; i < n_local; i += 2) {
        const int s = (int)(i % kConvStages);
        const uint32_t r = (uint32_t)(i / kConvStages);
        int v, row0;
        loc.at(p, i, v, row0);
        const int rs = p.rs[loc.a];
        {
          const long long t0 = clock64();
          mbar_wait_sleep(&bar_full[s], r & 1);
          const unsigned long long dt = (unsigned long long)(clock64() - t0);
          pw += dt;
          if (p.prof) atomicAdd(p.prof + 5 + loc.a, dt);
        }
        if (r > 0) tw(&bar_tfree[s], (r - 1) & 1, pw2);
        tc_fence_after();
        const uint32_t a0 = smem_u32(A + s * kConvA);
#pragma unroll
        for (int k = 0; k < KC / 16; ++k) {
          uint64_t ad;
          if (rs >= 64) ad = k < 4 ? swz_desc(a0 + 32u * k, 128) : swz_desc(a0 + 16384u + 32u * (k - 4), 64);
          else if (rs == 32) ad = swz_desc(a0 + 8192u * (k >> 1) + 32u * (k & 1), 64);
          else if (rs == 16) ad = swz_desc(a0 + 4096u * k, 32);
          else ad = nsw_desc(a0 + 32u * k, 16, 128);
          mma_f16(tmem + 32 * s, ad, nsw_desc(b0 + (uint32_t)k * 1024u, 512, 128), idesc, k > 0);
        }
        mma_commit(&bar_mma[s]);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue: kConvEpi warpgroups
    // taking tiles in turn; the clip's scale exponent is fetched before the accumulator wait
    const int q = warp & 3, eg = (warp - 4) >> 2;
    const int j_hi = min(p.n_filt, NCONV / 2);
    Loc loc;
    for (int64_t i = eg; i < n_local; i += kConvEpi) {
      const int s = (int)(i % kConvStages);
      const uint32_t r = (uint32_t)(i / kConvStages);
      int v, row0;
      loc.at(p, i, v, row0);
      const int a = loc.a;
      const int g = row0 + q * 32 + lane;
      const int b = g / p.U[a];
      const int t = p.copies[a] * (g - b * p.U[a]) + v;
      const bool live = b < p.B && t < p.T;
      const int ex = live ? exps_s[b] : 0;
      tw(&bar_mma[s], r & 1, pw);
      tc_fence_after();
      float acc[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 32 * s, acc);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_tfree[s]);
      if (!live) continue;
#ifdef NNAB_DBG_CONV_NOSTORE
      if (acc[0] != 12345.f) continue;
#endif
      const int lskip = max(0, a * p.bpo - p.first_bin), lrow0 = p.first_bin - a * p.bpo;
      const int eo = ex - kFiltLog2;  // 2^eo without ldexpf's call in the common range
      const float os = (eo > -126 && eo < 128) ? __int_as_float((eo + 127) << 23) : ldexpf(1.f, eo);
      const int64_t obase = ((int64_t)b * p.n_bins + lrow0) * p.T + t;
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
  if (p.prof) {
    if (warp == 0 && pw) atomicAdd(p.prof + 0, pw);
    if ((warp == 1 || warp == 2) && (pw | pw2)) { atomicAdd(p.prof + 1, pw); atomicAdd(p.prof + 2, pw2); }
    if (tid == 128) atomicAdd(p.prof + 3, pw);
    if (tid == 128) atomicAdd(p.prof + 4, (unsigned long long)(clock64() - tb));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<32 * kConvStages>(tmem);
}

// The shifted copies of the levels whose hop is below 8 (the conv reads 16-byte rows):
// copy v of level a, row b = copy 0's row b shifted left by v h samples (zero past it).
// Thread = 8 output samples: two aligned loads and a word select (v h is even).
struct CopyParams {
  const __half* src[kMaxOct];
  int32_t stride[kMaxOct], h[kMaxOct], copies[kMaxOct];
  int64_t copy_stride[kMaxOct];
  int32_t B, n_oct;
};
__global__ void cqt2010_copies_kernel(const __grid_constant__ CopyParams p) {
  for (int a = 0; a < p.n_oct; ++a) {
    if (p.copies[a] < 2) continue;
    const int n8 = p.stride[a] >> 3;               // 8-sample units per row
    const int per = (p.copies[a] - 1) * n8;        // units per clip
    const int n = p.B * per;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
      const int b = e / per;
      const int rem = e - b * per;
      const int v = 1 + rem / n8;
      const int k8 = rem - (v - 1) * n8;
      const int sh = v * p.h[a];                   // even
      const __half* row = p.src[a] + (int64_t)b * p.stride[a];
      const int i0 = 8 * k8 + sh, al = i0 & ~7;
      const uint4 z = make_uint4(0, 0, 0, 0);
      const uint4 w0 = al < p.stride[a] ? __ldg(reinterpret_cast<const uint4*>(row + al)) : z;
      const uint4 w1 = al + 8 < p.stride[a] ? __ldg(reinterpret_cast<const uint4*>(row + al + 8)) : z;
      const uint32_t wd[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
      const int q = (i0 & 7) >> 1;
      uint4 o;
      o.x = q == 0 ? wd[0] : q == 1 ? wd[1] : q == 2 ? wd[2] : wd[3];
      o.y = q == 0 ? wd[1] : q == 1 ? wd[2] : q == 2 ? wd[3] : wd[4];
      o.z = q == 0 ? wd[2] : q == 1 ? wd[3] : q == 2 ? wd[4] : wd[5];
      o.w = q == 0 ? wd[3] : q == 1 ? wd[4] : q == 2 ? wd[5] : wd[6];
      *reinterpret_cast<uint4*>(const_cast<__half*>(p.src[a]) + v * p.copy_stride[a] + (int64_t)b * p.stride[a] +
                                8 * k8) = o;
    }
  }
}

__device__ unsigned long long g_cqt_prof[16];
bool g_cqt_prof_on = false;
unsigned long long* cqt2010_prof_ptr() {
  if (!g_cqt_prof_on) return nullptr;
  void* ptr = nullptr;
  cudaGetSymbolAddress(&ptr, g_cqt_prof);
  return reinterpret_cast<unsigned long long*>(ptr);
}

struct Plan {
  TcParams p;
  size_t smem;
};

int32_t rnd(int64_t v, int a) { return (int32_t)((v + a - 1) / a * a); }

// Geometry and shared-memory plan of the fused kernel; NNAB_ENOTSUP outside its envelope.
int make_plan(int64_t L, int n_taps, const float* taps, int n_filt, int width, int early_stages, int n_oct,
              int kernel_hop, int T, int pad_mode, Plan* pl) {
  if (early_stages != 2 || n_taps != 255 || pad_mode != NNAB_PAD_REFLECT) return NNAB_ENOTSUP;
  if (n_filt > 16 || n_oct < 1 || n_oct > kMaxOct) return NNAB_ENOTSUP;
  const int pad = width / 2, pad_al = (pad + 7) & ~7;
  if (width + (pad_al - pad) > KC || pad_al > ML) return NNAB_ENOTSUP;
  float hmax = 0.f;  // half-band check: even offsets (odd tap indices) are negligible
  for (int i = 0; i < n_taps; ++i) hmax = std::max(hmax, std::fabs(taps[i]));
  for (int i = 1; i < n_taps; i += 2)
    if (i != 127 && std::fabs(taps[i]) > 1e-12f * hmax) return NNAB_ENOTSUP;
  TcParams& p = pl->p;
  p = TcParams{};
  const int64_t L1 = (L + 1) / 2, L0 = (L1 + 1) / 2;
  if (L0 > 256 * 128 || L1 > (1 << 30)) return NNAB_ENOTSUP;  // stage 2 in two M = 128 tiles
  p.L = L;
  p.L1 = (int32_t)L1;
  p.L0 = (int32_t)L0;
  p.n1_tiles = (int32_t)((L1 + kTile1 * 128 - 1) / (kTile1 * 128));
  p.n_oct = n_oct;
  p.kernel_hop = kernel_hop;
  p.pad = pad;
  p.pad_al = pad_al;
  p.T = T;
  p.rows2 = rnd(std::max(std::min(T, 256) - 128, 8), 8);
  int64_t n = L0;
  for (int a = 0; a < n_oct; ++a) {
    if (a > 0) n = (n + 1) / 2;
    if (n < ML + 2) return NNAB_ENOTSUP;  // reflect margins need n > ML + 1
    p.oct_len[a] = (int32_t)n;
    p.oct_blocks[a] = (int32_t)((n + 127) / 128);
    if (a > 0 && p.oct_blocks[a] > 128) return NNAB_ENOTSUP;  // one M = 128 tile per octave halving
  }
  // odd-phase planes of octave a feeding halving a+1: blocks + 1 rows, and the
  // right reflect image up to m = (n + 253) / 2
  for (int a = 0; a + 1 < n_oct; ++a)
    p.plane_rows[a] = rnd(std::max(p.oct_blocks[a + 1] + 1, (p.oct_len[a] + 253) / 2 / 128 + 1), 8);
  // shared memory (bytes): fixed | R1 = stage-1 operands, later octave 0 | R2 = stage-2 operands, later
  // octaves >= 1.  An M = 128 tile reads 129 plane rows whatever the signal length, so short plane
  // sets need up to 2064 B of readable memory behind them (slack).
  constexpr int kSlack = 2304;
  int off = 0;
  p.off_toep = off;  off += TOEP_CHUNKS * 16;
  off = rnd(off, 1024);
  p.off_filt = off;  off += KC / 8 * 512;
  p.off_ring = off;  off += 2 * kRing;
  const int r1 = off;
  p.pl_x = (kTile1 + 8) * 16 + 16;  // +16 B: consecutive planes start in different banks
  p.off_x = off;     off += p.pl_x * 16;
  p.off_xe = off;    off += kTile1 * 128 * 2;
  int r1_end = off;
  int o = r1;  // octave 0 (written by stage 2) reuses R1
  p.s_off[0] = o;    o += rnd((int64_t)p.oct_len[0] + 2 * ML, 128) * 2;
  if (n_oct > 1) { p.o_off[0] = o; o += p.plane_rows[0] * 256; }
  o += kSlack;
  r1_end = std::max(r1_end, o);
  const int r2 = rnd(r1_end, 128);
  p.y_rows = rnd(std::max((int)((L1 + 254) / 2 / 128) + 1, p.oct_blocks[0] + 1), 8);
  p.pl_y = p.y_rows * 16;
  p.off_y = r2;
  p.off_ye = r2 + p.pl_y * 16 + kSlack;
  p.off_stage = 0;  // set below (after the octave region)
  int r2_end = p.off_ye + rnd(L0 + 16, 128) * 2;  // whole 128-sample rows (swizzle stays inside)
  o = r2;  // octaves >= 1 and the im2col tile reuse R2; octave a only lives with a +- 1 (ping-pong)
  p.off_col = o;     o += (128 + p.rows2) * KC * 2;
  int s_sz[2] = {0, 0}, o_sz[2] = {0, 0};
  for (int a = 1; a < n_oct; ++a) {
    s_sz[a & 1] = std::max(s_sz[a & 1], rnd((int64_t)p.oct_len[a] + 2 * ML, 128) * 2);
    if (a + 1 < n_oct) o_sz[a & 1] = std::max(o_sz[a & 1], p.plane_rows[a] * 256);
  }
  const int s_base[2] = {o + s_sz[1], o};
  o += s_sz[0] + s_sz[1];
  const int o_base[2] = {o + o_sz[1], o};
  o += o_sz[0] + o_sz[1];
  for (int a = 1; a < n_oct; ++a) {
    p.s_off[a] = s_base[a & 1];
    if (a + 1 < n_oct) p.o_off[a] = o_base[a & 1];
  }
  o += kSlack;
  r2_end = std::max(r2_end, o);
  off = rnd(r2_end, 128);
  p.off_stage = off; off += rnd((int64_t)n_filt * std::min(T, 256) * 4, 128);  // one octave's output rows
  p.off_bars = off;  off += 128;
  pl->smem = 1024 + (size_t)off;
  if (pl->smem > 227 * 1024) return NNAB_ENOTSUP;
  return NNAB_OK;
}

// Level buffer geometry of the batched path: one [B][stride] FP16 row set per octave,
// stride = U rows of rs = max(h, 8) samples (the conv's TMA rows), plus copies - 1
// shifted copies when h < 8.
struct LvPlan {
  int32_t n[kMaxOct], stride[kMaxOct], rs[kMaxOct], U[kMaxOct], copies[kMaxOct], h[kMaxOct];
  size_t off[kMaxOct], exp_off, toep_off, filt_off, flag_off, list_off, total;
};
int lv_plan(const TcParams& tp, int64_t B, LvPlan* lp) {
  size_t off = ((size_t)B * 4 + 255) & ~size_t(255);  // exps first, then the operand images
  lp->exp_off = 0;
  lp->toep_off = off;
  off += (TOEP_CHUNKS * 16 + 255) & ~255;
  lp->filt_off = off;
  off += (KC / 8 * 512 + 255) & ~255;
  lp->flag_off = off;  // the front's fast-scale flags, then the flagged-clip list and its count
  off += ((size_t)B * 4 + 255) & ~size_t(255);
  lp->list_off = off;
  off += ((size_t)B * 4 + 4 + 255) & ~size_t(255);
  for (int a = 0; a < tp.n_oct; ++a) {
    const int h = tp.kernel_hop >> a;
    if (h < 1) return NNAB_ENOTSUP;
    lp->h[a] = h;
    lp->n[a] = tp.oct_len[a];
    lp->rs[a] = std::max(h, 8);
    lp->copies[a] = std::max(1, 8 / h);
    // rows of 256 samples (the chain's TMA view; a multiple of every conv row length rs):
    // the signal with its margins, and for a halving input the rows its last block's
    // window reads (block n reads rows n, n + 1)
    int rows = (tp.oct_len[a] + 2 * ML + 255) / 256;
    if (a + 1 < tp.n_oct) rows = std::max(rows, (tp.oct_len[a + 1] + 127) / 128 + 1);
    lp->stride[a] = 256 * rows;
    lp->U[a] = lp->stride[a] / lp->rs[a];
    if ((int64_t)lp->copies[a] * lp->U[a] < tp.T) return NNAB_ENOTSUP;
    lp->off[a] = off;
    // + slack read as 0-weight operands (HALVE windows, the conv rows' base offset)
    off += ((size_t)lp->copies[a] * B * lp->stride[a] * 2 + 4096 + 255) & ~size_t(255);
  }
  lp->total = off;
  return NNAB_OK;
}

}  // namespace

// Workspace the batched CQT2010v2 path needs (0 outside the fused kernel's envelope).
size_t cqt2010_levels_bytes(int64_t B, int64_t L, const float* taps, int n_taps, int n_filt, int width,
                            int early_stages, int n_oct, int kernel_hop, int T, int pad_mode) {
  Plan pl;
  if (make_plan(L, n_taps, taps, n_filt, width, early_stages, n_oct, kernel_hop, T, pad_mode, &pl)) return 0;
  LvPlan lp;
  if (lv_plan(pl.p, B, &lp)) return 0;
  return lp.total;
}

// The shifted level copies (hops below 8) and the batched conv of every octave.
int launch_cqt2010_conv(const LvPlan& lp, char* ws, int64_t B, int T, int n_oct, int n_bins, int first_bin, int bpo,
                        int n_filt, int pad_al, int out_kind, const int32_t* exps, const uint4* filt_img, float* out,
                        cudaStream_t st, bool copies_written = false) {
  CopyParams cp{};
  bool any_copy = false;
  if (B * (int64_t)lp.stride[0] * 8 > INT32_MAX) return NNAB_ENOTSUP;
  cp.B = (int32_t)B;
  cp.n_oct = n_oct;
  for (int a = 0; a < n_oct; ++a) {
    cp.src[a] = reinterpret_cast<const __half*>(ws + lp.off[a]);
    cp.stride[a] = lp.stride[a];
    cp.h[a] = lp.h[a];
    cp.copies[a] = lp.copies[a];
    cp.copy_stride[a] = B * (int64_t)lp.stride[a];
    any_copy |= lp.copies[a] > 1;
  }
  if (any_copy && !copies_written) {
    cqt2010_copies_kernel<<<2 * num_sms(), 256, 0, st>>>(cp);
    NNAB_LAUNCHED();
  }
  ConvParams* cv = new ConvParams{};  // > 2 KB of tensor maps: off the host stack
  ConvParams& c = *cv;
  c.B = B;
  c.n_oct = n_oct;
  c.T = T;
  c.n_bins = n_bins;
  c.first_bin = first_bin;
  c.bpo = bpo;
  c.n_filt = n_filt;
  c.out_kind = out_kind;
  c.exps = exps;
  c.filt_img = filt_img;
  c.prof = cqt2010_prof_ptr();
  c.out = out;
  int nm = 0;
  c.tile0[0] = 0;
  for (int i = 0; i < n_oct; ++i) c.ord[i] = n_oct - 1 - i;
  for (int a = 0; a < n_oct; ++a) {
    const int rs = lp.rs[a];
    if (rs != 8 && rs != 16 && rs != 32 && rs < 64) return NNAB_ENOTSUP;
    c.copies[a] = lp.copies[a];
    c.U[a] = lp.U[a];
    c.rs[a] = rs;
    c.map0[a] = nm;
    c.tiles_per_copy[a] = (B * (int64_t)lp.U[a] + 127) / 128;
    if (c.tiles_per_copy[a] * 128 >= INT32_MAX) { delete cv; return NNAB_ENOTSUP; }

    c.copy_stride[a] = B * (int64_t)lp.stride[a];
    const __half* lbase = reinterpret_cast<const __half*>(ws + lp.off[a]) + (ML - pad_al);
    c.rows[a] = lbase;
    if (rs == 8) continue;  // 1-D bulk copies
    for (int v = 0; v < lp.copies[a]; ++v) {
      const __half* base = lbase + (int64_t)v * c.copy_stride[a];
      const int nbox = rs >= 64 ? 2 : 1;
      if (nm + nbox > kConvMaps) { delete cv; return NNAB_ENOTSUP; }
      const uint32_t w0 = rs >= 64 ? 64 : (uint32_t)rs;
      int rc = make_tmap_2d(&c.map[nm++], base, (uint64_t)rs, (uint64_t)(B * lp.U[a]), (uint64_t)rs * 2, w0, 128,
                            (int)w0 * 2, 2);
      if (!rc && nbox == 2)
        rc = make_tmap_2d(&c.map[nm++], base, (uint64_t)rs, (uint64_t)(B * lp.U[a]), (uint64_t)rs * 2, 32, 128, 64, 2);
      if (rc) { delete cv; return rc; }
    }
  }
  for (int i = 0; i < n_oct; ++i) c.tile0[i + 1] = c.tile0[i] + c.tiles_per_copy[c.ord[i]] * lp.copies[c.ord[i]];
  const size_t smem_conv = 1024 + kConvStages * kConvA + KC / 8 * 512 + 3 * kConvStages * 8 + 16 + 4 * (size_t)B;
  if (smem_conv > 227 * 1024) { delete cv; return NNAB_ENOTSUP; }
  cudaError_t e = cudaFuncSetAttribute(cqt2010_conv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_conv);
  if (e == cudaSuccess) {
    cqt2010_conv_kernel<<<(int)std::min<int64_t>(c.tile0[n_oct], (int64_t)num_sms()), kConvThreads, smem_conv, st>>>(c);
    e = cudaGetLastError();
  }
  delete cv;
  NNAB_CUDA_TRY(e);
  note_launch();
  return NNAB_OK;
}

// The batched path: the fused kernel in front-only mode (stages 1-2 per clip, octave 0
// to the level buffer), then per octave one CONV launch and one HALVE launch over all clips.
int launch_cqt2010_levels(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, const float* k_re,
                          const float* k_im, int n_filt, int width, int early_stages, int n_oct, int kernel_hop,
                          int first_bin, int bpo, int n_bins, int pad_mode, int out_kind, int T, float* out,
                          void* workspace, size_t workspace_bytes, cudaStream_t st, int mode) {
  Plan pl;
  int rc = make_plan(L, n_taps, taps, n_filt, width, early_stages, n_oct, kernel_hop, T, pad_mode, &pl);
  if (rc) return rc;
  if (n_filt > 16) return NNAB_ENOTSUP;
  LvPlan lp;
  if (lv_plan(pl.p, B, &lp)) return NNAB_ENOTSUP;
  if (!workspace || workspace_bytes < lp.total) return NNAB_ENOTSUP;
  char* ws = reinterpret_cast<char*>(workspace);
  int32_t* exps = reinterpret_cast<int32_t*>(ws + lp.exp_off);
  TcParams& p = pl.p;
  p.x = x;
  p.B = B;
  p.first_bin = first_bin;
  p.bpo = bpo;
  p.n_bins = n_bins;
  p.n_filt = n_filt;
  p.width = width;
  p.out_kind = out_kind;
  p.h0 = taps[127];
  for (int j = 0; j < 128; ++j) p.g[j] = taps[2 * j];
  p.k_re = k_re;
  p.k_im = k_im;
  p.out = out;
  p.prof = nullptr;
  p.lv0 = reinterpret_cast<__half*>(ws + lp.off[0]);
  p.lv_exp = exps;
  p.lv0_stride = lp.stride[0];
  p.lv_mode = mode;
  for (int a = 0; a < n_oct; ++a) {
    p.lv[a] = reinterpret_cast<__half*>(ws + lp.off[a]);
    p.lv_stride[a] = lp.stride[a];
  }
  // mode 3: the warp-specialised front (cqt2010_front.cu) for stages 1-2, then as mode 1;
  // it also writes the bank images cqt2010_prep_kernel would
  CqtPrepArgs pa;
  pa.toep_img = reinterpret_cast<uint4*>(ws + lp.toep_off);
  pa.filt_img = reinterpret_cast<uint4*>(ws + lp.filt_off);
  pa.k_re = k_re;
  pa.k_im = k_im;
  pa.n_filt = n_filt;
  pa.width = width;
  pa.shift = p.pad_al - p.pad;
  pa.nconv = NCONV;
  pa.kc = KC;
  pa.filt_log2 = kFiltLog2;
  rc = mode == 3 ? launch_cqt2010_front(x, B, L, taps, n_taps, p.lv0, p.lv0_stride, exps,
                                        reinterpret_cast<int32_t*>(ws + lp.flag_off),
                                        reinterpret_cast<int32_t*>(ws + lp.list_off),
                                        reinterpret_cast<int32_t*>(ws + lp.list_off) + B, st, &pa)
                  : NNAB_ENOTSUP;
  const bool prepped = mode == 3 && rc == NNAB_OK;
  if (rc == NNAB_ENOTSUP) {
    if (mode == 3) p.lv_mode = 1;
    NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt2010_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    cqt2010_tc_kernel<<<(int)std::min<int64_t>(B, (int64_t)num_sms()), kThreads, pl.smem, st>>>(p);
    NNAB_LAUNCHED();
  } else if (rc) {
    return rc;
  }
  const bool mode3 = mode == 3;
  if (mode == 3) mode = 1;  // the halving launches below run only if the mode-3 back end is out of reach
  bool chained = false;
  LvParams q{};
  q.B = B;
  q.h0 = taps[127];
  for (int j = 0; j < 128; ++j) q.g[j] = taps[2 * j];
  q.exps = exps;
  q.T = T;
  q.pad = p.pad;
  q.pad_al = p.pad_al;
  q.n_filt = n_filt;
  q.n_bins = n_bins;
  q.out_kind = out_kind;
  q.width = width;
  q.k_re = k_re;
  q.k_im = k_im;
  q.out = out;
  q.prof = cqt2010_prof_ptr();
  q.toep_img = reinterpret_cast<const uint4*>(ws + lp.toep_off);
  q.filt_img = reinterpret_cast<const uint4*>(ws + lp.filt_off);
  if (!prepped) {
    cqt2010_prep_kernel<<<8, 256, 0, st>>>(q, reinterpret_cast<uint4*>(ws + lp.toep_off),
                                            reinterpret_cast<uint4*>(ws + lp.filt_off));
    NNAB_LAUNCHED();
  }
  if (mode3) {
    // mode 3: the octave chain and every octave's conv in one launch (cqt2010_back.cu); else the
    // chain launch (cqt2010_chain.cu) + the batched conv; else the HALVE launches + batched conv
    CqtBackArgs bg{};
    bg.n_oct = n_oct;
    bg.B = B;
    bg.taps = taps;
    bg.n_taps = n_taps;
    for (int a = 0; a < n_oct; ++a) {
      bg.lv[a] = reinterpret_cast<__half*>(ws + lp.off[a]);
      bg.n[a] = lp.n[a];
      bg.stride[a] = lp.stride[a];
      bg.h[a] = lp.h[a];
      bg.copies[a] = lp.copies[a];
      bg.U[a] = lp.U[a];
      bg.rs[a] = lp.rs[a];
    }
    bg.pad_al = p.pad_al;
    bg.T = T;
    bg.n_bins = n_bins;
    bg.first_bin = first_bin;
    bg.bpo = bpo;
    bg.n_filt = n_filt;
    bg.out_kind = out_kind;
    bg.exps = exps;
    bg.filt_img = reinterpret_cast<const uint4*>(ws + lp.filt_off);
    bg.out = out;
    static const bool no_back = [] { const char* e = getenv("NNAB_CQT2010_NOBACK"); return e && e[0] == '1'; }();
    rc = no_back ? NNAB_ENOTSUP : launch_cqt2010_back(bg, st);
    if (rc != NNAB_ENOTSUP) return rc;
    __half* lvp[kMaxOct];
    int32_t hh[kMaxOct], cc[kMaxOct];
    for (int a = 0; a < n_oct; ++a) {
      lvp[a] = reinterpret_cast<__half*>(ws + lp.off[a]);
      hh[a] = lp.h[a];
      cc[a] = lp.copies[a];
    }
    rc = launch_cqt2010_chain(B, n_oct, lvp, lp.stride, lp.n, hh, cc, taps, n_taps, st);
    if (rc && rc != NNAB_ENOTSUP) return rc;
    chained = rc == NNAB_OK;
    if (chained) mode = 3;
  }
  const size_t smem_halve = 1024 + 16 * kHPl + 129 * 256 + ((TOEP_CHUNKS * 16 + 127) & ~127) + 64;
  NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt2010_halve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_halve));
  q.n_lv = n_oct;
  q.kernel_hop = kernel_hop;
  q.first_bin = first_bin;
  q.bpo = bpo;
  for (int a = 0; a < n_oct; ++a) {
    q.lv[a] = reinterpret_cast<const __half*>(ws + lp.off[a]);
    q.lv_stride[a] = lp.stride[a];
    q.lv_n[a] = lp.n[a];
  }
  // the halvings octave by octave (mode 1; mode 2 ran them in the fused kernel), then every
  // octave's conv in one launch
  for (int a = 0; a < n_oct && mode == 1; ++a) {
    q.src = reinterpret_cast<const __half*>(ws + lp.off[a]);
    q.src_stride = lp.stride[a];
    q.n_src = lp.n[a];
    if (a + 1 < n_oct) {
      q.dst = reinterpret_cast<__half*>(ws + lp.off[a + 1]);
      q.dst_stride = lp.stride[a + 1];
      q.n_dst = lp.n[a + 1];
      q.nb = (q.n_dst + 127) / 128;
      const int64_t tiles = (B * (int64_t)(q.nb + 1) + 127) / 128;
      cqt2010_halve_kernel<<<(int)std::min<int64_t>(tiles, 2 * (int64_t)num_sms()), kLvThreads, smem_halve, st>>>(q);
      NNAB_LAUNCHED();
    }
  }
  return launch_cqt2010_conv(lp, ws, B, T, n_oct, n_bins, first_bin, bpo, n_filt, p.pad_al, out_kind, exps,
                             reinterpret_cast<const uint4*>(ws + lp.filt_off), out, st, chained);
  return NNAB_OK;
}

// Debug: enable per-phase cycle counters of the fused kernel (on != 0), or read
// and clear them into out[16] (on == 0).  Phases: 12 wait for the scale,
// 0 stage-1 build, 1 stage-1 MMA, 2 stage-1 epilogue, 4 stage-2 MMA,
// 5 stage-2 epilogue, 9 conv im2col, 10 conv (+ halving) MMA, 11 conv epilogue,
// 8 halving epilogue, 15 loop tail.
extern "C" int nnab_debug_cqt2010_profile(int on, unsigned long long* out) {
  if (on) {
    g_cqt_prof_on = true;
    unsigned long long z[16] = {};
    NNAB_CUDA_TRY(cudaMemcpyToSymbol(g_cqt_prof, z, sizeof(z)));
    return NNAB_OK;
  }
  g_cqt_prof_on = false;
  if (out) NNAB_CUDA_TRY(cudaMemcpyFromSymbol(out, g_cqt_prof, 16 * sizeof(unsigned long long)));
  return NNAB_OK;
}

// Fused tensor-core CQT2010v2; NNAB_ENOTSUP when the configuration is outside
// what the fused kernel holds on chip (the caller then runs the staged
// CUDA-core kernels).
int launch_cqt2010_tc(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, const float* k_re,
                      const float* k_im, int n_filt, int width, int early_stages, int n_oct, int kernel_hop,
                      int first_bin, int bpo, int n_bins, int pad_mode, int out_kind, int T, float* out,
                      cudaStream_t st) {
  Plan pl;
  int rc = make_plan(L, n_taps, taps, n_filt, width, early_stages, n_oct, kernel_hop, T, pad_mode, &pl);
  if (rc) return rc;
  TcParams& p = pl.p;
  const int grid = (int)std::min<int64_t>(B, (int64_t)num_sms());
  p.x = x;
  p.B = B;
  p.first_bin = first_bin;
  p.bpo = bpo;
  p.n_bins = n_bins;
  p.n_filt = n_filt;
  p.width = width;
  p.out_kind = out_kind;
  p.h0 = taps[127];
  for (int j = 0; j < 128; ++j) p.g[j] = taps[2 * j];
  p.k_re = k_re;
  p.k_im = k_im;
  p.out = out;
  p.prof = cqt2010_prof_ptr();
  NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt2010_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  cqt2010_tc_kernel<<<grid, kThreads, pl.smem, st>>>(p);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

}  // namespace nnab

// Debug (host only): the fused kernel's plan for a configuration -> shared-memory
// bytes (> 0), or minus the status code when the configuration is outside it.
extern "C" long long nnab_debug_cqt2010_plan(long long L, const float* taps, int n_taps, int n_filt, int width,
                                             int early_stages, int n_oct, int kernel_hop, int T, int pad_mode) {
  nnab::Plan pl;
  const int rc = nnab::make_plan(L, n_taps, taps, n_filt, width, early_stages, n_oct, kernel_hop, T, pad_mode, &pl);
  return rc ? -(long long)rc : (long long)pl.smem;
}
