// CQT2010v2 on the tensor cores: the whole octave recursion of one clip per
// CTA, two CTAs per SM so one clip's CUDA-core phases overlap the other's MMAs
// (transforms.py:290-313, signal.py:232-247).
//
// Operands are FP16 with an exact per-clip power-of-two scale (2^-e, e from the
// clip's peak), so they carry the same 11-bit significand as TF32 at twice the
// tcgen05 rate (kind::f16, K = 16); accumulation is FP32 and the scale is undone
// exactly in the conv epilogue.
//
// Half-band FIR as a banded Toeplitz MMA.  downsample2 keeps
//   y[i] = sum_d h[d] x_ext[2i + d],  d = -127..127 (reflect-extended x)
// and the cutoff-0.5 windowed sinc is half-band: every even d != 0 is <= 6.6e-17,
// so  y[i] = h0 * x[2i] + sum_{j<128} g_j * xo[i + j],  g_j = h[2j - 127],
// xo[m] = x_ext[2m - 127] (the odd phase).  A block of 128 outputs is
// Y[r] = sum_s T[r][s] W[s], T[r][s] = g_{s-r} (128 x 256 Toeplitz band), W = 256
// consecutive odd-phase samples; windows of consecutive blocks overlap by 128.
//   A = T with its rows reversed: A'[r'][s] = g[s + r' - 127] depends on s + r'
//       only, so the band lives in a 6 KB "diagonal" array (chunk j = 8 taps
//       g[j-127 ..]) that a no-swizzle K-major descriptor with LBO = SBO = 128 B
//       walks (toep_desc),
//   B = "planes": the odd phase stored once as rows of 128 samples, plane q
//       holding the 16-byte chunk q of every row (rows 16 B apart); block n's
//       window is rows n, n+1, i.e. a 16-byte start offset (LBO = plane stride).
// The MMA is issued transposed, D[block][r'] = sum_s W_block[s] T'[r'][s]
// (M = 128 blocks, N = 128 reversed offsets), so each TMEM lane holds 128
// consecutive outputs of one block and the epilogue stores 16-byte vectors.
// The producing epilogue writes every signal straight into the next stage's
// layouts (odd phase -> planes in shared memory, contiguous copy with reflect
// margins -> an L2-resident per-CTA scratch), so no separate deinterleave pass
// exists except for the clip itself (stage 1, built from global memory).
// Per-octave centred complex conv (<= 16 bins x <= 96 taps, hop h >> alpha):
// im2col MMA, A = 128 frames x 96 taps (built from the L2 copy), B = 32 rows
// (re/im of each bin) x 96 taps, D = 128 x 32 in TMEM; thread = frame in the
// epilogue so the (B, n_bins, T) output is written coalesced along T.
#include <algorithm>
#include <cmath>

#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kThreads = 256;
constexpr int kTile1 = 128;       // stage-1 blocks (N) per MMA tile
constexpr int ML = 128;           // reflect margins of the contiguous octave copies (fp16 elements)
constexpr int KC = 96;            // conv taps (K), padded
constexpr int NCONV = 32;         // conv N: re/im rows of <= 16 bins
constexpr int kFiltLog2 = 6;      // conv bank scaled by 2^6 before the FP16 rounding
constexpr int kMaxOct = 12;
constexpr int TOEP_CHUNKS = 8 * 31 + 128;  // 376 diagonal chunks of 8 taps
constexpr uint32_t kConvCol = 128;          // TMEM columns of the conv accumulators

struct TcParams {
  const float* x;
  int64_t B, L;
  int32_t L1, L0, n1_tiles;
  int32_t n_oct, kernel_hop, first_bin, bpo, n_bins, n_filt, width, T, out_kind;
  int32_t pad, pad_al;
  int32_t oct_len[kMaxOct];         // signal length of octave alpha
  int32_t oct_blocks[kMaxOct];      // 128-output blocks of the halving that produces octave alpha
  int32_t plane_rows[kMaxOct];      // rows of the odd-phase planes that feed halving alpha+1
  int64_t s_off[kMaxOct];           // scratch offset (fp16 elements) of octave alpha's contiguous copy
  int64_t ye_off, cta_stride;       // stage-1 even phase; per-CTA scratch size
  __half* scratch;
  float h0;                         // centre tap
  float g[128];                     // odd taps g_j = h[2j - 127]
  const float* k_re;                // top-octave bank (n_filt, width), device
  const float* k_im;
  float* out;
  // shared-memory carve-up (bytes from the 1 KB-aligned base)
  int32_t off_toep, off_filt, off_ra, off_rb, off_bars;
  int32_t pl_x, pl_y, y_rows;       // plane strides (bytes) of the stage-1 / stage-2 inputs; stage-2 plane rows
  unsigned long long* prof;         // optional per-phase cycle counters (nnab_debug_cqt2010_profile)
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

NNAB_DEV int64_t refl(int64_t j, int64_t n) {
  if (j < 0) j = -j;
  if (j >= n) j = 2 * (n - 1) - j;
  return j;
}

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

struct Ctx {
  const TcParams& p;
  uint8_t* base;
  uint32_t tmem;
  uint64_t* bar;      // MMA completion
  uint32_t phase;
  Prof pf;
  NNAB_DEV void wait_mma() {
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
  }
};

// Issue the Toeplitz FIR of 128 consecutive blocks (plane rows row0 ..) into TMEM
// column d_col; thread 0 only (the caller commits).  D[block][r'] = sum_s W_block[s] * T'[r'][s]:
// A = the odd-phase windows (M = 128 blocks, K-major planes), B = the reversed
// Toeplitz (N = 128 output offsets, the diagonal array), K = 256 in 16 steps.
// Rows past a signal's end only feed discarded blocks, so they may hold
// anything; the descriptors stay inside the CTA's shared memory.
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
// columns, i.e. 16 consecutive outputs i0 .. i0+15 (i0 = 128 n + rbase) per
// thread.  cen16(i0, c) loads their centre-tap samples, out16(i0, y) stores them
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
// outputs y[0..15] of i0 .. i0+15 (i0 % 16 == 0): odd ones (-> planes at
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

// Edge pass of a signal of length n held as a contiguous copy s (with ML margins)
// and, optionally, odd-phase planes: write the reflect images (np.pad "reflect",
// signal.py:245) from the already-stored samples.  One image per thread.
NNAB_DEV void edge_pass(__half* s, uint8_t* planes, uint32_t pl, int rows, int n) {
  for (int e = threadIdx.x; e < 2 * ML; e += kThreads) {
    const int i = e < ML ? e + 1 : n - 1 - ML + (e - ML);  // left: 1..ML, right: n-1-ML .. n-2
    const int dst = e < ML ? -i : 2 * (n - 1) - i;         // ext position of the image
    const __half v = s[ML + i];
    s[ML + dst] = v;
    if (planes && (dst & 1)) {
      const int m = (dst + 127) >> 1;
      if (m >= 0 && (m >> 7) < rows) *reinterpret_cast<__half*>(planes + plane_off(m, pl)) = v;
    }
  }
}

// Stage-1 planes for blocks [n0, n0 + rows - 1) (rows <= 129): odd phase of the
// clip, scaled, FP16.  Thread -> plane row r = tid & 127 (row 128 by the first 16
// threads afterwards) and plane chunks qq = tid >> 7 + 2u; four 64-byte chunk
// loads in flight per round.
NNAB_DEV void x_chunk(const float* xb, int64_t L, bool vec, int64_t j0, float* f) {
  if (vec && j0 >= 1 && j0 + 15 <= L) {
    const float4* src = reinterpret_cast<const float4*>(xb + j0 - 1);
    const float4 a = __ldg(src), b = __ldg(src + 1), cq = __ldg(src + 2), d = __ldg(src + 3);
    f[0] = a.y; f[1] = a.w; f[2] = b.y; f[3] = b.w; f[4] = cq.y; f[5] = cq.w; f[6] = d.y; f[7] = d.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int64_t j = j0 + 2 * k;
      if (j < 0) j = -j;
      if (j >= L) j = 2 * (L - 1) - j;
      f[k] = (j >= 0 && j < L) ? __ldg(xb + j) : 0.f;  // beyond one reflection: never a kept output
    }
  }
}
NNAB_DEV void put_x_chunk(uint8_t* planes, uint32_t pl, int r, int qq, const float* f, float scale) {
  __align__(16) __half2 hv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) hv[k] = __floats2half2_rn(f[2 * k] * scale, f[2 * k + 1] * scale);
  *reinterpret_cast<uint4*>(planes + (uint32_t)qq * pl + (uint32_t)r * 16u) = *reinterpret_cast<uint4*>(hv);
}
NNAB_DEV void build_x_planes(Ctx& c, const float* xb, float scale, int n0, int rows, uint8_t* planes, uint32_t pl,
                             bool vec) {
  const int64_t L = c.p.L;
  const int r = threadIdx.x & 127, q0 = threadIdx.x >> 7;  // q0 in {0, 1}
  if (r < rows) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float f[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int qq = q0 + 2 * (4 * h + u);
        x_chunk(xb, L, vec, 2 * ((int64_t)(n0 + r) * 128 + qq * 8) - 127, f[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) put_x_chunk(planes, pl, r, q0 + 2 * (4 * h + u), f[u], scale);
    }
  }
  if (rows > 128 && threadIdx.x < 16) {
    float f[8];
    x_chunk(xb, L, vec, 2 * ((int64_t)(n0 + 128) * 128 + threadIdx.x * 8) - 127, f);
    put_x_chunk(planes, pl, 128, threadIdx.x, f, scale);
  }
}

// Centred complex conv of octave alpha from its contiguous copy.
NNAB_DEV void octave_conv(Ctx& c, const __half* sig, int alpha, int64_t b, float out_scale) {
  const TcParams& p = c.p;
  const int h = p.kernel_hop >> alpha;
  const int skip = max(0, alpha * p.bpo - p.first_bin);
  const int row0 = p.first_bin - alpha * p.bpo;
  uint8_t* ca = c.base + p.off_ra;
  for (int t0 = 0; t0 < p.T; t0 += 256) {
    const int ntile = min(2, (p.T - t0 + 127) / 128);
    // im2col: tile u, chunk cc (8 taps) of frame t at u*24576 + cc*2048 + t*16; all of a
    // thread's 16-byte loads are issued before any store
    constexpr int kPer = 2 * 128 * (KC / 8) / kThreads;  // 12
    uint4 v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = threadIdx.x + k * kThreads;
      const int t = e & 127, rest = e >> 7, cc = rest % (KC / 8), u = rest / (KC / 8);
      const int tt = t0 + u * 128 + t;
      v[k] = make_uint4(0, 0, 0, 0);
      if (tt < p.T) {
        const __half* s = sig + ML + tt * h - p.pad_al + cc * 8;
        if ((h & 7) == 0) {
          v[k] = *reinterpret_cast<const uint4*>(s);
        } else if ((h & 3) == 0) {
          const uint2 a = reinterpret_cast<const uint2*>(s)[0], bb = reinterpret_cast<const uint2*>(s)[1];
          v[k] = make_uint4(a.x, a.y, bb.x, bb.y);
        } else {
          const uint32_t* w = reinterpret_cast<const uint32_t*>(s);
          v[k] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = threadIdx.x + k * kThreads;
      const int t = e & 127, rest = e >> 7, cc = rest % (KC / 8), u = rest / (KC / 8);
      if (u < ntile) *reinterpret_cast<uint4*>(ca + u * 24576 + cc * 2048 + t * 16) = v[k];
    }
    fence_proxy_async_smem();
    __syncthreads();
    c.pf.mark(p, 9);
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t idesc = idesc_f16(128, NCONV);
      const uint32_t a0 = smem_u32(ca), b0 = smem_u32(c.base + p.off_filt);
      for (int u = 0; u < ntile; ++u) {
#pragma unroll
        for (int k = 0; k < KC / 16; ++k)
          mma_f16(c.tmem + kConvCol + 32 * u, nsw_desc(a0 + u * 24576 + 2 * k * 2048, 2048, 128),
                  nsw_desc(b0 + 2 * k * 512, 512, 128), idesc, k > 0);
      }
      mma_commit(c.bar);
    }
    c.wait_mma();
    c.pf.mark(p, 10);
    {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      const int q = warp & 3, u = warp >> 2;
      const int t = t0 + u * 128 + q * 32 + lane;
      if (u < ntile) {
        float v[32];
        tmem_ld32(c.tmem + ((uint32_t)(q * 32) << 16) + kConvCol + 32 * u, v);
        tmem_ld_wait();
        if (t < p.T) {
#pragma unroll
          for (int j = 0; j < NCONV / 2; ++j) {
            if (j < skip || j >= p.n_filt) continue;
            const float re = v[2 * j] * out_scale, im = v[2 * j + 1] * out_scale;
            const int64_t o = (b * p.n_bins + row0 + j) * (int64_t)p.T + t;
            if (p.out_kind == NNAB_OUT_COMPLEX) {
              reinterpret_cast<float2*>(p.out)[o] = make_float2(re, im);
            } else if (p.out_kind == NNAB_OUT_POWER) {
              p.out[o] = fmaf(re, re, im * im);
            } else {
              p.out[o] = sqrtf(fmaf(re, re, im * im));
            }
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    c.pf.mark(p, 11);
  }
}

__global__ void __launch_bounds__(kThreads, 2) cqt2010_tc_kernel(const __grid_constant__ TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + p.off_bars);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);  // bars[0] MMA, bars[1..3] scan ring
  __shared__ float red[kThreads / 32];
  __shared__ unsigned long long prof_acc[16];
  const int tid = threadIdx.x, warp = tid >> 5;

  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  // zero the operand regions once (rows past a signal's end only feed discarded
  // outputs, but must hold finite values)
  for (int i = tid; i < (p.off_bars - p.off_ra) / 16; i += kThreads)
    reinterpret_cast<uint4*>(base + p.off_ra)[i] = make_uint4(0, 0, 0, 0);
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
  // conv bank B: row n = 2j (+1 for Im), chunk cc at cc*512 + n*16; column m holds tap m - shift
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

  Ctx c{p, base, *tslot, &bars[0], 0, {}};
  c.pf.acc = prof_acc;
  if (tid < 16) prof_acc[tid] = 0;
  if (p.prof && tid == 0) c.pf.t = clock64();
  const bool vec = (p.L % 4) == 0;
  uint8_t* xp = base + p.off_ra;   // stage-1 planes (aliases the conv im2col tiles)
  uint8_t* yp = base + p.off_rb;   // stage-2 planes (later: octave planes)
  const uint32_t xp_s = smem_u32(xp), yp_s = smem_u32(yp);
  uint32_t scan_seq = 0;  // bulk-copy ring uses so far (slot = seq % 3, parity = seq / 3)

  for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
    const float* xb = p.x + b * p.L;
    __half* scr = p.scratch + blockIdx.x * p.cta_stride;
    // ------------------------------------------------ per-clip scale 2^-e (peak -> [0.5, 1))
    // the clip streams through a 3 x 16 KB ring of bulk copies (TMA engine: the
    // whole clip is in flight at HBM bandwidth and lands in L2 for stage 1)
    float mx = 0.f;
    if (vec) {
      constexpr uint32_t kChunk = 16384;
      const uint32_t bytes = (uint32_t)(p.L * 4);
      const int nch = (int)((bytes + kChunk - 1) / kChunk);
      const char* src = reinterpret_cast<const char*>(xb);
      auto issue = [&](int k) {
        const uint32_t sz = std::min(kChunk, bytes - (uint32_t)k * kChunk);
        const int slot = (int)((scan_seq + k) % 3);
        mbar_expect_tx(&bars[1 + slot], sz);
        bulk_load(xp + slot * kChunk, src + (size_t)k * kChunk, sz, &bars[1 + slot]);
      };
      if (tid == 0)
        for (int k = 0; k < 3 && k < nch; ++k) issue(k);
      for (int k = 0; k < nch; ++k) {
        const uint32_t seq = scan_seq + k;
        mbar_wait(&bars[1 + seq % 3], (seq / 3) & 1);
        const uint32_t sz = std::min(kChunk, bytes - (uint32_t)k * kChunk);
        const float4* b4 = reinterpret_cast<const float4*>(xp + (seq % 3) * kChunk);
        for (int i = tid; i < (int)(sz / 16); i += kThreads) {
          const float4 a = b4[i];
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
        }
        __syncthreads();  // slot consumed by every thread before it is refilled
        if (tid == 0 && k + 3 < nch) issue(k + 3);
      }
      scan_seq += (uint32_t)nch;
    } else {
      for (int64_t i = tid; i < p.L; i += kThreads) mx = fmaxf(mx, fabsf(__ldg(xb + i)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[warp] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; ++w) mx = fmaxf(mx, red[w]);
    int ex = 0;
    if (mx > 0.f && mx < INFINITY) frexpf(mx, &ex);
    const float scale = ldexpf(1.f, -ex), out_scale = ldexpf(1.f, ex - kFiltLog2);
    c.pf.mark(p, 12);

    // ------------------------------------------------ stage 1: x -> y1 (odd -> planes, even -> scratch)
    __half* ye = scr + p.ye_off;
    const int L1 = p.L1, nt = p.n1_tiles;
    auto tile_blocks = [&](int t) { return min(kTile1, (L1 - t * kTile1 * 128 + 127) / 128); };
    build_x_planes(c, xb, scale, 0, tile_blocks(0) + 1, xp, p.pl_x, vec);
    fence_proxy_async_smem();
    __syncthreads();
    c.pf.mark(p, 0);
    if (tid == 0) {
      issue_fir(c, xp_s, p.pl_x, 0, 0);
      mma_commit(c.bar);
    }
    for (int t = 0; t < nt; ++t) {
      c.wait_mma();
      c.pf.mark(p, 1);
      if (t + 1 < nt) {  // next tile's planes (its MMAs overlap this tile's epilogue)
        build_x_planes(c, xb, scale, (t + 1) * kTile1, tile_blocks(t + 1) + 1, xp, p.pl_x, vec);
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
          issue_fir(c, xp_s, p.pl_x, 0, ((t + 1) & 1) * 128);
          mma_commit(c.bar);
        }
        c.pf.mark(p, 0);
      }
      fir_epilogue(
          c, t * kTile1, 0, L1, (t & 1) * 128, p.h0 * scale,
          [&](int i0, float* cv) {
            if (vec) {
              const float4* s4 = reinterpret_cast<const float4*>(xb + 2 * (int64_t)i0);
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float4 w = __ldg(s4 + k);
                cv[2 * k] = w.x;
                cv[2 * k + 1] = w.z;
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) cv[e] = __ldg(xb + 2 * (int64_t)(i0 + e));
            }
          },
          [&](int i) { return __ldg(xb + 2 * (int64_t)i); },
          [&](int i0, const float* y) {
            __align__(16) __half2 od[4], ev[4];
            pack_odd(y, od);
            pack_even(y, ev);
            store_planes8(yp, p.pl_y, p.y_rows, i0 / 2 + 64, od);                            // stage-2 planes
            *reinterpret_cast<uint4*>(ye + i0 / 2) = *reinterpret_cast<const uint4*>(ev);  // stage-2 centre taps
          },
          [&](int i, float y) {
            if (i & 1) store_plane1(yp, p.pl_y, p.y_rows, (i + 127) >> 1, h16(y));
            else ye[i >> 1] = h16(y);
          });
      tc_fence_before();
      __syncthreads();
      c.pf.mark(p, 2);
    }
    // reflect images of y1's odd phase (left: -i, right: 2(L1-1) - i, i odd)
    for (int e = tid; e < 128; e += kThreads) {
      const int i = e < 64 ? 2 * e + 1 : ((L1 - 128) | 1) + 2 * (e - 64);
      const int dst = e < 64 ? -i : 2 * (L1 - 1) - i;
      if (i <= L1 - 2) {
        const __half v = *reinterpret_cast<const __half*>(yp + plane_off((i + 127) >> 1, p.pl_y));
        store_plane1(yp, p.pl_y, p.y_rows, (dst + 127) >> 1, v);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();

    // FIR epilogue functors of a signal held as a contiguous copy (centre taps at
    // src[2i] or src[i]) writing a contiguous copy + the next halving's planes
    auto contig_out16 = [&](__half* dst, uint8_t* planes, uint32_t pl, int rows) {
      return [=](int i0, const float* y) {
        __align__(16) __half2 al[8];
        pack_all(y, al);
        uint4* d4 = reinterpret_cast<uint4*>(dst + ML + i0);
        d4[0] = reinterpret_cast<const uint4*>(al)[0];
        d4[1] = reinterpret_cast<const uint4*>(al)[1];
        if (planes) {
          __align__(16) __half2 od[4];
          pack_odd(y, od);
          store_planes8(planes, pl, rows, i0 / 2 + 64, od);
        }
      };
    };
    auto contig_out1 = [&](__half* dst, uint8_t* planes, uint32_t pl, int rows) {
      return [=](int i, float y) {
        const __half v = h16(y);
        dst[ML + i] = v;
        if (planes && (i & 1)) store_plane1(planes, pl, rows, (i + 127) >> 1, v);
      };
    };

    // ------------------------------------------------ stage 2: y1 -> octave 0
    __half* s0 = scr + p.s_off[0];
    const int n2 = p.oct_len[0];
    const int nb2 = p.oct_blocks[0];
    const int row_b = nb2 > 128 ? nb2 - 128 : 0;  // second tile covers the last 128 blocks
    if (tid == 0) {
      issue_fir(c, yp_s, p.pl_y, 0, 0);
      if (nb2 > 128) issue_fir(c, yp_s, p.pl_y, row_b, 128);
      mma_commit(c.bar);
    }
    c.wait_mma();
    c.pf.mark(p, 4);
    {
      uint8_t* o0 = p.n_oct > 1 ? yp : nullptr;  // octave planes overwrite the (consumed) y1 planes
      const uint32_t pl0 = (uint32_t)p.plane_rows[0] * 16u;
      auto cen16 = [&](int i0, float* cv) {
        const uint4* s4 = reinterpret_cast<const uint4*>(ye + i0);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint4 w = s4[k];
          const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 f = __half22float2(h2[u]);
            cv[8 * k + 2 * u] = f.x;
            cv[8 * k + 2 * u + 1] = f.y;
          }
        }
      };
      auto cen1 = [&](int i) { return __half2float(ye[i]); };
      // the first tile's MMA has completed, but its epilogue must not write the
      // planes the second tile still reads: both tiles are committed together, so
      // every MMA is done here
      fir_epilogue(c, 0, 0, n2, 0, p.h0, cen16, cen1, contig_out16(s0, o0, pl0, p.plane_rows[0]),
                   contig_out1(s0, o0, pl0, p.plane_rows[0]));
      if (nb2 > 128)
        fir_epilogue(c, row_b, 128, n2, 128, p.h0, cen16, cen1, contig_out16(s0, o0, pl0, p.plane_rows[0]),
                     contig_out1(s0, o0, pl0, p.plane_rows[0]));
      __syncthreads();
      edge_pass(s0, o0, pl0, p.plane_rows[0], n2);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    c.pf.mark(p, 5);

    // ------------------------------------------------ octaves: conv, halve, repeat
    uint8_t* o_in = yp;
    uint8_t* o_out = yp + p.plane_rows[0] * 16 * 16;
    for (int a = 0; a < p.n_oct; ++a) {
      const __half* sa = scr + p.s_off[a];
      if (a > 0) {
        const __half* sp = scr + p.s_off[a - 1];
        __half* sd = scr + p.s_off[a];
        const int n_out = p.oct_len[a];
        const uint32_t pl_in = (uint32_t)p.plane_rows[a - 1] * 16u;
        if (tid == 0) {
          issue_fir(c, smem_u32(o_in), pl_in, 0, 0);
          mma_commit(c.bar);
        }
        c.wait_mma();
        c.pf.mark(p, 7);
        uint8_t* po = a + 1 < p.n_oct ? o_out : nullptr;
        const uint32_t pl_out = (uint32_t)p.plane_rows[a] * 16u;
        fir_epilogue(
            c, 0, 0, n_out, 0, p.h0,
            [&](int i0, float* cv) {
              const uint4* s4 = reinterpret_cast<const uint4*>(sp + ML + 2 * i0);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint4 w = s4[k];
                const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
                for (int u = 0; u < 4; ++u) cv[4 * k + u] = __low2float(h2[u]);
              }
            },
            [&](int i) { return __half2float(sp[ML + 2 * i]); }, contig_out16(sd, po, pl_out, p.plane_rows[a]),
            contig_out1(sd, po, pl_out, p.plane_rows[a]));
        __syncthreads();
        edge_pass(sd, po, pl_out, p.plane_rows[a], n_out);
        fence_proxy_async_smem();
        tc_fence_before();
        uint8_t* tmp = o_in;
        o_in = o_out;
        o_out = tmp;
        __syncthreads();
        c.pf.mark(p, 8);
      }
      octave_conv(c, sa, a, b, out_scale);
    }
    c.pf.mark(p, 15);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<256>(*tslot);
  if (p.prof && tid == 0)
    for (int i = 0; i < 16; ++i) atomicAdd(p.prof + i, prof_acc[i]);
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
  int ctas_per_sm;
  size_t scratch_bytes_per_cta;
};

int64_t rnd8(int64_t v) { return (v + 7) & ~int64_t(7); }

// Geometry and shared-memory plan of the fused kernel; NNAB_ENOTSUP outside its envelope.
int make_plan(int64_t L, int n_taps, const float* taps, int n_filt, int width, int early_stages, int n_oct,
              int kernel_hop, int pad_mode, Plan* pl) {
  if (early_stages != 2 || n_taps != 255 || pad_mode != NNAB_PAD_REFLECT) return NNAB_ENOTSUP;
  if (n_filt > NCONV / 2 || n_oct < 1 || n_oct > kMaxOct) return NNAB_ENOTSUP;
  const int pad = width / 2, pad_al = (pad + 7) & ~7;
  if (width + (pad_al - pad) > KC || pad_al > ML) return NNAB_ENOTSUP;
  float hmax = 0.f;  // half-band check: even offsets (odd tap indices) are negligible
  for (int i = 0; i < n_taps; ++i) hmax = std::max(hmax, std::fabs(taps[i]));
  for (int i = 1; i < n_taps; i += 2)
    if (i != 127 && std::fabs(taps[i]) > 1e-12f * hmax) return NNAB_ENOTSUP;
  TcParams& p = pl->p;
  p = TcParams{};
  const int64_t L1 = (L + 1) / 2, L0 = (L1 + 1) / 2;
  if (L0 > 255 * 128 || L1 > 1 << 30) return NNAB_ENOTSUP;  // stage 2 in one MMA tile (N <= 256)
  p.L = L;
  p.L1 = (int32_t)L1;
  p.L0 = (int32_t)L0;
  p.n1_tiles = (int32_t)((L1 + kTile1 * 128 - 1) / (kTile1 * 128));
  p.n_oct = n_oct;
  p.kernel_hop = kernel_hop;
  p.pad = pad;
  p.pad_al = pad_al;
  int64_t n = L0;
  int64_t off = rnd8(L0);  // ye
  p.ye_off = 0;
  for (int a = 0; a < n_oct; ++a) {
    if (a > 0) n = (n + 1) / 2;
    if (n < ML + 2) return NNAB_ENOTSUP;  // reflect margins need n > ML + 1
    p.oct_len[a] = (int32_t)n;
    p.oct_blocks[a] = (int32_t)((n + 127) / 128);
    if (a > 0 && p.oct_blocks[a] > 128) return NNAB_ENOTSUP;  // one M = 128 tile per octave halving
    p.s_off[a] = off;
    off += rnd8(n + 2 * ML);
  }
  // odd-phase planes of octave a feeding halving a+1: blocks + 1 rows, and the
  // right reflect image up to m = (n + 253) / 2
  for (int a = 0; a + 1 < n_oct; ++a)
    p.plane_rows[a] = (std::max(p.oct_blocks[a + 1] + 1, (p.oct_len[a] + 253) / 2 / 128 + 1) + 7) & ~7;
  p.cta_stride = rnd8(off);
  // shared memory: toep | filt | RA = max(x planes, conv tiles) | RB = max(y planes, octave planes) + slack
  // (an M = 128 tile reads 129 plane rows whatever the signal length: up to 2064 B past a short plane set)
  p.pl_x = (kTile1 + 8) * 16;
  // odd phase of y1 incl. its right reflect image: m < (L1 + 254) / 2; stage 2 reads blocks + 1 rows
  p.y_rows = (std::max((int)((L1 + 254) / 2 / 128) + 1, p.oct_blocks[0] + 1) + 7) & ~7;
  p.pl_y = p.y_rows * 16;
  const size_t ra = std::max<size_t>((size_t)p.pl_x * 16, 2 * 24576);
  size_t oct_planes = 0;
  for (int a = 0; a + 1 < n_oct; ++a)
    oct_planes = std::max(oct_planes, (size_t)(p.plane_rows[0] + (a + 2 < n_oct ? p.plane_rows[a + 1] : 0)) * 256);
  const size_t rb = std::max((size_t)p.pl_y * 16, oct_planes) + 2304;
  p.off_toep = 0;
  p.off_filt = 6144;
  p.off_ra = 6144 + 6144;
  p.off_rb = p.off_ra + (int32_t)((ra + 1023) & ~size_t(1023));
  p.off_bars = p.off_rb + (int32_t)((rb + 127) & ~size_t(127));
  pl->smem = 1024 + (size_t)p.off_bars + 64;
  if (pl->smem > 227 * 1024) return NNAB_ENOTSUP;
  pl->ctas_per_sm = pl->smem <= 113 * 1024 ? 2 : 1;
  pl->scratch_bytes_per_cta = (size_t)p.cta_stride * 2;
  return NNAB_OK;
}

}  // namespace

// Debug: enable per-phase cycle counters of the fused kernel (on != 0), or read
// and clear them into out[16] (on == 0).  Phases: 12 scale scan, 0 stage-1 planes,
// 1 stage-1 MMA wait, 2 stage-1 epilogue, 4 stage-2 MMA, 5 stage-2 epilogue,
// 7 octave MMA, 8 octave epilogue / CUDA-core halving, 9 conv im2col,
// 10 conv MMA, 11 conv epilogue, 15 loop tail.
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

size_t cqt2010_tc_scratch_bytes(int64_t B, int64_t L, const float* taps, int n_taps, int n_filt, int width,
                                int early_stages, int n_oct, int kernel_hop, int pad_mode) {
  Plan pl;
  if (!taps || make_plan(L, n_taps, taps, n_filt, width, early_stages, n_oct, kernel_hop, pad_mode, &pl)) return 0;
  const int64_t grid = std::min<int64_t>(B, (int64_t)num_sms() * pl.ctas_per_sm);
  return (size_t)grid * pl.scratch_bytes_per_cta + 256;
}

// Fused tensor-core CQT2010v2; NNAB_ENOTSUP when the configuration is outside
// what the fused kernel holds on chip (the caller then runs the staged
// CUDA-core kernels).
int launch_cqt2010_tc(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, const float* k_re,
                      const float* k_im, int n_filt, int width, int early_stages, int n_oct, int kernel_hop,
                      int first_bin, int bpo, int n_bins, int pad_mode, int out_kind, int T, float* out,
                      void* workspace, size_t workspace_bytes, cudaStream_t st) {
  Plan pl;
  int rc = make_plan(L, n_taps, taps, n_filt, width, early_stages, n_oct, kernel_hop, pad_mode, &pl);
  if (rc) return rc;
  TcParams& p = pl.p;
  const int grid = (int)std::min<int64_t>(B, (int64_t)num_sms() * pl.ctas_per_sm);
  if (!workspace || workspace_bytes < (size_t)grid * pl.scratch_bytes_per_cta ||
      reinterpret_cast<uintptr_t>(workspace) % 16)
    return NNAB_ENOTSUP;
  p.x = x;
  p.B = B;
  p.first_bin = first_bin;
  p.bpo = bpo;
  p.n_bins = n_bins;
  p.n_filt = n_filt;
  p.width = width;
  p.T = T;
  p.out_kind = out_kind;
  p.h0 = taps[127];
  for (int j = 0; j < 128; ++j) p.g[j] = taps[2 * j];
  p.k_re = k_re;
  p.k_im = k_im;
  p.out = out;
  p.scratch = reinterpret_cast<__half*>(workspace);
  p.prof = cqt2010_prof_ptr();
  NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt2010_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  cqt2010_tc_kernel<<<grid, kThreads, pl.smem, st>>>(p);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

}  // namespace nnab
