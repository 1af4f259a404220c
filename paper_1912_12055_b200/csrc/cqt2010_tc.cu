// CQT2010v2 on the tensor cores, one persistent CTA per SM, one clip at a time,
// the whole chain on chip so HBM sees only the clip and its output
// (transforms.py:290-313, signal.py:232-247).
//
// Half-band FIR as a banded Toeplitz MMA.  downsample2 keeps
//   y[i] = sum_d h[d] x_ext[2i + d],  d = -127..127 (reflect-extended x)
// and the cutoff-0.5 windowed sinc is half-band: every even d != 0 is <= 6.6e-17,
// so  y[i] = h0 * x[2i] + sum_{j=0}^{127} g_j * xo[i + j],  g_j = h[2j - 127],
// xo[n] = x_ext[2n - 127 + 2*i0] (the odd phase).  A block of 128 outputs is
// Y[r] = sum_s T[r][s] W[s], T[r][s] = g_{s-r} (a 128 x 256 Toeplitz band) and
// W = 256 consecutive odd-phase samples; blocks overlap by 128 samples.
//   A = T with its rows reversed: A'[r'][s] = g[s + r' - 127] depends on s + r'
//       only, so the whole band lives in a 6 KB "diagonal" smem array that a
//       no-swizzle K-major descriptor with LBO = 64 B walks (toep_desc),
//   B = the windows of NB blocks: odd-phase samples stored once in smem as 32
//       "planes" of 16 bytes x (NB+1) rows; block n's window is rows n, n+1,
//       which the no-swizzle K-major UMMA descriptor expresses as a 16-byte
//       start offset (LBO = plane stride, SBO = 8 rows).
//   D = TMEM, lanes = 127 - output offset, columns = blocks -> the epilogue adds
//       the centre tap h0 * x[2i] in FP32 and writes the next stage.
// A K=8 tcgen05.mma costs ~100 cycles whatever N <= 128 is (measured,
// tools/mma_probe.cu: the 4 KB A read dominates), so chunks carry as many blocks
// as shared memory allows (64 for stage 1, read straight from global memory; 32
// for stage 2) and the K = 256 reduction is split over 4 independent accumulators.
// Per-octave centred complex conv (12 bins x 90 taps, hop 128 >> alpha) is an
// im2col MMA: A = 128 frames x 96 taps (SW128, built from smem), B = 32 rows
// (re/im of each bin) x 96 taps, D = 128 x 32 in TMEM.
// TF32 operands are rounded to nearest (not truncated) when staged, so the
// 8-stage cascade carries no rounding bias.
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kThreads = 512;
constexpr int NB1 = 64;               // blocks per chunk: stage 1 (x from global) and octave halvings
constexpr int NB2 = 32;               // blocks per chunk: stage 2 (from the stage-1 window)
constexpr int CH1 = NB1 * 128;        // 8192 outputs
constexpr int CH2 = NB2 * 128;        // 4096 outputs
constexpr int KCH = 4;                // independent accumulator chains (K quarters)
constexpr int MARG = 128;             // reflect margin of the smem octave signals
constexpr int E1W = 2 * CH2 + 256 + CH1;  // rolling window of stage-1 outputs (16640)
constexpr int KC = 96;                // conv taps padded (3 K blocks of 32)
constexpr int NCONV = 32;             // conv B rows (re/im of <= 16 bins)
// im2col column m' holds signal offset m' - pad_al (pad_al = pad rounded up to 4) so
// every 16-byte A chunk is one aligned float4; the filters move right by pad_al - pad.
constexpr int PLANES_BYTES = 32 * (NB1 + 1) * 16;
constexpr int TOEP_CHUNKS = 256 + 128;  // 16-byte chunks of the diagonal Toeplitz layout
constexpr int TOEP_BYTES = TOEP_CHUNKS * 16;

struct TcParams {
  const float* x;
  int64_t B, L;
  int32_t L0;                        // octave-0 length after the two early halvings
  int32_t n_oct, kernel_hop, first_bin, bpo, n_bins, n_filt, width, T, out_kind;
  float h0;                          // centre tap
  float g[128];                      // odd taps g_j = h[2j - 127]
  const float* k_re;                 // top-octave bank (n_filt, width), device
  const float* k_im;
  float* out;
  int32_t sig0_cap, sig1_cap;        // floats
  unsigned long long* prof;          // optional per-phase cycle counters (nnab_debug_cqt2010_profile)
};

// Phase clock for thread 0 of each CTA (only when p.prof is set).
struct Prof {
  long long t = 0;
  unsigned long long acc[16] = {};
  NNAB_DEV void mark(const TcParams& p, int i) {
    if (p.prof && threadIdx.x == 0) {
      const long long n = clock64();
      acc[i] += (unsigned long long)(n - t);
      t = n;
    }
  }
};

struct Smem {
  uint8_t* toep;    // TOEP_BYTES: chunk j = (g[j-127], g[j-126], g[j-125], g[j-124])
  uint8_t* planes;  // PLANES_BYTES
  float* sig0;      // sig0_cap
  float* e1w;       // E1W          (early phase)
  float* sig1;      // sig1_cap     (octave phase; aliases e1w)
  uint8_t* convA;   // 3 x 16 KB    (octave phase)
  uint8_t* convB;   // 3 x 4 KB
  uint64_t* bars;   // [0] mma
  uint32_t* tslot;
};

NNAB_DEV int64_t refl(int64_t j, int64_t n) {
  if (j < 0) j = -j;
  if (j >= n) j = 2 * (n - 1) - j;
  return j;
}

template <int NB>
NNAB_DEV uint64_t plane_desc(uint32_t addr) {  // no-swizzle K-major: LBO = plane stride, SBO = 8 rows x 16 B
  constexpr uint32_t plane = (NB + 1) * 16;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((plane >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// Reversed-row Toeplitz A'[r'][s] = g[s + r' - 127] depends on s + r' only, so with a
// no-swizzle K-major descriptor of LBO = 64 B (next 4 K) and SBO = 128 B (next 8
// rows) every 16-byte core-matrix row (r', s..s+3) lands on chunk s + r' of a
// 6 KB array: the whole 128 x 256 band in 6 KB of smem instead of 128 KB.
NNAB_DEV uint64_t toep_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(64 >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
NNAB_DEV uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Source of a halving chunk in shared memory: src[0] = ext[2*o0 - 128].
struct SmemSrc {
  const float* src;
  NNAB_DEV float4 odd4(int c) const {  // ext[2*o0 - 127 + 8c + {0,2,4,6}]
    const float4 a = *reinterpret_cast<const float4*>(src + 8 * c);
    const float4 b = *reinterpret_cast<const float4*>(src + 8 * c + 4);
    return make_float4(a.y, a.w, b.y, b.w);
  }
  NNAB_DEV float centre(int i) const { return src[2 * i + 128]; }
};
// Stage-1 source straight from the clip in global memory (reflect at its ends).
struct GlobalSrc {
  const float* xb;
  int64_t s0, L;  // s0 = 2*o0 - 128
  bool vec;       // interior span and 16-byte aligned: float4 loads
  NNAB_DEV float at(int64_t u) const { return __ldg(xb + refl(s0 + u, L)); }
  NNAB_DEV float4 odd4(int c) const {
    if (vec) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(xb + s0 + 8 * c));
      const float4 b = __ldg(reinterpret_cast<const float4*>(xb + s0 + 8 * c + 4));
      return make_float4(a.y, a.w, b.y, b.w);
    }
    return make_float4(at(8 * c + 1), at(8 * c + 3), at(8 * c + 5), at(8 * c + 7));
  }
  NNAB_DEV float centre(int i) const { return vec ? __ldg(xb + s0 + 2 * i + 128) : at(2 * i + 128); }
};

// One FIR halving chunk: out[i] = h0*ext[2(o0+i)] + sum_j g_j xo[i+j], i < n_out (<= NB*128),
// delivered to emit(i, value).  All threads call; thread 0 issues the MMAs.
template <int NB, class Src, class Emit>
NNAB_DEV void fir_chunk(const TcParams& p, const Smem& s, const Src& src, int n_out, uint32_t tmem_a,
                        uint32_t tmem_d, uint32_t& mma_phase, Emit emit, Prof& pf, int ph) {
  constexpr int PROWS = NB + 1, PLANE = PROWS * 16;
  const int tid = threadIdx.x;
  // 1. odd phase -> planes (rows of 128 samples, 16-byte chunk q of a row in plane q),
  //    TF32-rounded.  Only the rows the n_out outputs need are built; stale rows
  //    only feed discarded columns.
  const int rows = min(PROWS, (n_out + 127) / 128 + 1);
  for (int c = tid; c < rows * 32; c += kThreads) {
    const float4 a = src.odd4(c);
    const int row = c >> 5, q = c & 31;
    *reinterpret_cast<float4*>(s.planes + q * PLANE + row * 16) =
        make_float4(tf32_rne(a.x), tf32_rne(a.y), tf32_rne(a.z), tf32_rne(a.w));
  }
  fence_proxy_async_smem();
  __syncthreads();
  pf.mark(p, ph + 0);
  // 2. 32 MMAs (K = 256 in steps of 8) over KCH accumulators issued round-robin
  if (tid == 0) {
    tc_fence_after();
    const uint32_t idesc = idesc_tf32(128, NB);
    const uint32_t pbase = smem_u32(s.planes), tbase_s = smem_u32(s.toep);
#pragma unroll 1
    for (int kk = 0; kk < 32 / KCH; ++kk) {
#pragma unroll
      for (int c = 0; c < KCH; ++c) {
        const int k = c * (32 / KCH) + kk;
        const int sidx = 8 * k;  // window index of this K step
        const uint32_t addr = pbase + ((sidx & 127) >> 2) * PLANE + (sidx >> 7) * 16;
        mma_tf32(tmem_d + c * NB, toep_desc(tbase_s + 16 * sidx), plane_desc<NB>(addr), idesc, kk > 0);
      }
    }
    mma_commit(&s.bars[0]);
  }
  mbar_wait(&s.bars[0], mma_phase);
  mma_phase ^= 1;
  tc_fence_after();
  pf.mark(p, ph + 1);
  // 3. epilogue: all 16 warps; warp w reads lane quarter w%4, blocks [g*NB/4, (g+1)*NB/4), g = w/4
  {
    const int warp = tid >> 5, quarter = warp & 3, grp = warp >> 2;
    const int r = 127 - (quarter * 32 + (tid & 31));  // accumulator rows are reversed output offsets
    constexpr int NPG = NB / 4;  // blocks per warp group
    float acc[NPG], v[NPG];
    const uint32_t lane_base = tmem_d + ((uint32_t)(quarter * 32) << 16) + grp * NPG;
#pragma unroll
    for (int c = 0; c < KCH; ++c) {
      if constexpr (NPG == 16) tmem_ld16(lane_base + c * NB, v);
      else tmem_ld8(lane_base + c * NB, v);
      tmem_ld_wait();
#pragma unroll
      for (int n = 0; n < NPG; ++n) acc[n] = c ? acc[n] + v[n] : v[n];
    }
    float cen[NPG];
#pragma unroll
    for (int n = 0; n < NPG; ++n) {  // issue every centre-tap load before using any
      const int i = (grp * NPG + n) * 128 + r;
      cen[n] = i < n_out ? src.centre(i) : 0.f;
    }
#pragma unroll
    for (int n = 0; n < NPG; ++n) {
      const int i = (grp * NPG + n) * 128 + r;
      if (i < n_out) emit(i, fmaf(p.h0, cen[n], acc[n]));
    }
  }
  tc_fence_before();
  __syncthreads();
  pf.mark(p, ph + 2);
}

// Fill the reflect margins of a smem signal sig[MARG + i], i < n (np.pad "reflect").
NNAB_DEV void fill_margins(float* sig, int n, int right) {
  for (int m = threadIdx.x + 1; m <= MARG; m += kThreads) sig[MARG - m] = sig[MARG + (int)refl(-m, n)];
  for (int m = threadIdx.x; m < right; m += kThreads) {  // beyond one reflection: zero (never a kept output)
    const int j = 2 * (n - 1) - (n + m);
    sig[MARG + n + m] = j >= 0 ? sig[MARG + j] : 0.f;
  }
  __syncthreads();
}

// Centred complex conv of one octave (frames t < T), written to out rows.
NNAB_DEV void octave_conv(const TcParams& p, const Smem& s, const float* sig, int hop, int alpha, int64_t b,
                          uint32_t tmem_d, uint32_t& mma_phase, Prof& pf) {
  const int tid = threadIdx.x;
  const int pad = p.width / 2;
  const int skip = max(0, alpha * p.bpo - p.first_bin);
  const int row0 = p.first_bin - alpha * p.bpo;
  for (int tile = 0; tile * 128 < p.T; ++tile) {
    // im2col A (128 frames x 96 taps), SW128 K-major: K block kb at kb*16 KB,
    // row t at t*128 B, 16-byte chunk c stored at chunk (c ^ (t & 7)).
    const int pad_al = (pad + 3) & ~3;
    for (int e = tid; e < 128 * (KC / 4); e += kThreads) {
      const int t = e / (KC / 4), c = e - t * (KC / 4);  // chunk c = columns 4c..4c+3
      const int tt = tile * 128 + t;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (tt < p.T) {
        const float* src = sig + MARG + tt * hop - pad_al + 4 * c;
        float4 w;
        if ((hop & 3) == 0) {
          w = *reinterpret_cast<const float4*>(src);  // 16-byte aligned
        } else {
          w = make_float4(src[0], src[1], src[2], src[3]);
        }
        v = make_float4(tf32_rne(w.x), tf32_rne(w.y), tf32_rne(w.z), tf32_rne(w.w));
      }
      const int kb = c >> 3, cc = c & 7;
      *reinterpret_cast<float4*>(s.convA + kb * 16384 + t * 128 + ((cc ^ (t & 7)) << 4)) = v;
    }
    fence_proxy_async_smem();
    __syncthreads();
    pf.mark(p, 9);
    if (tid == 0) {
      tc_fence_after();
      const uint32_t idesc = idesc_tf32(128, NCONV);
      const uint32_t a0 = smem_u32(s.convA), b0 = smem_u32(s.convB);
#pragma unroll 1
      for (int k = 0; k < KC / 8; ++k) {
        const int kb = k >> 2, ks = k & 3;
        mma_tf32(tmem_d, sw128_desc(a0 + kb * 16384) + (uint64_t)(ks * 2), sw128_desc(b0 + kb * 4096) + (uint64_t)(ks * 2),
                 idesc, k > 0);
      }
      mma_commit(&s.bars[0]);
    }
    mbar_wait(&s.bars[0], mma_phase);
    mma_phase ^= 1;
    tc_fence_after();
    pf.mark(p, 10);
    {  // warp w: lane quarter w%4 (frames), columns [8g, 8g+8) = bins 4g..4g+3, g = w/4
      const int warp = tid >> 5, quarter = warp & 3, grp = warp >> 2;
      const int t = tile * 128 + quarter * 32 + (tid & 31);
      float v[8];
      tmem_ld8(tmem_d + ((uint32_t)(quarter * 32) << 16) + grp * 8, v);
      tmem_ld_wait();
      if (t < p.T) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = grp * 4 + jj;
          if (j < skip || j >= p.n_filt) continue;
          const float re = v[2 * jj], im = v[2 * jj + 1];
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
    tc_fence_before();
    __syncthreads();
    pf.mark(p, 11);
  }
}

__global__ void __launch_bounds__(kThreads, 1) cqt2010_tc_kernel(const __grid_constant__ TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Smem s;
  uint8_t* q = base;
  s.convB = q;                                   q += 3 * 4096;
  s.toep = q;                                    q += TOEP_BYTES;
  s.planes = q;                                  q += PLANES_BYTES;
  q = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(q) + 1023) & ~uintptr_t(1023));
  s.convA = q;                                   q += 3 * 16384;   // octave phase
  s.sig1 = reinterpret_cast<float*>(q);          // octave phase
  s.e1w = reinterpret_cast<float*>(s.convA);     // early phase: aliases convA + sig1
  const size_t late = (size_t)p.sig1_cap * 4, early = (size_t)E1W * 4 - 3 * 16384;
  q += late > early ? late : early;
  s.sig0 = reinterpret_cast<float*>(q);          q += (size_t)p.sig0_cap * 4;
  s.bars = reinterpret_cast<uint64_t*>(q);       q += 4 * 8;
  s.tslot = reinterpret_cast<uint32_t*>(q);

  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&s.bars[0], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(s.tslot);
  // conv B (filters): row 2j = Re k_j, 2j+1 = Im k_j; SW128 K-major, TF32; column m
  // holds tap m - shift (shift = pad_al - pad, see octave_conv)
  const int shift = ((p.width / 2 + 3) & ~3) - p.width / 2;
  for (int e = tid; e < NCONV * KC; e += kThreads) {
    const int n = e / KC, m = e % KC, j = n >> 1, tap = m - shift;
    float v = 0.f;
    if (j < p.n_filt && tap >= 0 && tap < p.width) v = tf32_rne(((n & 1) ? p.k_im : p.k_re)[(int64_t)j * p.width + tap]);
    const int kb = m >> 5, cc = (m & 31) >> 2;
    reinterpret_cast<float*>(s.convB + kb * 4096 + n * 128 + ((cc ^ (n & 7)) << 4))[m & 3] = v;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *s.tslot;
  const uint32_t tmem_a = tbase, tmem_d = tbase + 256;
  // diagonal Toeplitz chunks (see toep_desc), TF32-rounded
  for (int j = tid; j < TOEP_CHUNKS; j += kThreads) {
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int gi = j - 127 + e;
      v[e] = (gi >= 0 && gi < 128) ? tf32_rne(p.g[gi]) : 0.f;
    }
    *reinterpret_cast<float4*>(s.toep + 16 * j) = make_float4(v[0], v[1], v[2], v[3]);
  }
  fence_proxy_async_smem();
  __syncthreads();

  uint32_t mma_phase = 0;
  Prof pf;
  if (p.prof && tid == 0) pf.t = clock64();
  const int64_t L1 = (p.L + 1) / 2;
  const int L0 = p.L0;
  const int nc2 = (L0 + CH2 - 1) / CH2;
  for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
    // ------------------------------------------------ early stages: x -> E1 -> E2 (= octave 0)
    const float* xb = p.x + b * p.L;
    int64_t computed = 0;  // stage-1 positions [0, computed) produced so far
    for (int c = 0; c < nc2; ++c) {
      const int64_t ws = 2ll * CH2 * c - 128;  // stage-1 position of e1w[0]
      const int64_t need0 = 2ll * CH2 * c + 2 * CH2 + 128;
      const int64_t need = need0 < L1 ? need0 : L1;
      while (computed < need) {
        const int64_t o0 = computed;  // chunk start (multiple of CH1)
        const int n_out = (int)(L1 - o0 < CH1 ? L1 - o0 : CH1);
        GlobalSrc src{xb, 2 * o0 - 128, p.L, false};
        src.vec = src.s0 >= 0 && src.s0 + 2ll * n_out + 512 <= p.L && (p.L % 4) == 0;
        float* w = s.e1w + (o0 - ws);
        fir_chunk<NB1>(p, s, src, n_out, tmem_a, tmem_d, mma_phase, [&](int i, float v) { w[i] = v; }, pf, 0);
        computed = o0 + n_out;
      }
      // reflect stage 1 about its ends (downsample2 pads its input, signal.py:245)
      for (int u = tid; u < 2 * CH2 + 256; u += kThreads) {
        const int64_t pos = ws + u;
        if (pos < 0 || pos >= L1) s.e1w[u] = s.e1w[refl(pos, L1) - ws];
      }
      __syncthreads();
      pf.mark(p, 14);
      const int n2 = min(CH2, L0 - CH2 * c);
      float* o = s.sig0 + MARG + CH2 * c;
      fir_chunk<NB2>(p, s, SmemSrc{s.e1w}, n2, tmem_a, tmem_d, mma_phase, [&](int i, float v) { o[i] = v; }, pf, 3);
      const int64_t keep = computed - (ws + 2 * CH2);
      for (int64_t u = tid; u < keep; u += kThreads) s.e1w[u] = s.e1w[u + 2 * CH2];
      __syncthreads();
      pf.mark(p, 14);
    }
    // ------------------------------------------------ octaves: conv, halve, repeat (all in smem)
    fill_margins(s.sig0, L0, 512);
    float* sig = s.sig0;
    float* nxt = s.sig1;
    int n = L0;
    for (int a = 0; a < p.n_oct; ++a) {
      pf.mark(p, 15);
      octave_conv(p, s, sig, p.kernel_hop >> a, a, b, tmem_d, mma_phase, pf);
      if (a + 1 == p.n_oct) break;
      const int nl = (n + 1) / 2;
      for (int o0 = 0; o0 < nl; o0 += CH1) {
        float* o = nxt + MARG + o0;
        fir_chunk<NB1>(p, s, SmemSrc{sig + 2 * o0}, min(CH1, nl - o0), tmem_a, tmem_d, mma_phase,
                       [&](int i, float v) { o[i] = v; }, pf, 6);
      }
      fill_margins(nxt, nl, 512);
      float* t = sig;
      sig = nxt;
      nxt = t;
      n = nl;
    }
    pf.mark(p, 15);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tbase);
  if (p.prof && tid == 0)
    for (int i = 0; i < 16; ++i) atomicAdd(p.prof + i, pf.acc[i]);
}

__device__ unsigned long long g_cqt_prof[16];
bool g_cqt_prof_on = false;
unsigned long long* cqt2010_prof_ptr() {
  if (!g_cqt_prof_on) return nullptr;
  void* ptr = nullptr;
  cudaGetSymbolAddress(&ptr, g_cqt_prof);
  return reinterpret_cast<unsigned long long*>(ptr);
}

}  // namespace

// Debug: enable per-phase cycle counters of the fused kernel (on != 0), or read
// and clear them into out[16] (on == 0).  Phases: 0-2 stage-1 build/mma/epilogue,
// 3-5 stage 2, 6-8 octave halvings, 9-11 conv build/mma/epilogue, 14 stage-1
// reflect + window shift, 15 octave margins + loop.
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

// Fused tensor-core CQT2010v2; returns NNAB_ENOTSUP when the configuration is
// outside what the fused kernel holds on chip (caller falls back to the staged
// CUDA-core kernels).
int launch_cqt2010_tc(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, const float* k_re,
                      const float* k_im, int n_filt, int width, int early_stages, int n_oct, int kernel_hop,
                      int first_bin, int bpo, int n_bins, int pad_mode, int out_kind, int T, float* out,
                      cudaStream_t st) {
  if (early_stages != 2 || n_taps != 255 || pad_mode != NNAB_PAD_REFLECT) return NNAB_ENOTSUP;
  if (n_filt > NCONV / 2 || width + 3 > KC || n_oct < 1) return NNAB_ENOTSUP;
  const int64_t L1 = (L + 1) / 2, L0 = (L1 + 1) / 2;
  if (L0 > 24576 || L0 < 256) return NNAB_ENOTSUP;
  // half-band check: even offsets (odd tap indices) are negligible
  float hmax = 0.f;
  for (int i = 0; i < n_taps; ++i) hmax = std::max(hmax, std::fabs(taps[i]));
  for (int i = 1; i < n_taps; i += 2)
    if (i != 127 && std::fabs(taps[i]) > 1e-12f * hmax) return NNAB_ENOTSUP;
  TcParams p{};
  p.x = x;
  p.B = B;
  p.L = L;
  p.L0 = (int32_t)L0;
  p.n_oct = n_oct;
  p.kernel_hop = kernel_hop;
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
  p.prof = cqt2010_prof_ptr();
  p.sig0_cap = (int32_t)((MARG + L0 + 512 + 3) & ~3);  // multiples of 4 floats: float4-aligned buffers
  p.sig1_cap = (int32_t)((MARG + (L0 + 1) / 2 + 512 + 3) & ~3);
  const size_t late = (size_t)p.sig1_cap * 4, early = (size_t)E1W * 4 - 3 * 16384;
  const size_t smem = 1024 + 3 * 4096 + TOEP_BYTES + PLANES_BYTES + 1024 + 3 * 16384 + std::max(late, early) +
                      (size_t)p.sig0_cap * 4 + 64;
  if (smem > 227 * 1024) return NNAB_ENOTSUP;
  NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt2010_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>(B, num_sms());
  cqt2010_tc_kernel<<<grid, kThreads, smem, st>>>(p);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

}  // namespace nnab
