// CQT2010v2 front: the two early halvings (x -> y1 -> octave 0, signal.py:232-247 applied
// twice by transforms.py:290-292) of every clip, x streamed from HBM once, y1 kept on chip,
// octave 0 written to the level buffer the batched halvings / convs read
// (cqt2010_tc.cu).  One persistent CTA per SM walks its clips; every role is its own
// warp set so the HBM stream, the operand conversion, the tensor-core FIRs and the
// epilogues of consecutive tiles and clips overlap:
//
//   warp 5       scan: the peak of the NEXT clip's first kPeek samples (the whole clip in
//                the exact relaunch) -> the clip's power-of-two scale exponent
//   warps 0-3    epilogue: stage-1 D -> y1 (odd phase -> stage-2 planes, even ->
//                stage-2 centre planes), y1's reflect images, stage-2 D -> octave 0 (+
//                its reflect margins) in the level buffer
//   warp 4       MMA issue (one thread) + TMEM allocation (512 columns)
//   warps 6-19   converters: the tile's clip segment from HBM (10 float4 loads in flight
//                per thread) -> scaled FP16, odd phase -> stage-1 "planes", even phase ->
//                centre-tap planes, into one of two stage-1 operand buffers
//
// The half-band FIR as tensor-core MMAs (the fused kernel's formulation, cqt2010_tc.cu):
// y[i] = h0 x[2i] + sum_j g_j xo[i + j], xo[m] = x_ext[2m - 127]; block n = 128 outputs,
// D[n][r'] (r' = 127 - r) = sum_s xo[128 n + s] g[s - r]  (K = 256: odd planes rows n, n+1,
// B = the Toeplitz band as a diagonal chunk array) + sum_s xe[128 n + s] h0 [s = r]
// (K = 128: the even phase, B = h0 on the reversed diagonal) -- the centre tap is an MMA
// too, so the epilogue reads nothing but TMEM.  24 MMAs (M = N = 128, K = 16) per tile.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace nnab {
namespace {

constexpr int kML = 128;                 // level-buffer reflect margins (cqt2010_tc.cu ML)
constexpr int kToepChunks = 8 * 31 + 128;  // Toeplitz diagonal chunks (cqt2010_tc.cu TOEP_CHUNKS)
constexpr int kCenChunks = 256;
constexpr int kScanWarps = 1;
constexpr int kScanBatch = 24;           // float4 loads in flight per scan thread
constexpr int kEpiWarp0 = 0, kMmaWarp = 4, kScanWarp0 = 5, kConvWarp0 = 6, kConvWarps = 14;  // 20 warps (12: 0.322 ms, 16 / 18: 0.318 / 0.320;
                                                                                             // 8 epilogue warps: 0.323-0.33)
constexpr int kCT = 32 * kConvWarps;     // converter threads
constexpr int kRowU = kCT / 64;          // plane rows one float4 step of every converter thread covers
constexpr int kConvBatch = 10;           // float4 loads in flight per converter thread
constexpr int kThreads = (kConvWarp0 + kConvWarps) * 32;
static_assert(kScanWarps == 1, "the scan role is one warp");

struct FrontParams {
  const float* x;
  int64_t B;
  int32_t L, L1, L0;
  int32_t nb1, n1;          // stage-1 blocks / tiles
  int32_t nb2, row_b;       // stage-2 blocks; first row of the second stage-2 tile (0: one tile)
  int32_t pl1, pe1, pl2, pe2, yr;  // plane strides (bytes), stage-2 plane rows
  int32_t off_toep, off_cen, off_a1[2], off_yo, off_ye, off_bars;  // a1: odd planes, then even planes
  float h0;
  float g[128];
  __half* lv0;
  int32_t lv0_stride;
  int32_t* exps;
  unsigned long long* prof;  // debug: per-role wait cycles (nnab_debug_cqt2010_front_profile), or null
  // scale: exact = 0 (fast): the scale comes from the clip's first kPeek samples with kHead
  // bits of headroom, and a clip whose peak would leave that headroom (or whose first
  // kPeek samples are all zero) is appended to out_list; exact = 1: the exact peak of the
  // whole clip (a full scan), over the clips listed in list[0 .. *list_n) (the flagged ones)
  int32_t exact;
  CqtPrepArgs prep;       // fast launch: the back end's bank images (toep_img null: none)
  int32_t* out_list;      // fast launch: flagged clips appended here ...
  int32_t* out_list_n;    // ... (count, zeroed before the launch)
  const int32_t* list;
  const int32_t* list_n;
};
constexpr int kPeek = 2048;  // samples the fast scale looks at
constexpr int kHead = 8;     // headroom bits of the fast scale: the rest of the clip may be 2^(kHead + 13) louder

NNAB_DEV uint64_t nsw(uint32_t addr, uint32_t lbo, uint32_t sbo) {  // no-swizzle K-major descriptor
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

NNAB_DEV float4 ldg_keep(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// mbar_wait that adds the cycles spent to acc (debug profile)
// (the waiting thread is suspended in mbarrier.try_wait up to a time hint instead of
// spinning: a dozen waiting warps would otherwise take issue slots from the converters)
NNAB_DEV bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(20000u) : "memory");
  return ok != 0;
}
// per-role wait cycles only in a profiling build (-DNNAB_FRONT_PROF): the accumulators would
// otherwise sit in local memory on every wait of the production kernel
NNAB_DEV void wait_p(uint64_t* bar, uint32_t parity, unsigned long long& acc) {
#ifdef NNAB_FRONT_PROF
  const long long t0 = clock64();
#endif
  for (uint32_t it = 0; !mbar_try_wait_hint(bar, parity); ++it)
    if (it > (1u << 22)) __trap();  // a pipeline bug traps instead of hanging the GPU
#ifdef NNAB_FRONT_PROF
  acc += (unsigned long long)(clock64() - t0);
#else
  (void)acc;
#endif
}

__device__ long long g_front_tl[16 * 12];
NNAB_DEV void tl_mark(const FrontParams& p, int k, int ev, long long t0) {
  if (p.prof && blockIdx.x == 0 && k < 16) g_front_tl[12 * k + ev] = clock64() - t0;
}

NNAB_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

NNAB_DEV float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
NNAB_DEV void sts32(uint32_t a, uint32_t v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }

NNAB_DEV uint32_t pack2(float a, float b);
// float4 at ext index e of a clip at its edges: the reflect images (np.pad "reflect",
// signal.py:245) from L2; zeros past the tile end e1 (never a kept output)
__device__ __noinline__ float4 edge_float4(int e, int e1, int L, const float* xb) {
  float w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int r = e + q;
    if (r < 0) r = -r;
    if (r >= L) r = 2 * (L - 1) - r;
    w[q] = (e < e1 && r >= 0 && r < L) ? __ldg(xb + r) : 0.f;
  }
  return make_float4(w[0], w[1], w[2], w[3]);
}

NNAB_DEV uint32_t pack2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// one FIR tile: 16 odd-phase K steps (planes rows row0, row0 + 1) + 8 centre-tap K steps
NNAB_DEV void issue_tile(uint32_t d_tmem, uint32_t odd, uint32_t pl, uint32_t even, uint32_t pe, int row0,
                         uint32_t toep, uint32_t cen) {
  constexpr uint32_t idesc = idesc_f16(128, 128);
#pragma unroll
  for (int k = 0; k < 16; ++k)
    mma_f16(d_tmem, nsw(odd + (uint32_t)(2 * (k & 7)) * pl + (uint32_t)(row0 + (k >> 3)) * 16u, pl, 128),
            nsw(toep + 256u * k, 128, 128), idesc, k > 0);
#pragma unroll
  for (int k = 0; k < 8; ++k)
    mma_f16(d_tmem, nsw(even + (uint32_t)(2 * k) * pe + (uint32_t)row0 * 16u, pe, 128), nsw(cen + 256u * k, 128, 128),
            idesc, 1);
}

__global__ void __launch_bounds__(kThreads, 1) cqt2010_front_kernel(const __grid_constant__ FrontParams p) {
  // the exact relaunch over the flagged clips: CTAs without a listed clip leave at once
  // (usually all of them: no TMEM allocation, no shared-memory setup)
  if (p.list && (int64_t)*p.list_n <= (int64_t)blockIdx.x) return;
  if (p.prep.toep_img) {  // the back end's bank images (cqt2010_prep_kernel's formulas), spread over the grid
    const int gt = blockIdx.x * kThreads + threadIdx.x, gn = gridDim.x * kThreads;
    for (int j = gt; j < kToepChunks; j += gn) {  // chunk j = g[j - 127 + e]
      __align__(16) __half v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int gi = j - 127 + e;
        v[e] = __float2half_rn((gi >= 0 && gi < 128) ? p.g[gi] : 0.f);
      }
      p.prep.toep_img[j] = *reinterpret_cast<uint4*>(v);
    }
    __half* f = reinterpret_cast<__half*>(p.prep.filt_img);
    for (int e = gt; e < p.prep.nconv * p.prep.kc; e += gn) {
      const int n = e / p.prep.kc, m = e % p.prep.kc, j = n >> 1, tap = m - p.prep.shift;
      float v = 0.f;
      if (j < p.prep.n_filt && tap >= 0 && tap < p.prep.width)
        v = ldexpf(((n & 1) ? p.prep.k_im : p.prep.k_re)[(int64_t)j * p.prep.width + tap], p.prep.filt_log2);
      f[(m >> 3) * (8 * p.prep.nconv) + n * 8 + (m & 7)] = __float2half_rn(v);
    }
  }
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + p.off_bars);
  uint64_t* ex_ready = bars;                        // [2] scan
  uint64_t* conv_start = ex_ready + 2;              // converter took a clip's exponent
  uint64_t* a_full = conv_start + 1;                // [2] converter threads
  uint64_t* a_empty = a_full + 2;                   // [2] commit
  uint64_t* s1_done = a_empty + 2;                  // [2] commit
  uint64_t* s1_free = s1_done + 2;                  // [2] 4 epilogue warps
  uint64_t* s2_ready = s1_free + 2;                 // 128 epilogue threads
  uint64_t* s2_done = s2_ready + 1;                 // commit
  uint64_t* s2_free = s2_done + 1;                  // 4 epilogue warps
  uint32_t* tslot = reinterpret_cast<uint32_t*>(s2_free + 1);
  int* ex_slot = reinterpret_cast<int*>(tslot + 1);     // [2] scale exponent, [2] peek-was-zero
  float* scan_part = reinterpret_cast<float*>(ex_slot + 4);  // [2][kScanWarps]
  unsigned* conv_max = reinterpret_cast<unsigned*>(scan_part + 2 * kScanWarps);  // [2] converter peak bits
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    mbar_init(&ex_ready[0], 1);
    mbar_init(&ex_ready[1], 1);
    mbar_init(conv_start, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], kConvWarps);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s1_done[i], 1);
      mbar_init(&s1_free[i], 4);
    }
    mbar_init(s2_ready, 128);
    mbar_init(s2_done, 1);
    mbar_init(s2_free, 4);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tslot);
  if (tid < 2) conv_max[tid] = 0u;
  // operand regions start zeroed: the stage-2 windows of real blocks read plane rows past
  // the signal at zero Toeplitz weight (0 * NaN would poison them); everything written
  // later is finite
  for (int i = tid; i < (p.off_bars - p.off_a1[0]) / 16; i += kThreads)
    reinterpret_cast<uint4*>(base + p.off_a1[0])[i] = make_uint4(0, 0, 0, 0);
  for (int j = tid; j < kToepChunks; j += kThreads) {  // chunk j = g[j - 127 + e]
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int gi = j - 127 + e;
      v[e] = __float2half_rn((gi >= 0 && gi < 128) ? p.g[gi] : 0.f);
    }
    *reinterpret_cast<uint4*>(base + p.off_toep + 16 * j) = *reinterpret_cast<uint4*>(v);
  }
  for (int j = tid; j < kCenChunks; j += kThreads) {  // chunk c = h0 at e = 127 - c
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float2half_rn(j + e == 127 ? p.h0 : 0.f);
    *reinterpret_cast<uint4*>(base + p.off_cen + 16 * j) = *reinterpret_cast<uint4*>(v);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  unsigned long long pf[4] = {0, 0, 0, 0};
  const long long t_begin = clock64();
  const int64_t n_all = p.list ? (int64_t)*p.list_n : p.B;  // clips this launch walks
  const int n_clips = n_all > blockIdx.x ? (int)((n_all - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
  auto clip_of = [&](int k) {
    const int64_t i = (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
    return p.list ? (int64_t)p.list[i] : i;
  };

  if (warp == kScanWarp0) {
    const int st = tid - kScanWarp0 * 32;
    // ------------------------------------------------------------ scan: exponent of each clip
    const uint64_t keep = policy_evict_last();
    const int n4 = p.L / 4;
    for (int k = 0; k < n_clips; ++k) {
      if (k > 0) wait_p(conv_start, (k - 1) & 1, pf[0]);  // the converter is on clip k - 1
      if (st == 0) tl_mark(p, k, 0, t_begin);
      const float* xb = p.x + clip_of(k) * p.L;
      // (no L2 bulk prefetch of the clip: prefetching the next one ahead of the converters
      // made the route 0.325 -> 0.357 ms, two or three clips ahead 0.38 ms -- the prefetches
      // compete with the converters' demand loads)
      float mx = 0.f;
      const int n4s = p.exact ? n4 : min(n4, kPeek / 4);  // fast: the first kPeek samples
      for (int f0 = st; f0 < n4s; f0 += kScanBatch * 32) {
        float4 v[kScanBatch];
#pragma unroll
        for (int u = 0; u < kScanBatch; ++u) {
          const int f = f0 + u * 32;
          v[u] = f < n4s ? ldg_keep(xb + 4 * f, keep) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kScanBatch; ++u)
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (st == 0) {
        const float m = mx;
        int ex = 0;
        if (m > 0.f && m < INFINITY) frexpf(m, &ex);
        ex_slot[k & 1] = p.exact ? ex : ex + kHead;
        ex_slot[2 + (k & 1)] = !p.exact && !(m > 0.f && m < INFINITY);  // fast scale undefined: flag
        mbar_arrive(&ex_ready[k & 1]);
        tl_mark(p, k, 1, t_begin);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issue
    if (elect_one()) {
      const uint32_t toep = smem_u32(base + p.off_toep), cen = smem_u32(base + p.off_cen);
      const uint32_t yo = smem_u32(base + p.off_yo), ye = smem_u32(base + p.off_ye);
      uint32_t g1 = 0;  // stage-1 tile sequence
      auto stage2 = [&](int k) {  // clip k's stage 2 (both tiles), after its y1 is complete
        wait_p(s2_ready, k & 1, pf[2]);
        if (k > 0) wait_p(s2_free, (k - 1) & 1, pf[3]);
        tc_fence_after();
        issue_tile(tmem + 256, yo, (uint32_t)p.pl2, ye, (uint32_t)p.pe2, 0, toep, cen);
        if (p.row_b > 0) issue_tile(tmem + 384, yo, (uint32_t)p.pl2, ye, (uint32_t)p.pe2, p.row_b, toep, cen);
        mma_commit(s2_done);
        tl_mark(p, k, 6, t_begin);
      };
      for (int k = 0; k < n_clips; ++k) {
        for (int t = 0; t < p.n1; ++t, ++g1) {
          const int slot = (int)(g1 & 1);
          wait_p(&a_full[slot], (g1 >> 1) & 1, pf[0]);
          if (g1 >= 2) wait_p(&s1_free[slot], ((g1 >> 1) - 1) & 1, pf[1]);
          tc_fence_after();
          const uint32_t a1 = smem_u32(base + p.off_a1[slot]);
          issue_tile(tmem + 128u * slot, a1, (uint32_t)p.pl1, a1 + 16u * p.pl1, (uint32_t)p.pe1, 0, toep, cen);
          mma_commit(&s1_done[slot]);
          mma_commit(&a_empty[slot]);
          if (t == 0 && k > 0) stage2(k - 1);  // the previous clip's stage 2 runs under this clip's conversion
        }
        tl_mark(p, k, 4, t_begin);
      }
      if (n_clips > 0) stage2(n_clips - 1);
    }
  } else if (warp >= kConvWarp0 && warp < kConvWarp0 + kConvWarps) {
    // ------------------------------------------------------------ converters
    // the tile's ext segment [e0, e1) as float4 f = ct + kCT u: its samples d = 4 f are
    //   odd  d + 1, d + 3 -> odd row f / 64 = ct / 64 + 4 u, odd index 2 (ct % 64) (+1)
    //   even d, d + 2     -> even row (f - 32) / 64 = (ct - 32) / 64 + 4 u, index 2 ((ct - 32) % 64)
    // so both store addresses are per-thread constants plus 64 B per u
    const int ct = tid - kConvWarp0 * 32;  // 0 .. kCT - 1
    const int uo = 2 * (ct & 63), ue = 2 * ((ct - 32) & 63);
    const int ro = ct >> 6, re = ((ct - 32 + 64) >> 6) - 1;
    const uint32_t oo = (uint32_t)((uo >> 3) * p.pl1 + (uo & 7) * 2 + ro * 16);
    const uint32_t oe = (uint32_t)(16 * p.pl1 + (ue >> 3) * p.pe1 + (ue & 7) * 2 + 16 * re);  // row re at u = 0
    const uint64_t last = policy_evict_first();  // (evict_unchanged / evict_last: no faster)
    uint32_t g1 = 0;
    for (int k = 0; k < n_clips; ++k) {
      const int64_t b = clip_of(k);
      const float* xb = p.x + b * p.L;
      wait_p(&ex_ready[k & 1], (k >> 1) & 1, pf[0]);
      const int ex = ex_slot[k & 1];
      if (ct == 0) {
        mbar_arrive(conv_start);
        p.exps[b] = ex;
        tl_mark(p, k, 2, t_begin);
      }
      const bool zero_peek = ex_slot[2 + (k & 1)] != 0;
      const float scale = ldexpf(1.f, -ex);
      float cmax = 0.f;  // the clip's peak as converted (fast-scale overflow check)
      for (int t = 0; t < p.n1; ++t, ++g1) {
        const int slot = (int)(g1 & 1);
        const int n0 = 128 * t, nb = min(128, p.nb1 - n0);
        const int e0 = 256 * n0 - 128, e1 = 256 * (n0 + nb + 1) - 128;
        const int n4 = (e1 - e0) / 4;
        if (g1 >= 2) wait_p(&a_empty[slot], ((g1 >> 1) - 1) & 1, pf[1]);  // this buffer's last MMAs are done
        const uint32_t a1 = smem_u32(base + p.off_a1[slot]);
        const float* pb = xb + e0 + 4 * ct;  // float4 u of this thread: pb + 1024 u
        for (int u0 = 0; kCT * u0 < n4; u0 += kConvBatch) {
          const uint32_t so = a1 + oo + 16u * kRowU * u0, se = a1 + oe + 16u * kRowU * u0;
          const int rl0 = re + kRowU * u0;  // even row of v[0]
          const float* q = pb + 4 * kCT * u0;  // float4 u at q + 4 kCT u (immediate offsets)
          const int fr = n4 - (ct + kCT * u0);  // float4 u of this thread is live iff kCT u < fr
          // every load of the batch inside the clip (no reflect image): predicated loads only
          const bool inside = e0 + 4 * kCT * u0 >= 0 && e0 + 4 * kCT * (u0 + kConvBatch) <= p.L;
          float4 v[kConvBatch];
          if (inside) {
#pragma unroll
#ifdef NNAB_DBG_FRONT_NOLOAD
            for (int u = 0; u < kConvBatch; ++u) v[u] = make_float4((float)u0, (float)u, 0.5f, 0.25f);
#else
            for (int u = 0; u < kConvBatch; ++u)
              v[u] = kCT * u < fr ? ldg_keep(q + 4 * kCT * u, last) : make_float4(0.f, 0.f, 0.f, 0.f);
#endif
          } else {
#pragma unroll
            for (int u = 0; u < kConvBatch; ++u) {
              const int e = e0 + 4 * (ct + kCT * (u0 + u));
              v[u] = kCT * u >= fr ? make_float4(0.f, 0.f, 0.f, 0.f)
                             : (e >= 0 && e + 4 <= p.L) ? ldg_keep(q + 4 * kCT * u, last) : edge_float4(e, e1, p.L, xb);
            }
          }
#pragma unroll
          for (int u = 0; u < kConvBatch; ++u) {
            if (kCT * u >= fr) break;
            cmax = fmaxf(cmax, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
            sts32(so + 16u * kRowU * u, pack2(v[u].y * scale, v[u].w * scale));
            if ((unsigned)(rl0 + kRowU * u) < (unsigned)nb) sts32(se + 16u * kRowU * u, pack2(v[u].x * scale, v[u].z * scale));
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[slot]);
      }
      if (ct == 0) tl_mark(p, k, 3, t_begin);
      if (!p.exact) {  // flag the clip when the fast scale left less than 2 bits below FP16's range
#pragma unroll
        for (int o = 16; o; o >>= 1) cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
        if (lane == 0) atomicMax(&conv_max[k & 1], __float_as_uint(cmax));
        named_sync(4, 32 * kConvWarps);
        if (ct == 0) {
          const float m = __uint_as_float(conv_max[k & 1]);
          // flagged: appended to the exact relaunch's list (any order: each listed clip is
          // redone on its own, so the output does not depend on it)
          if (zero_peek || !(m * scale < 16384.f)) p.out_list[atomicAdd(p.out_list_n, 1)] = (int32_t)b;
          conv_max[k & 1] = 0u;  // reused by clip k + 2, after clip k + 1's barrier
        }
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int et = tid - kEpiWarp0 * 32;  // 0..127
    uint8_t* yo = base + p.off_yo;
    uint8_t* ye = base + p.off_ye;
    const int L1 = p.L1, L0 = p.L0;
    uint32_t g1 = 0;
    auto store_yo1 = [&](int m, float v) {  // odd-phase sample m of y1 (stage-2 planes)
      if (m >= 0 && m < 128 * p.yr)
        *reinterpret_cast<__half*>(yo + ((m & 127) >> 3) * p.pl2 + (m >> 7) * 16 + (m & 7) * 2) = __float2half_rn(v);
    };
    // stage 2 of clip k: octave 0 assembled in shared memory as the clip's whole level row
    // (reflect margins, signal, zero tail; staged in the y1 even planes, which stage 2 has
    // finished reading) and written with one bulk copy
    __half* stage = reinterpret_cast<__half*>(ye);
    auto stage2_epi = [&](int k) {
      wait_p(s2_done, k & 1, pf[2]);
      if (et == 0) tl_mark(p, k, 8, t_begin);
      tc_fence_after();
      for (int tt = 0; tt < (p.row_b > 0 ? 2 : 1); ++tt) {
        const int n = (tt ? p.row_b : 0) + q * 32 + lane;
        const bool blk_ok = (tt == 0 || n >= 128) && n < p.nb2;
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + 256u + 128u * tt;
#pragma unroll 1
        for (int kp = 0; kp < 8; kp += 2) {
          float v2[32];
          const long long tq0 = clock64();
          tmem_ld32(ta + 16 * kp, v2);
          tmem_ld_wait();
          pf[3] += (unsigned long long)(clock64() - tq0);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float* v = v2 + 16 * h;
            const int i0 = 128 * n + 112 - 16 * (kp + h);
            if (!blk_ok || i0 >= L0) continue;
            float y[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) y[e] = v[15 - e];
            if (i0 + 16 <= L0) {
              *reinterpret_cast<uint4*>(stage + kML + i0) =
                  make_uint4(pack2(y[0], y[1]), pack2(y[2], y[3]), pack2(y[4], y[5]), pack2(y[6], y[7]));
              *reinterpret_cast<uint4*>(stage + kML + i0 + 8) =
                  make_uint4(pack2(y[8], y[9]), pack2(y[10], y[11]), pack2(y[12], y[13]), pack2(y[14], y[15]));
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (i0 + e < L0) stage[kML + i0 + e] = __float2half_rn(y[e]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s2_free);
      for (int jz = L0 + 2 * kML + et; jz < p.lv0_stride; jz += 128) stage[jz] = __float2half_rn(0.f);  // zero tail
      named_sync(3, 128);
      // reflect images of the level (np.pad "reflect", signal.py:245), two per thread:
      // left ML - i = sample i (1 <= i <= ML), right ML + 2 (L0 - 1) - i (L0 - 1 - ML <= i <= L0 - 2)
      for (int r = et; r < 2 * kML; r += 128) {
        const int i = r < kML ? r + 1 : L0 - 1 - kML + (r - kML);
        stage[r < kML ? kML - i : kML + 2 * (L0 - 1) - i] = stage[kML + i];
      }
      fence_proxy_async_smem();
      const long long tq1 = clock64();
      named_sync(3, 128);
      pf[1] += (unsigned long long)(clock64() - tq1);
      if (et == 0) {
        bulk_store(p.lv0 + clip_of(k) * (int64_t)p.lv0_stride, stage, (uint32_t)p.lv0_stride * 2u);
        tl_mark(p, k, 7, t_begin);
      }
    };
    auto stage_reusable = [&]() {  // the bulk store has read the staged row
      if (et == 0) bulk_wait_read();
      named_sync(3, 128);
    };
    for (int k = 0; k < n_clips; ++k) {
      for (int t = 0; t < p.n1; ++t, ++g1) {
        const int slot = (int)(g1 & 1);
        if (t == 0 && k > 0) {  // clip k-1's stage 2 first: it frees the y1 planes this tile writes
          stage2_epi(k - 1);
          stage_reusable();
        }
        wait_p(&s1_done[slot], (g1 >> 1) & 1, pf[0]);
        if (et == 0 && t == 0) tl_mark(p, k, 9, t_begin);
        tc_fence_after();
        const int n = 128 * t + q * 32 + lane;  // block
        const bool blk_ok = q * 32 + lane < min(128, p.nb1 - 128 * t);
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + 128u * slot;
#pragma unroll 1
        for (int kp = 0; kp < 8; kp += 2) {
          float v2[32];
          tmem_ld32(ta + 16 * kp, v2);
          tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
          const int kk = kp + h;
          const float* v = v2 + 16 * h;
          const int i0 = 128 * n + 112 - 16 * kk;  // outputs i0 .. i0 + 15 of y1
          if (!blk_ok || i0 >= L1) continue;
          float y[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) y[e] = v[15 - e];
          if (i0 + 16 <= L1) {
            const int m0 = (i0 >> 1) + 64;  // odd outputs -> yo[m0 .. m0 + 7]
            *reinterpret_cast<uint4*>(yo + ((m0 & 127) >> 3) * p.pl2 + (m0 >> 7) * 16) =
                make_uint4(pack2(y[1], y[3]), pack2(y[5], y[7]), pack2(y[9], y[11]), pack2(y[13], y[15]));
            const int u0 = i0 >> 1;  // even outputs -> ye[u0 .. u0 + 7]
            *reinterpret_cast<uint4*>(ye + ((u0 & 127) >> 3) * p.pe2 + (u0 >> 7) * 16) =
                make_uint4(pack2(y[0], y[2]), pack2(y[4], y[6]), pack2(y[8], y[10]), pack2(y[12], y[14]));
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int i = i0 + e;
              if (i >= L1) break;
              if (i & 1) {
                store_yo1((i + 127) >> 1, y[e]);
              } else {
                const int u = i >> 1;
                *reinterpret_cast<__half*>(ye + ((u & 127) >> 3) * p.pe2 + (u >> 7) * 16 + (u & 7) * 2) =
                    __float2half_rn(y[e]);
              }
            }
          }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s1_free[slot]);
      }
      // y1's odd-phase reflect images (left: -i, right: 2 (L1 - 1) - i, i odd), then stage 2 may run
      if (et == 0) tl_mark(p, k, 10, t_begin);
      named_sync(2, 128);
      if (et == 0) tl_mark(p, k, 11, t_begin);
      {
        const int e = et;
        const int i = e < 64 ? 2 * e + 1 : ((L1 - 128) | 1) + 2 * (e - 64);
        const int dst = e < 64 ? -i : 2 * (L1 - 1) - i;
        if (i <= L1 - 2) {
          const int ms = (i + 127) >> 1;
          const __half v = *reinterpret_cast<const __half*>(yo + ((ms & 127) >> 3) * p.pl2 + (ms >> 7) * 16 + (ms & 7) * 2);
          store_yo1((dst + 127) >> 1, __half2float(v));
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(s2_ready);
      if (et == 0) tl_mark(p, k, 5, t_begin);
    }
    if (n_clips > 0) stage2_epi(n_clips - 1);
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the last row is written
  }
  if (p.prof) {  // role leaders: [4 role slots] x 5 roles + total
    const int role = warp == kScanWarp0 ? 0 : warp == kMmaWarp ? 2 : warp >= kConvWarp0 ? 3 : 4;
    const bool lead = tid == kScanWarp0 * 32 || tid == kMmaWarp * 32 || tid == kConvWarp0 * 32 || tid == kEpiWarp0 * 32;
    if ((lead || role == 2) && (pf[0] | pf[1] | pf[2] | pf[3]))
      for (int i = 0; i < 4; ++i) atomicAdd(p.prof + 4 * role + i, pf[i]);
    if (tid == 0) atomicAdd(p.prof + 20, (unsigned long long)(clock64() - t_begin));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

__device__ unsigned long long g_front_prof[24];
bool g_front_prof_on = false;

// the flagged clips' indices (order irrelevant: clips are independent) and their count
}  // namespace

// Shared-memory plan + launches; NNAB_ENOTSUP outside the kernel's envelope (the caller
// then runs the fused kernel's front-only mode).  Fast launch (scale from the first kPeek
// samples) over every clip, then the flagged clips (zero / too quiet start, a later peak
// beyond the headroom) again with the exact whole-clip scale.  flags / list: B ints each,
// list_n: one int, in the caller's workspace.
int launch_cqt2010_front(const float* x, int64_t B, int64_t L, const float* taps, int n_taps, __half* lv0,
                         int32_t lv0_stride, int32_t* exps, int32_t* flags, int32_t* list, int32_t* list_n,
                         cudaStream_t st, const CqtPrepArgs* prep) {
  if (n_taps != 255 || L % 4 != 0 || L < 1024 || L > (1 << 24) || !flags || !list || !list_n) return NNAB_ENOTSUP;
  FrontParams p{};

  p.x = x;
  p.B = B;
  p.L = (int32_t)L;
  p.L1 = (int32_t)((L + 1) / 2);
  p.L0 = (p.L1 + 1) / 2;
  p.nb1 = (p.L1 + 127) / 128;
  p.n1 = (p.nb1 + 127) / 128;
  p.nb2 = (p.L0 + 127) / 128;
  if (p.nb2 > 256 || p.L0 + 2 * kML > lv0_stride) return NNAB_ENOTSUP;
  p.row_b = p.nb2 > 128 ? p.nb2 - 128 : 0;
  p.yr = (std::max(std::max(p.nb2 + 1, (p.L1 + 253) / 2 / 128 + 1), p.row_b + 129) + 7) / 8 * 8;
  p.pl1 = 130 * 16 + 16;  // +16 B: consecutive planes start in different banks
  p.pe1 = 128 * 16 + 16;
  p.pl2 = p.yr * 16 + 16;
  p.pe2 = p.yr * 16 + 16;
  int off = 0;
  auto take = [&](int bytes, int align) {
    off = (off + align - 1) / align * align;
    const int o = off;
    off += bytes;
    return o;
  };
  p.off_toep = take(kToepChunks * 16, 1024);
  p.off_cen = take(kCenChunks * 16, 128);
  p.off_a1[0] = take(16 * (p.pl1 + p.pe1), 128);
  p.off_a1[1] = take(16 * (p.pl1 + p.pe1), 128);
  p.off_yo = take(16 * p.pl2, 128);  // yr >= the 129 rows an M = 128 tile reads
  p.off_ye = take(16 * p.pe2, 128);
  p.off_bars = take(256, 128);
  const size_t smem = 1024 + (size_t)off;
  if (smem > 227 * 1024 || 16 * p.pe2 < 2 * lv0_stride) return NNAB_ENOTSUP;
  p.h0 = taps[127];
  for (int j = 0; j < 128; ++j) p.g[j] = taps[2 * j];
  p.lv0 = lv0;
  p.lv0_stride = lv0_stride;
  p.exps = exps;
  p.prof = nullptr;
  if (g_front_prof_on) {
    void* ptr = nullptr;
    NNAB_CUDA_TRY(cudaGetSymbolAddress(&ptr, g_front_prof));
    p.prof = reinterpret_cast<unsigned long long*>(ptr);
  }
  NNAB_CUDA_TRY(cudaFuncSetAttribute(cqt2010_front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>(B, (int64_t)num_sms());
  (void)flags;
  NNAB_CUDA_TRY(cudaMemsetAsync(list_n, 0, 4, st));
  p.exact = 0;
  if (prep) p.prep = *prep;
  p.out_list = list;
  p.out_list_n = list_n;
  cqt2010_front_kernel<<<grid, kThreads, smem, st>>>(p);
  NNAB_LAUNCHED();
  p.exact = 1;
  p.prep = CqtPrepArgs{};
  p.out_list = nullptr;
  p.out_list_n = nullptr;
  p.list = list;
  p.list_n = list_n;
  p.prof = nullptr;
  cqt2010_front_kernel<<<grid, kThreads, smem, st>>>(p);
  NNAB_LAUNCHED();
  return NNAB_OK;
}

}  // namespace nnab

// Debug: per-role wait cycles of the CQT2010v2 front (on != 0 clears and enables; on == 0
// copies [24] out and disables): role r at 4 r .. 4 r + 3 (scan: conv_start; loader:
// -; MMA: a_full, s1_free, s2_ready, s2_free; converter: ex_ready, a_empty, -; epilogue: s1_done, s2_done (stage 1), s2_done (stage 2)), [20] elapsed.
extern "C" int nnab_debug_cqt2010_front_profile(int on, unsigned long long* out) {
  using nnab::cuda_fail;
  if (on) {
    nnab::g_front_prof_on = true;
    unsigned long long z[24] = {};
    NNAB_CUDA_TRY(cudaMemcpyToSymbol(nnab::g_front_prof, z, sizeof(z)));
    return NNAB_OK;
  }
  nnab::g_front_prof_on = false;
  if (out) NNAB_CUDA_TRY(cudaMemcpyFromSymbol(out, nnab::g_front_prof, 24 * sizeof(unsigned long long)));
  return NNAB_OK;
}

extern "C" int nnab_debug_cqt2010_front_timeline(long long* out) {
  using nnab::cuda_fail;
  NNAB_CUDA_TRY(cudaMemcpyFromSymbol(out, nnab::g_front_tl, 16 * 12 * sizeof(long long)));
  return NNAB_OK;
}
