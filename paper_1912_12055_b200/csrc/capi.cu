// extern "C" boundary of libnnab plus host-side helpers (tensor maps, errors).
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace nnab {

static thread_local char g_last_error[256] = "";
static std::atomic<uint64_t> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int cuda_fail(cudaError_t e, const char* where) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
  return NNAB_ECUDA;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                 uint32_t box_inner, uint32_t box_outer, int swizzle_bytes, int elem_bytes) {
  auto enc = get_encode();
  if (!enc) {
    std::snprintf(g_last_error, sizeof(g_last_error), "cuTensorMapEncodeTiled unavailable");
    return NNAB_ECUDA;
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0 || row_bytes % 16 != 0) return NNAB_EINVAL;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  // -128: 32-byte atoms swizzled within 128 B (the MN-major TF32 UMMA layout)
  CUtensorMapSwizzle sw = swizzle_bytes == -128 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                          : swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(map, elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::snprintf(g_last_error, sizeof(g_last_error), "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return NNAB_ECUDA;
  }
  return NNAB_OK;
}

// Per-device attribute caches: the current device is read on every call, so a
// process driving several GPUs (one host thread each) gets each one's own values.
constexpr int kMaxDevices = 64;

int num_sms() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t stage_bytes(const FrameGeom& g) { return align256((size_t)g.B * g.R * g.row_len * sizeof(float)); }

// Staged-frames workspace: [hi rows][lo rows (split modes)][per-clip scale exponents (FP16 modes)];
// rows are fp32 (TF32 modes) or FP16, laid out with the precision's K alignment.
struct StageLayout {
  FrameGeom g;
  size_t half_bytes = 0, lo_off = 0, exp_off = 0, total = 0;
};
static int stage_layout(const nnab_frames* f, int32_t precision, StageLayout* s) {
  if (!prec_valid(precision)) return NNAB_EINVAL;
  int rc = frame_geometry(f, &s->g, prec_kalign(precision));
  if (rc) return rc;
  const size_t elem = prec_is_f16(precision) ? 2 : 4;
  s->half_bytes = align256((size_t)s->g.B * s->g.R * s->g.row_len * elem);
  s->lo_off = s->half_bytes;
  s->exp_off = s->half_bytes * (prec_is_split(precision) ? 2 : 1);
  s->total = s->exp_off + (prec_is_f16(precision) ? align256((size_t)s->g.B * 4) : 0);
  return NNAB_OK;
}

static int check_device() {
  static std::atomic<int> cache[kMaxDevices];  // 0 unknown, 1 sm_100, 2 other / error
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return NNAB_ENODEV;
  int v = dev < kMaxDevices ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (v == 0) {
    int major = 0;
    v = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess && major == 10 ? 1 : 2;
    if (dev < kMaxDevices) cache[dev].store(v, std::memory_order_relaxed);
  }
  return v == 1 ? NNAB_OK : NNAB_ENODEV;
}

}  // namespace nnab

using namespace nnab;

extern "C" int nnab_version(void) { return 1; }

extern "C" const char* nnab_strerror(int code) {
  switch (code) {
    case NNAB_OK: return "ok";
    case NNAB_EINVAL: return "invalid argument";
    case NNAB_ECUDA: return "CUDA error";
    case NNAB_ENOTSUP: return "configuration not supported by the sm_100a kernels";
    case NNAB_ENODEV: return "no sm_100 (B200) device";
    default: return "unknown nnab status";
  }
}

extern "C" const char* nnab_last_error(void) { return g_last_error; }

extern "C" uint64_t nnab_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int nnab::staged_views(const nnab_frames* f, int32_t precision, const void* workspace, size_t workspace_bytes,
                 FrameGeom* g, const void** hi, const void** lo, const int32_t** exps) {
  StageLayout sl;
  int rc = stage_layout(f, precision, &sl);
  if (rc) return rc;
  *g = sl.g;
  if (sl.g.B > 0 && (!workspace || workspace_bytes < sl.total)) return NNAB_EINVAL;
  const char* w = reinterpret_cast<const char*>(workspace);
  *hi = w;
  *lo = prec_is_split(precision) ? w + sl.lo_off : nullptr;
  *exps = prec_is_f16(precision) ? reinterpret_cast<const int32_t*>(w + sl.exp_off) : nullptr;
  return NNAB_OK;
}

extern "C" size_t nnab_stft_workspace_bytes(const nnab_frames* f, int32_t precision) {
  StageLayout sl;
  if (stage_layout(f, precision, &sl)) return 0;
  return sl.total;
}

static int validate_kind(int32_t out_kind, int32_t n_bins, const float* mel_w, int32_t n_mels, int32_t mel_ld,
                         int32_t n_tiles) {
  if (out_kind & NNAB_OUT_LOG) {
    out_kind &= ~NNAB_OUT_LOG;
    if (out_kind != NNAB_OUT_MAGNITUDE && out_kind != NNAB_OUT_POWER && out_kind != NNAB_OUT_MEL) return NNAB_EINVAL;
  }
  if (out_kind < NNAB_OUT_MAGNITUDE || out_kind > NNAB_OUT_SMOOTH_MAG) return NNAB_EINVAL;
  if (out_kind == NNAB_OUT_MEL) {
    if (!mel_w || n_mels < 1) return NNAB_EINVAL;
    if (mel_ld < std::max(n_tiles * 128, n_bins)) return NNAB_EINVAL;
  }
  return NNAB_OK;
}

extern "C" int nnab_stft_forward(const nnab_frames* f, const float* x, const float* packed_hi,
                                 const float* packed_lo, int32_t n_bins, int32_t fold_nyquist, int32_t precision,
                                 int32_t out_kind, float power, float eps, const float* mel_w, int32_t n_mels,
                                 int32_t mel_ld, const int32_t* mel_band, float* out, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  int rc = check_device();
  if (rc) return rc;
  FrameGeom g;
  if ((rc = frame_geometry(f, &g))) return rc;
  if (!prec_valid(precision)) return NNAB_EINVAL;
  const int split = prec_is_split(precision);
  if (!x || !packed_hi || (split && !packed_lo) || !out || n_bins < 1) return NNAB_EINVAL;
  if (fold_nyquist && n_bins < 2) return NNAB_EINVAL;
  const int32_t tiles = nnab_dft_bank_tiles(n_bins, fold_nyquist);
  if ((rc = validate_kind(out_kind, n_bins, mel_w, n_mels, mel_ld, tiles))) return rc;
  if (g.B == 0) return NNAB_OK;
  if ((rc = nnab_stage_frames(f, x, precision, workspace, workspace_bytes, stream))) return rc;
  return nnab_stft_forward_staged(f, packed_hi, packed_lo, n_bins, fold_nyquist, precision, out_kind, power, eps,
                                  mel_w, n_mels, mel_ld, mel_band, out, workspace, workspace_bytes, stream);
}

extern "C" int nnab_stage_frames(const nnab_frames* f, const float* x, int32_t precision, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  int rc = check_device();
  if (rc) return rc;
  StageLayout sl;
  if ((rc = stage_layout(f, precision, &sl))) return rc;
  const FrameGeom& g = sl.g;
  if (g.B == 0) return NNAB_OK;
  if (!x || !workspace || workspace_bytes < sl.total) return NNAB_EINVAL;
  const int split = prec_is_split(precision);
  char* w = reinterpret_cast<char*>(workspace);
  if (prec_is_f16(precision))
    return stage_frames_f16(g, x, w, split ? w + sl.lo_off : nullptr, reinterpret_cast<int32_t*>(w + sl.exp_off),
                            split, (cudaStream_t)stream);
  return stage_frames(g, x, reinterpret_cast<float*>(w), split ? reinterpret_cast<float*>(w + sl.lo_off) : nullptr,
                      split, (cudaStream_t)stream);
}

extern "C" int nnab_stft_forward_staged(const nnab_frames* f, const float* packed_hi, const float* packed_lo,
                                        int32_t n_bins, int32_t fold_nyquist, int32_t precision, int32_t out_kind,
                                        float power, float eps, const float* mel_w, int32_t n_mels, int32_t mel_ld,
                                        const int32_t* mel_band, float* out, const void* workspace,
                                        size_t workspace_bytes, void* stream) {
  int rc = check_device();
  if (rc) return rc;
  StageLayout sl;
  if ((rc = stage_layout(f, precision, &sl))) return rc;
  const FrameGeom& g = sl.g;
  const int split = prec_is_split(precision);
  if (!packed_hi || (split && !packed_lo) || !out || n_bins < 1) return NNAB_EINVAL;
  if (fold_nyquist && n_bins < 2) return NNAB_EINVAL;
  const int32_t tiles = nnab_dft_bank_tiles(n_bins, fold_nyquist);
  if ((rc = validate_kind(out_kind, n_bins, mel_w, n_mels, mel_ld, tiles))) return rc;
  if (g.B == 0) return NNAB_OK;
  if (!workspace || workspace_bytes < sl.total) return NNAB_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const char* w = reinterpret_cast<const char*>(workspace);
  StftGemmArgs a{};
  a.a_hi = reinterpret_cast<const float*>(w);
  a.a_lo = split ? reinterpret_cast<const float*>(w + sl.lo_off) : nullptr;
  if (prec_is_f16(precision)) {
    a.a_exp = reinterpret_cast<const int32_t*>(w + sl.exp_off);
    a.b_exp = reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(packed_hi) +
                                               nnab_dft_bank_bytes_prec(n_bins, g.width, fold_nyquist, precision) -
                                               256) + 1;
  }
  a.b_hi = packed_hi;
  a.b_lo = packed_lo;
  a.n_tiles = tiles;
  a.n_bins = n_bins;
  a.fold = fold_nyquist ? 1 : 0;
  a.out_kind = out_kind;
  a.power = power;
  a.eps = eps;
  a.mel_w = mel_w;
  a.n_mels = n_mels;
  a.mel_ld = mel_ld;
  a.mel_band = mel_band;
  a.out = out;
  return launch_stft_gemm(g, a, precision, s);
}

// ------------------------------------------------------------ host variant
static size_t pipeline_bytes(int64_t chunk, int64_t L, int64_t out_per_clip) {
  return 2 * (align256((size_t)chunk * L * 4) + align256((size_t)chunk * out_per_clip * 4));
}

static int64_t out_elems_per_clip(int32_t out_kind, int32_t n_bins, int32_t n_mels, int32_t T) {
  out_kind &= ~NNAB_OUT_LOG;
  if (out_kind == NNAB_OUT_MEL) return (int64_t)n_mels * T;
  if (out_kind == NNAB_OUT_COMPLEX) return 2ll * n_bins * T;
  return (int64_t)n_bins * T;
}

extern "C" size_t nnab_stft_host_scratch_bytes(const nnab_frames* f, int32_t precision, int32_t out_rows,
                                               int64_t chunk_clips) {
  FrameGeom g;
  if (frame_geometry(f, &g) || chunk_clips < 1) return 0;
  nnab_frames fc = *f;
  fc.batch = std::min<int64_t>(chunk_clips, f->batch);
  return pipeline_bytes(fc.batch, g.L, (int64_t)out_rows * g.T) + nnab_stft_workspace_bytes(&fc, precision);
}

// Three-stage software pipeline over clip chunks shared by the host-buffer entry
// points: copy-in on `cin`, compute(x_dev, n_clips, out_dev) on the caller's
// stream, copy-out on `cout`; events order the hand-offs, two slots each.
// Streams and events of one host_pipeline call, released on every return path.
struct PipelineRes {
  cudaStream_t cin = nullptr, cout = nullptr;
  cudaEvent_t start = nullptr, in_done[2] = {}, comp_done[2] = {}, out_done[2] = {};
  ~PipelineRes() {
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
    cudaEvent_t* all[] = {&start, &in_done[0], &in_done[1], &comp_done[0], &comp_done[1], &out_done[0], &out_done[1]};
    for (cudaEvent_t* e : all)
      if (*e) cudaEventDestroy(*e);
  }
  int create() {
    NNAB_CUDA_TRY(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking));
    NNAB_CUDA_TRY(cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking));
    NNAB_CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      NNAB_CUDA_TRY(cudaEventCreateWithFlags(&in_done[i], cudaEventDisableTiming));
      NNAB_CUDA_TRY(cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming));
      NNAB_CUDA_TRY(cudaEventCreateWithFlags(&out_done[i], cudaEventDisableTiming));
    }
    return NNAB_OK;
  }
};

// Three-stage software pipeline over clip chunks shared by the host-buffer entry
// points: copy-in on `cin`, compute(x_dev, n_clips, out_dev) on the caller's
// stream, copy-out on `cout`; events order the hand-offs, two slots each.
// (Stream destruction is deferred by the driver until queued work completes.)
template <class Compute>
static int host_pipeline(int64_t B, int64_t L, int64_t out_per_clip, int64_t chunk, const float* x_host,
                         float* out_host, char* base, cudaStream_t s, Compute compute) {
  const size_t xin = align256((size_t)chunk * L * 4);
  const size_t ob = align256((size_t)chunk * out_per_clip * 4);
  float* xd[2] = {reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + xin)};
  float* od[2] = {reinterpret_cast<float*>(base + 2 * xin), reinterpret_cast<float*>(base + 2 * xin + ob)};
  PipelineRes r;
  int rc = r.create();
  if (rc) return rc;
  NNAB_CUDA_TRY(cudaEventRecord(r.start, s));
  NNAB_CUDA_TRY(cudaStreamWaitEvent(r.cin, r.start, 0));
  NNAB_CUDA_TRY(cudaStreamWaitEvent(r.cout, r.start, 0));
  const int64_t n_chunks = (B + chunk - 1) / chunk;
  for (int64_t i = 0; i < n_chunks && rc == NNAB_OK; ++i) {
    const int slot = (int)(i & 1);
    const int64_t c0 = i * chunk;
    const int64_t nb = std::min<int64_t>(chunk, B - c0);
    if (i >= 2) NNAB_CUDA_TRY(cudaStreamWaitEvent(r.cin, r.comp_done[slot], 0));  // x slot free
    NNAB_CUDA_TRY(cudaMemcpyAsync(xd[slot], x_host + c0 * L, (size_t)nb * L * 4, cudaMemcpyHostToDevice, r.cin));
    NNAB_CUDA_TRY(cudaEventRecord(r.in_done[slot], r.cin));
    NNAB_CUDA_TRY(cudaStreamWaitEvent(s, r.in_done[slot], 0));
    if (i >= 2) NNAB_CUDA_TRY(cudaStreamWaitEvent(s, r.out_done[slot], 0));  // out slot drained
    rc = compute(xd[slot], nb, od[slot]);
    NNAB_CUDA_TRY(cudaEventRecord(r.comp_done[slot], s));
    NNAB_CUDA_TRY(cudaStreamWaitEvent(r.cout, r.comp_done[slot], 0));
    NNAB_CUDA_TRY(cudaMemcpyAsync(out_host + c0 * out_per_clip, od[slot], (size_t)nb * out_per_clip * 4,
                                  cudaMemcpyDeviceToHost, r.cout));
    NNAB_CUDA_TRY(cudaEventRecord(r.out_done[slot], r.cout));
  }
  // join: the caller's stream waits for the last copy-out (also after a failed compute,
  // so no copy still reads the caller's buffers when this returns)
  NNAB_CUDA_TRY(cudaEventRecord(r.out_done[0], r.cout));
  NNAB_CUDA_TRY(cudaStreamWaitEvent(s, r.out_done[0], 0));
  return rc;
}

extern "C" int nnab_stft_forward_host(const nnab_frames* f, const float* x_host, const float* packed_hi,
                                      const float* packed_lo, int32_t n_bins, int32_t fold_nyquist,
                                      int32_t precision, int32_t out_kind, float power, float eps,
                                      const float* mel_w, int32_t n_mels, int32_t mel_ld, const int32_t* mel_band,
                                      float* out_host, int64_t chunk_clips, void* device_scratch,
                                      size_t scratch_bytes, void* stream) {
  int rc = check_device();
  if (rc) return rc;
  FrameGeom g;
  if ((rc = frame_geometry(f, &g))) return rc;
  if (!x_host || !out_host || chunk_clips < 1) return NNAB_EINVAL;
  if (g.B == 0) return NNAB_OK;
  const int64_t per_clip_out = out_elems_per_clip(out_kind, n_bins, n_mels, g.T);
  const int32_t out_rows = (int32_t)(per_clip_out / g.T);
  const int64_t chunk = std::min<int64_t>(chunk_clips, g.B);
  if (!device_scratch || scratch_bytes < nnab_stft_host_scratch_bytes(f, precision, out_rows, chunk))
    return NNAB_EINVAL;
  nnab_frames fc = *f;
  fc.batch = chunk;
  char* base = reinterpret_cast<char*>(device_scratch);
  void* ws = base + pipeline_bytes(chunk, g.L, per_clip_out);
  const size_t ws_bytes = nnab_stft_workspace_bytes(&fc, precision);
  return host_pipeline(g.B, g.L, per_clip_out, chunk, x_host, out_host, base, (cudaStream_t)stream,
                       [&](const float* xd, int64_t nb, float* od) {
                         fc.batch = nb;
                         return nnab_stft_forward(&fc, xd, packed_hi, packed_lo, n_bins, fold_nyquist, precision,
                                                  out_kind, power, eps, mel_w, n_mels, mel_ld, mel_band, od, ws,
                                                  ws_bytes, stream);
                       });
}

extern "C" size_t nnab_cqt1992v2_host_scratch_bytes(const nnab_frames* f, int32_t precision, int32_t n_bins,
                                                    int32_t out_kind, int64_t chunk_clips) {
  FrameGeom g;
  if (frame_geometry(f, &g) || chunk_clips < 1) return 0;
  nnab_frames fc = *f;
  fc.batch = std::min<int64_t>(chunk_clips, f->batch);
  const int64_t per = (out_kind == NNAB_OUT_COMPLEX ? 2ll : 1ll) * n_bins * g.T;
  return pipeline_bytes(fc.batch, g.L, per) + nnab_stft_workspace_bytes(&fc, precision);
}

extern "C" int nnab_cqt1992v2_forward_host(const nnab_frames* f, const float* x_host, const float* packed_hi,
                                           const float* packed_lo, int32_t n_bins, const uint32_t* schedule,
                                           int32_t n_entries, int32_t precision, int32_t out_kind, float eps,
                                           float* out_host, int64_t chunk_clips, void* device_scratch,
                                           size_t scratch_bytes, void* stream) {
  int rc = check_device();
  if (rc) return rc;
  FrameGeom g;
  if ((rc = frame_geometry(f, &g))) return rc;
  if (!x_host || !out_host || chunk_clips < 1) return NNAB_EINVAL;
  if (g.B == 0) return NNAB_OK;
  const int64_t chunk = std::min<int64_t>(chunk_clips, g.B);
  if (!device_scratch || scratch_bytes < nnab_cqt1992v2_host_scratch_bytes(f, precision, n_bins, out_kind, chunk))
    return NNAB_EINVAL;
  const int64_t per = (out_kind == NNAB_OUT_COMPLEX ? 2ll : 1ll) * n_bins * g.T;
  nnab_frames fc = *f;
  fc.batch = chunk;
  char* base = reinterpret_cast<char*>(device_scratch);
  void* ws = base + pipeline_bytes(chunk, g.L, per);
  const size_t ws_bytes = nnab_stft_workspace_bytes(&fc, precision);
  return host_pipeline(g.B, g.L, per, chunk, x_host, out_host, base, (cudaStream_t)stream,
                       [&](const float* xd, int64_t nb, float* od) {
                         fc.batch = nb;
                         return nnab_cqt1992v2_forward(&fc, xd, packed_hi, packed_lo, n_bins, schedule, n_entries,
                                                       precision, out_kind, eps, od, ws, ws_bytes, stream);
                       });
}

// Hybrid CQT1992v2 (nnab_cqt1992v2_hybrid_staged) streamed from pinned host
// memory; scratch as nnab_cqt1992v2_host_scratch_bytes(f, precision, n_bins, ...).
extern "C" int nnab_cqt1992v2_hybrid_forward_host(const nnab_frames* f, const float* x_host, const float* eg_bank,
                                                  const float* eg_bank_lo, const uint16_t* col_table,
                                                  const int32_t* group_rows, int32_t n_groups, int32_t r_max,
                                                  const float* sched_bank, const float* sched_bank_lo,
                                                  const uint32_t* schedule, int32_t n_entries, int32_t n_long,
                                                  int32_t n_bins, int32_t precision, int32_t out_kind, float eps,
                                                  float* out_host, int64_t chunk_clips, void* device_scratch,
                                                  size_t scratch_bytes, void* stream) {
  int rc = check_device();
  if (rc) return rc;
  FrameGeom g;
  if ((rc = frame_geometry(f, &g))) return rc;
  if (!x_host || !out_host || chunk_clips < 1) return NNAB_EINVAL;
  if (g.B == 0) return NNAB_OK;
  const int64_t chunk = std::min<int64_t>(chunk_clips, g.B);
  if (!device_scratch || scratch_bytes < nnab_cqt1992v2_host_scratch_bytes(f, precision, n_bins, out_kind, chunk))
    return NNAB_EINVAL;
  const int64_t per = (out_kind == NNAB_OUT_COMPLEX ? 2ll : 1ll) * n_bins * g.T;
  nnab_frames fc = *f;
  fc.batch = chunk;
  char* base = reinterpret_cast<char*>(device_scratch);
  void* ws = base + pipeline_bytes(chunk, g.L, per);
  const size_t ws_bytes = nnab_stft_workspace_bytes(&fc, precision);
  return host_pipeline(g.B, g.L, per, chunk, x_host, out_host, base, (cudaStream_t)stream,
                       [&](const float* xd, int64_t nb, float* od) {
                         fc.batch = nb;
                         return nnab_cqt1992v2_hybrid_forward(&fc, xd, eg_bank, eg_bank_lo, col_table, group_rows,
                                                              n_groups, r_max, sched_bank, sched_bank_lo, schedule,
                                                              n_entries, n_long, n_bins, precision, out_kind, eps, od,
                                                              ws, ws_bytes, stream);
                       });
}

extern "C" size_t nnab_cqt2010v2_host_scratch_bytes(int64_t L, int32_t early_stages, int32_t n_bins, int32_t T,
                                                    int32_t out_kind, int64_t chunk_clips) {
  if (chunk_clips < 1 || L < 1) return 0;
  const int64_t per = (out_kind == NNAB_OUT_COMPLEX ? 2ll : 1ll) * n_bins * T;
  return pipeline_bytes(chunk_clips, L, per) + nnab_cqt2010v2_workspace_bytes(chunk_clips, L, early_stages);
}

extern "C" int nnab_cqt2010v2_forward_host(const float* x_host, int64_t B, int64_t L, const float* taps,
                                           int32_t n_taps, const float* k_re, const float* k_im, int32_t n_filters,
                                           int32_t width, int32_t early_stages, int32_t n_octaves,
                                           int32_t kernel_hop, int32_t first_bin, int32_t bins_per_octave,
                                           int32_t n_bins, int32_t pad_mode, int32_t out_kind, int32_t precision,
                                           float* out_host, int64_t chunk_clips, void* device_scratch,
                                           size_t scratch_bytes, void* stream) {
  int rc = check_device();
  if (rc) return rc;
  if (!x_host || !out_host || chunk_clips < 1 || B < 0) return NNAB_EINVAL;
  int32_t T = 0;  // validate the configuration and get the frame count (B = 0: no launch)
  float dummy = 0.f;
  if ((rc = nnab_cqt2010v2_forward(&dummy, 0, L, taps, n_taps, k_re, k_im, n_filters, width, early_stages,
                                   n_octaves, kernel_hop, first_bin, bins_per_octave, n_bins, pad_mode, out_kind,
                                   precision, &dummy, &T, nullptr, 0, stream)))
    return rc;
  if (B == 0) return NNAB_OK;
  const int64_t chunk = std::min<int64_t>(chunk_clips, B);
  if (!device_scratch || scratch_bytes < nnab_cqt2010v2_host_scratch_bytes(L, early_stages, n_bins, T, out_kind, chunk))
    return NNAB_EINVAL;
  const int64_t per = (out_kind == NNAB_OUT_COMPLEX ? 2ll : 1ll) * n_bins * T;
  char* base = reinterpret_cast<char*>(device_scratch);
  void* ws = base + pipeline_bytes(chunk, L, per);
  const size_t ws_bytes = nnab_cqt2010v2_workspace_bytes(chunk, L, early_stages);
  return host_pipeline(B, L, per, chunk, x_host, out_host, base, (cudaStream_t)stream,
                       [&](const float* xd, int64_t nb, float* od) {
                         return nnab_cqt2010v2_forward(xd, nb, L, taps, n_taps, k_re, k_im, n_filters, width,
                                                       early_stages, n_octaves, kernel_hop, first_bin,
                                                       bins_per_octave, n_bins, pad_mode, out_kind, precision, od,
                                                       nullptr, ws, ws_bytes, stream);
                       });
}
