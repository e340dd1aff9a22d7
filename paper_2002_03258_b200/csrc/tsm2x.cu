// libtsm2x.so — C ABI (include/tsm2x.h), validation, kernel dispatch, workspace management and
// the pipelined host-buffer path. Kernels live in the *.cuh files next to this one.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <pthread.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tsm2x.h"
#include "ablation.cuh"
#include "common.cuh"
#include "tsm2l.cuh"
#include "tsm2l_splitn.cuh"
#include "tsm2r_stream.cuh"
#include "tsm2r_tma.cuh"
#include "tsm2r_tma_static.cuh"
#include "tsm2r_tc32.cuh"

namespace tsm2x {

// ------------------------------------------------------------------------------------------
// errors
static thread_local std::string t_err;
static thread_local cudaEvent_t t_ev_start = nullptr, t_ev_stop = nullptr;
static std::atomic<int64_t> g_launches{0};

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}
#define TSM2X_CUDA(expr)                                                                          \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess) return fail(TSM2X_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)
#define TSM2X_TRY(expr)        \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != TSM2X_OK) return rc_; \
  } while (0)

// Kernel-timing events (tsm2x_set_kernel_events): inside a stream capture they become external
// event-record nodes, so every replay of the graph records them and they stay timeable.
static cudaError_t record_kernel_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t err = cudaStreamIsCapturing(s, &cs);
  if (err != cudaSuccess) return err;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                             : cudaEventRecord(e, s);
}

static int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TSM2X_ECUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
  return TSM2X_OK;
}

// ------------------------------------------------------------------------------------------
// validation — the reference's ValueError conditions, in the reference's order:
//   dims positive (core.py:94-95 via Matrix), _check_dims (kernels.py:36-44),
//   KernelParams.__post_init__ (core.py:176-181), validate_for (core.py:183-190).
static int validate(int variant, int precision, int64_t m, int64_t k, int64_t n, const tsm2x_params* p) {
  if (variant < TSM2X_V0 || variant > TSM2X_L_OPT2) return fail(TSM2X_EINVAL, "unknown kernel variant %d", variant);
  if (precision != TSM2X_SINGLE && precision != TSM2X_DOUBLE)
    return fail(TSM2X_EINVAL, "unknown precision %d; expected 0 (single) or 1 (double)", precision);
  if (m < 1 || k < 1 || n < 1)
    return fail(TSM2X_EINVAL, "matrix dimensions must be positive, got m=%lld k=%lld n=%lld", (long long)m,
                (long long)k, (long long)n);
  if (!p) return fail(TSM2X_EINVAL, "params must not be NULL");
  const char* names[4] = {"t1", "t2", "t3", "tcf"};
  const int32_t vals[4] = {p->t1, p->t2, p->t3, p->tcf};
  for (int i = 0; i < 4; ++i)
    if (vals[i] < 1) return fail(TSM2X_EINVAL, "%s must be >= 1, got %d", names[i], vals[i]);
  if (p->t3 > p->t1) return fail(TSM2X_EINVAL, "t3 (%d) must not exceed t1 (%d)", p->t3, p->t1);
  if ((int64_t)p->t2 > n) return fail(TSM2X_EINVAL, "t2 (%d) must not exceed n (%lld)", p->t2, (long long)n);
  if (p->t1 % 32 != 0) return fail(TSM2X_EINVAL, "t1 (%d) must be a multiple of warp size 32", p->t1);
  const bool params_tsm2l = p->variant == TSM2X_L_OPT1 || p->variant == TSM2X_L_OPT2;
  if (p->tcf > 1 && !params_tsm2l) return fail(TSM2X_EINVAL, "tcf > 1 is only meaningful for the TSM2L variants");
  return TSM2X_OK;
}

// ------------------------------------------------------------------------------------------
// device properties
struct DevInfo {
  int sms = 0;
  int major = 0, minor = 0;
  bool ok = false;
};
static std::mutex g_dev_mu;
static std::map<int, DevInfo> g_devs;

static int device_info(int dev, DevInfo* out) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_devs.find(dev);
  if (it == g_devs.end()) {
    DevInfo d;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) return fail(TSM2X_ECUDA, "cudaGetDeviceProperties(%d): %s", dev, cudaGetErrorString(e));
    d.sms = prop.multiProcessorCount;
    d.major = prop.major;
    d.minor = prop.minor;
    d.ok = (prop.major == 10 && prop.minor == 0);
    it = g_devs.emplace(dev, d).first;
  }
  *out = it->second;
  if (!out->ok)
    return fail(TSM2X_EUNSUPPORTED, "libtsm2x.so is built for sm_100a (B200); device %d is sm_%d%d", dev, out->major,
                out->minor);
  return TSM2X_OK;
}

template <typename K>
static int occupancy(K kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = reinterpret_cast<const void*>(kernel);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  cache[key] = occ;
  return occ;
}

// ------------------------------------------------------------------------------------------
// per-(device, stream) workspace: Bt + stream-K partials (grown on demand) and arrival
// counters (zeroed on allocation, restored to zero by the kernels themselves).
struct Workspace {
  std::mutex mu;  // held for the whole enqueue of one call
  void* buf = nullptr;
  size_t cap = 0;
  int* counters = nullptr;
  size_t ccap = 0;
  int* flag = nullptr;  // zero-C check result
};
static std::mutex g_ws_mu;
static std::map<std::pair<int, cudaStream_t>, std::unique_ptr<Workspace>> g_ws;

static Workspace* workspace_for(int dev, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& slot = g_ws[{dev, s}];
  if (!slot) slot.reset(new Workspace());
  return slot.get();
}

// Growing the workspace inside a stream capture would bake graph-owned memory (and an un-run
// zeroing memset) into the workspace: refuse, the caller makes one eager call of the same (or a
// larger) shape on the stream before capturing. Graphs captured on one stream share that
// stream's workspace (queue counters, Bt, accumulators): they must not replay concurrently with
// each other or with eager calls on the same stream (see tsm2x.h).
static int ws_reserve(Workspace* w, size_t bytes, size_t counters, cudaStream_t s) {
  bytes = std::max<size_t>(bytes, 1 << 20);
  const size_t cwant = std::max<size_t>(counters + 1, 4096);
  if (bytes > w->cap || cwant > w->ccap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TSM2X_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(TSM2X_EUNSUPPORTED,
                  "workspace of this stream must grow (%zu -> %zu bytes) during a CUDA graph capture: make one "
                  "eager call of this shape on the stream before capturing",
                  w->cap, std::max(bytes, w->cap));
  }
  if (bytes > w->cap) {
    if (w->buf) TSM2X_CUDA(cudaFreeAsync(w->buf, s));
    w->buf = nullptr;
    size_t cap = std::max(bytes, w->cap * 2);
    if (cudaMallocAsync(&w->buf, cap, s) != cudaSuccess) {
      cudaGetLastError();
      w->cap = 0;
      return fail(TSM2X_ENOMEM, "workspace allocation of %zu bytes failed", cap);
    }
    w->cap = cap;
  }
  counters = std::max<size_t>(counters + 1, 4096);
  if (counters > w->ccap) {
    if (w->counters) TSM2X_CUDA(cudaFreeAsync(w->counters, s));
    w->counters = nullptr;
    size_t cap = std::max(counters, w->ccap * 2);
    if (cudaMallocAsync(reinterpret_cast<void**>(&w->counters), cap * sizeof(int), s) != cudaSuccess) {
      cudaGetLastError();
      w->ccap = 0;
      return fail(TSM2X_ENOMEM, "counter allocation failed");
    }
    TSM2X_CUDA(cudaMemsetAsync(w->counters, 0, cap * sizeof(int), s));
    w->ccap = cap;
    w->flag = w->counters + (cap - 1);
  }
  return TSM2X_OK;
}

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
static inline int nt_for(int w) { return w <= 1 ? 1 : w <= 2 ? 2 : w <= 4 ? 4 : w <= 8 ? 8 : 16; }
static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ------------------------------------------------------------------------------------------

// ---- TMA descriptor for A (2-D: dim0 = rows, dim1 = columns; OOB elements read as zero)
// Experiment knobs read once per process: TSM2X_L2POL (L2 policy of the A stream, policy_for) and
// TSM2X_L2PROMO (tensor-map L2 promotion: 0, 64, 128, 256 bytes; default 128 — sustained A/B,
// profiles/l2promo_r02.json: 256 B was 0.3-3.5 % slower on every workload, 0 / 64 / 128 tie).
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static int l2_policy() {
  static const int v = env_int("TSM2X_L2POL", 0);
  return v;
}
static CUtensorMapL2promotion l2_promotion() {
  static const int v = env_int("TSM2X_L2PROMO", 128);
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
         : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                    : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

static int encode_a_map(CUtensorMap* map, const void* A, int64_t m, int64_t k, int64_t lda, size_t eb, int box_rows,
                        int box_cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode) return fail(TSM2X_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)k};
  cuuint64_t strides[1] = {(cuuint64_t)(lda * eb)};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, eb == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      const_cast<void*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TSM2X_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TSM2X_OK;
}

// A as a 3-D tensor {16 rows, k columns, ceil(m/16) row chunks} for the swizzled DMMA layout
// (DmmaConsumer<..., SWZ = true>): a box {16, KC, R/16} lands as [chunk][column][16 rows] with the
// 128-byte swizzle. Needs lda >= roundup(m, 16) (the last chunk's rows past m are read, never
// stored) — swz_layout_ok.
// The 3-D maps read whole row chunks: the last column's rows m .. roundup(m, chunk) - 1 are read
// (never used). Those elements lie inside A's allocation unless A is a sub-view ending near the
// end of its buffer (e.g. big[40:64, :] of a 64-row buffer); tail_in_allocation checks the
// allocation range with the driver whenever m is not a chunk multiple.
static bool tail_in_allocation(const void* A, int64_t m, int64_t k, int64_t lda, size_t eb, int64_t chunk) {
  if (m % chunk == 0) return true;
  using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static AddrRangeFn range = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range = reinterpret_cast<AddrRangeFn>(fn);
  });
  if (!range) return false;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)A) != CUDA_SUCCESS) {
    cudaGetLastError();
    return false;
  }
  const uint64_t end = (uint64_t)(uintptr_t)A + (uint64_t)((k - 1) * lda + (m + chunk - 1) / chunk * chunk) * eb;
  return end <= (uint64_t)base + size;
}
static bool swz_layout_ok(const void* A, int64_t m, int64_t k, int64_t lda) {
  static const bool on = env_int("TSM2X_SWZ", 1) != 0;  // TSM2X_SWZ=0: plain layout (A/B experiments)
  return on && aligned16(A) && (lda % 2) == 0 && lda >= (m + 15) / 16 * 16 && tail_in_allocation(A, m, k, lda, 8, 16);
}
static int encode_a_map_swz(CUtensorMap* map, const double* A, int64_t m, int64_t k, int64_t lda, int kc, int r) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode) return fail(TSM2X_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[3] = {16, (cuuint64_t)k, (cuuint64_t)((m + 15) / 16)};
  cuuint64_t strides[2] = {(cuuint64_t)(lda * 8), 128};
  cuuint32_t box[3] = {16, (cuuint32_t)kc, (cuuint32_t)(r / 16)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult res = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(A), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS) return fail(TSM2X_ECUDA, "cuTensorMapEncodeTiled (swizzled fp64) failed (%d)", (int)res);
  return TSM2X_OK;
}

// A as a 3-D tensor {32 rows, k columns, ceil(m/32) row chunks} for tsm2r_stream_tc32: a box
// {32, 16, 16} lands in smem as [chunk][column][32 rows] with the 128B / 32B-atom swizzle — the
// UMMA SWIZZLE_128B_BASE32B MN-major layout. Needs lda >= roundup(m, 32) (the last chunk's rows
// past m are read, never stored).
static int encode_a_map_tc32(CUtensorMap* map, const float* A, int64_t m, int64_t k, int64_t lda) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode) return fail(TSM2X_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[3] = {32, (cuuint64_t)k, (cuuint64_t)((m + 31) / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)(lda * 4), 128};
  cuuint32_t box[3] = {32, (cuuint32_t)Tc32Cfg::KC, (cuuint32_t)(Tc32Cfg::R / 32)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(A), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, l2_promotion(),
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TSM2X_ECUDA, "cuTensorMapEncodeTiled (tc32) failed (%d)", (int)r);
  return TSM2X_OK;
}

// ---- paper ablation kernels (V0/V1/V2), launched with the caller's t1/t2/t3 -----------------
template <typename T, int NT>
static int launch_ablation_nt(int variant, int64_t m, int64_t k, int64_t n, const T* A, int64_t lda, const T* B,
                              int64_t ldb, T* C, int64_t ldc, int t1, int t2, int t3, bool c_is_zero, cudaStream_t s) {
  const unsigned grid = (unsigned)((m + t1 - 1) / t1);
  if (variant == TSM2X_V1) {
    ablation_v1<T, NT><<<grid, t1, 0, s>>>(A, lda, B, ldb, C, ldc, m, k, n, t2, c_is_zero);
  } else {
    const size_t smem = (size_t)t1 * NT * sizeof(T);
    if (smem > 48 * 1024)
      TSM2X_CUDA(cudaFuncSetAttribute(ablation_v2<T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ablation_v2<T, NT><<<grid, t1, smem, s>>>(A, lda, B, ldb, C, ldc, m, k, n, t2, t3, c_is_zero);
  }
  return check_launch("ablation");
}

template <typename T>
static int run_ablation(int variant, int64_t m, int64_t k, int64_t n, const T* A, int64_t lda, const T* B, int64_t ldb,
                        T* C, int64_t ldc, const tsm2x_params* p, bool c_is_zero, cudaStream_t s) {
  if (p->t1 > 1024) return fail(TSM2X_EUNSUPPORTED, "ablation kernels need t1 <= 1024 (one thread per row), got %d", p->t1);
  if (variant == TSM2X_V0) {
    ablation_v0<T><<<(unsigned)((m + p->t1 - 1) / p->t1), p->t1, 0, s>>>(A, lda, B, ldb, C, ldc, m, k, n, c_is_zero);
    return check_launch("ablation_v0");
  }
  const int t2 = std::min(p->t2, 16);  // register width of one pass (wider t2 runs as 16-wide passes)
  const int t3 = p->t3;
  switch (nt_for(t2)) {
    case 1: return launch_ablation_nt<T, 1>(variant, m, k, n, A, lda, B, ldb, C, ldc, p->t1, t2, t3, c_is_zero, s);
    case 2: return launch_ablation_nt<T, 2>(variant, m, k, n, A, lda, B, ldb, C, ldc, p->t1, t2, t3, c_is_zero, s);
    case 4: return launch_ablation_nt<T, 4>(variant, m, k, n, A, lda, B, ldb, C, ldc, p->t1, t2, t3, c_is_zero, s);
    case 8: return launch_ablation_nt<T, 8>(variant, m, k, n, A, lda, B, ldb, C, ldc, p->t1, t2, t3, c_is_zero, s);
    default: return launch_ablation_nt<T, 16>(variant, m, k, n, A, lda, B, ldb, C, ldc, p->t1, t2, t3, c_is_zero, s);
  }
}

// ---- TSM2R pass: C[:, p:p+w] (+)= A * B[:, p:p+w] -----------------------------------------
// Bt (this pass of B, row-major, zero padded to kpad rows) at the front of the workspace.
// frag = true: DMMA fragment order instead (prep_bfrag; fp64, NT in {8, 16}).
template <typename T, int NT>
static int stage_bt(Workspace* ws, int64_t k, int64_t kpad, int w, const T* B, int64_t ldb, size_t extra_bytes,
                    size_t counters, cudaStream_t s, T** Bt, char** rest, bool frag = false) {
  const size_t bt_bytes = align_up((size_t)kpad * NT * sizeof(T), 256);
  TSM2X_TRY(ws_reserve(ws, bt_bytes + extra_bytes, counters, s));
  *Bt = reinterpret_cast<T*>(ws->buf);
  *rest = static_cast<char*>(ws->buf) + bt_bytes;
  const int64_t tot = kpad * NT;
  if constexpr (sizeof(T) == 8 && (NT == 8 || NT == 16)) {
    if (frag) {
      prep_bfrag<NT><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(B, ldb, k, kpad, w, *Bt);
      return check_launch("prep_bfrag");
    }
  }
  prep_bt<T, NT><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(B, ldb, k, kpad, w, *Bt);
  return check_launch("prep_bt");
}

// ---- parameter selection (the B200 re-derivation of the paper's t1/t2/t3/tcf choice) ---------
// Process-wide tuning knobs (tsm2x_set_tuning); zeros mean "B200 default" — the values below
// were picked from on-device sweeps (tools/tune.py, profiles/tuning_*.json).
struct Tuning {
  int consumer = 0;   // 0 auto, 1 fma, 2 dmma, 3 ffma2
  int small_kb = 0;   // A bytes per small item (KB); default min(512, max(64, per-CTA share / 48))
  int big_kb = 0;     // A bytes per big item (KB);   default min(4096, max(small, per-CTA share / 6))
  int tail_pct = 0;   // % of each row block's columns dispatched as small items; default 20
  int batch_kb = 0;   // single-chunk row blocks (TSM2L): A bytes per queue grab (tcf analogue); default 1024
  int combine = 0;    // split row blocks: 0 auto (fp64 atomics; chunk-ordered when DETERMINISTIC is asked),
                      // 1 chunk-ordered via tickets (bitwise reproducible), 2 fp64 atomics, 3 static split
};
static std::mutex g_tune_mu;
static Tuning g_tune;
static Tuning current_tuning() {
  std::lock_guard<std::mutex> lk(g_tune_mu);
  return g_tune;
}

// Consumer choice (tsm2r_tma.cuh, tsm2r_tc32.cuh): DMMA for fp64 passes of width 8 or 16 (fewer
// issue slots and less energy per FMA than DFMA), split-precision tf32 tensor cores for fp32
// 16-column passes, packed FFMA2 for other fp32 widths, plain FMA otherwise.
// TSM2X_CONSUMER=fma|dmma|ffma2|tc in the environment overrides (ablation runs).
// kDmmaS / kDmmaPS: kDmma / kDmmaP on the swizzled A layout (internal; chosen by layout, not tuning)
enum ConsumerKind { kFma = 0, kDmma = 1, kFfma2 = 2, kNull = 3, kTc = 4, kDmmaP = 5, kDmmaS = 6, kDmmaPS = 7 };

static int pick_consumer_rt(size_t eb, int nt, bool split, const Tuning& tu) {
  static const int env = [] {
    const char* e = getenv("TSM2X_CONSUMER");
    if (!e) return -1;
    if (!strcmp(e, "fma")) return (int)kFma;
    if (!strcmp(e, "dmma")) return (int)kDmma;
    if (!strcmp(e, "ffma2")) return (int)kFfma2;
    if (!strcmp(e, "tc")) return (int)kTc;
    if (!strcmp(e, "dmmap")) return (int)kDmmaP;  // DMMA, k-step software-pipelined loop  // fp32: split-precision tf32 on tcgen05 (tsm2r_tc32.cuh)
    if (!strcmp(e, "null")) return (int)kNull;  // diagnostic: pipeline only, wrong results
    return -1;
  }();
  if (env == kNull) return kNull;
  const int want = env >= 0 ? env
                            : (tu.consumer == 1   ? kFma
                               : tu.consumer == 2 ? kDmma
                               : tu.consumer == 3 ? kFfma2
                               : tu.consumer == 4 ? kTc
                               : tu.consumer == 5 ? kDmmaP
                                                  : -1);
  const bool dmma_ok = eb == 8 && (nt == 8 || nt == 16);
  const bool ffma2_ok = eb == 4 && nt >= 2;
  if (want == kFma) return kFma;
  if (want == kDmma) return dmma_ok ? kDmma : kFma;
  if (want == kDmmaP) return dmma_ok ? kDmmaP : kFma;
  if (want == kFfma2) return ffma2_ok ? kFfma2 : kFma;
  if (want == kTc) return eb == 4 ? kTc : (dmma_ok ? kDmma : kFma);
  // fp64 8- and 16-column passes: DMMA. At n=8 DMMA and DFMA take the same time under the 1000 W
  // cap on most parts (DMMA runs ~300 MHz higher for the same energy) and DMMA is up to 3 %
  // faster on others (profiles/envab_r01.json); at n=16 DMMA wins outright. Split row blocks
  // (TSM2R) use the k-step software-pipelined loop (-4.8 % n=16, -1.1 % n=8 sustained);
  // single-chunk row blocks (TSM2L, two stages per item) the plain loop (pipelining +25 %)
  if (dmma_ok) return split ? kDmmaP : kDmma;
  // fp32 16-column passes with split row blocks (TSM2R): split-precision tf32 on the tensor cores
  // (tsm2r_tc32.cuh; taken when the layout allows, else FFMA2): -13 % burst, -13 % sustained vs
  // FFMA2 (profiles/envab_r01.json). Single-chunk row blocks (TSM2L) stay on FFMA2, whose
  // direct-store epilogue streams C at 0.89 of the copy rate (2^24 x 16 x 16: 0.368 vs 0.597 ms
  // sustained, profiles/tsm2l_fp32_r02.json)
  if (eb == 4 && nt == 16) return split ? kTc : kFfma2;
  if (ffma2_ok) return kFfma2;
  return kFma;
}

// TSM2X_CONSUMER=tc in the environment (A/B runs, tests) forces the tensor cores everywhere
static bool env_forces_tc() {
  static const bool v = [] {
    const char* e = getenv("TSM2X_CONSUMER");
    return e && !strcmp(e, "tc");
  }();
  return v;
}

// "Small" calls (A <= 256 MB): launch-bound, so they take the single-launch variants (inline B;
// fp32 reductions into C).
static inline bool small_call(int64_t m, int64_t k, size_t eb) {
  return (double)m * (double)k * (double)eb <= 256.0 * 1048576.0;
}
// fp32 C += calls up to 128 MB of A skip the tensor cores' three launches (prep, tc32, finalize)
// for one FFMA2 launch with fp32 reductions into C: 512^2..4096^2 x 16 12-27 % faster, 8192^2
// (256 MB) 6 % slower (tools/small_vs_cublas.py, profiles/small_vs_cublas_r02.jsonl)
static inline bool f32_direct_call(int64_t m, int64_t k) {
  return (double)m * (double)k * 4.0 <= 128.0 * 1048576.0;
}

// Whether an fp32 pass of width nt splits its row blocks into several column chunks (TSM2R) or
// runs them as single chunks (TSM2L shapes), on the FFMA2 geometry (make_items below).
static bool fp32_split(int sms, int64_t m, int64_t k, int nt);

// fp32 split row blocks: the fp64 accumulator -> C pass, launched with programmatic dependent
// launch so its launch latency hides behind the stream kernel's tail (the stream kernels trigger
// their dependents once every CTA is resident; tsm2_finalize waits for their completion).
template <typename T>
static int launch_finalize(unsigned grid, const double* acc, int64_t ldacc, T* C, int64_t ldc, int64_t m, int w,
                           int c_is_zero, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TSM2X_CUDA(cudaLaunchKernelEx(&cfg, tsm2_finalize<T>, acc, ldacc, C, ldc, m, w, c_is_zero));
  return check_launch("tsm2_finalize");
}

// fp64 3- and 4-column passes run on the DMMA kernel's 8-column tile (B zero-padded): since the
// swizzled layout a DMMA call at n=8 costs less energy than a DFMA one at n=4 (profiles/
// energy_r01.log), so under the power cap: sustained 30720^2 n=4 -4.2 %, n=3 -3.9 %, TSM2L
// 2^25 x 16 x 4 -8.1 % (profiles/swizzle_r01.txt). Not when a consumer is forced (tuning knob or
// TSM2X_CONSUMER); TSM2X_N4_DMMA=0 turns it off.
static bool n4_on_dmma(const Tuning& tu) {
  static const bool on = env_int("TSM2X_N4_DMMA", 1) != 0 && getenv("TSM2X_CONSUMER") == nullptr;
  return on && tu.consumer == 0 && tu.combine != 3;
}

// Item geometry of the dynamic TMA kernel for one pass (rows_per_block = R, KC columns/stage).
// A bytes per CTA up to which make_items uses equal items (TSM2X_MID_MB overrides, read once)
static double mid_size_cap() {
  static const double v = env_int("TSM2X_MID_MB", 24) * 1048576.0;
  return v;
}
static void make_items(int sms, int64_t m, int64_t k, size_t eb, int R, int KC, int nt, const Tuning& tu, Items* it,
                       int64_t* grid) {
  const int64_t G_full = sms;  // one CTA per SM (smem-bound by design)
  it->num_rb = (m + R - 1) / R;
  const double col_bytes = (double)R * eb;  // one column of one row block
  const double per_cta = (double)m * k * eb / (double)G_full;
  // 16-column passes and the fp64 DMMA passes: fewer, larger items and a shorter small-item
  // tail (fewer item epilogues and fp64 reductions per byte; sustained A/B,
  // profiles/abtest_r01.json, and for the 64 KB-stage DMMA passes small 1 MB + tail 10 % + big
  // 8 MB: n=8 -1.6 %, big 8 MB at n=16 -0.7 %). The caps only bind for large problems.
  const bool dmma_pass = eb == 8 && nt >= 8;
  const double small_cap = (nt >= 16 || dmma_pass) ? 1024.0 * 1024 : 512.0 * 1024;
  const double big_cap = dmma_pass ? 8.0 * 1024 * 1024 : 4.0 * 1024 * 1024;
  const double small_b = tu.small_kb > 0 ? tu.small_kb * 1024.0 : std::min(small_cap, std::max(64.0 * 1024, per_cta / 48));
  const double big_b =
      tu.big_kb > 0 ? std::max(small_b, tu.big_kb * 1024.0) : std::min(big_cap, std::max(small_b, per_cta / 6));
  const int64_t ksmall = std::max<int64_t>(KC, (int64_t)align_up((size_t)(small_b / col_bytes), KC));
  const int64_t kbig = std::max<int64_t>(ksmall, (int64_t)align_up((size_t)(big_b / col_bytes), KC));
  // single-chunk dispatch batch: 64 KB (one row block at k=16) — burst sweep (tuning_r01.json) and
  // sustained A/B (-0.5 %) agree on it with the current kernel; 256 KB was the earlier choice
  const double batch_b = tu.batch_kb > 0 ? tu.batch_kb * 1024.0 : 64.0 * 1024;
  const bool mid = tu.small_kb == 0 && tu.big_kb == 0 && tu.tail_pct == 0 && per_cta <= mid_size_cap();
  const bool single_ok = (double)k * col_bytes <= 1024.0 * 1024 || k <= ksmall;
  // fewer row blocks than CTAs: the equal-split rule below decides whether to split (an unsplit
  // fp32 512 x 512 x 16 ran on one CTA: 45 us vs 12 us for cuBLAS)
  if (single_ok && !(mid && it->num_rb < G_full)) {
    // single-chunk row blocks (TSM2L shapes): no split, batched dispatch
    it->nbig = 0;
    it->kbig = KC;
    it->kbig_end = 0;
    it->nsmall = 1;
    it->ksmall = (int64_t)align_up((size_t)k, KC);
    it->batch = std::max<int64_t>(1, (int64_t)(batch_b / ((double)k * col_bytes)));
  } else if (mid) {
    // up to ~24 MB of A per CTA (m = k = 20480 fp64): equal column ranges per row block, in as few
    // rounds of one item per CTA as the makespan allows. Per-item epilogues and the ramp, not
    // HBM, bound mid-size problems, and the queue's tail balancing buys nothing there (ncu cold:
    // 2048^2 n=16 25 -> 17 us, 4096^2 n=16 36 -> 29 us, 6144^2 n=16 69 -> 51 us; sustained: 6144^2
    // n=16 -29 %, 8192^2 -9 / -14 %, 12288^2 -5 / -6 %, 16384^2 -2 / -3 %, 20480^2 -2 %; 30720^2
    // unchanged within noise, so the large-problem split below stays; profiles/midsize_r01.jsonl)
    // pieces per row block: minimise the makespan (rounds of items per CTA x item columns, plus a
    // per-item cost of ~KC columns for the epilogue)
    int64_t c = (int64_t)align_up((size_t)k, KC);
    double best = 1e300;
    for (int64_t p = 1; p <= 256; ++p) {
      const int64_t cp = std::max<int64_t>(KC, (int64_t)align_up((size_t)((k + p - 1) / p), KC));
      const int64_t np = (k + cp - 1) / cp;
      const int64_t rounds = (it->num_rb * np + G_full - 1) / G_full;
      const double cost = (double)rounds * (double)(cp + KC);
      if (cost < best) {
        best = cost;
        c = cp;
      }
      if (cp == KC) break;
    }
    it->nbig = 0;
    it->kbig = c;
    it->kbig_end = 0;
    it->ksmall = c;
    it->nsmall = (k + c - 1) / c;
    it->batch = 1;
  } else {
    const int pct = tu.tail_pct > 0 ? std::min(tu.tail_pct, 100) : ((nt >= 16 || dmma_pass) ? 10 : 20);
    const int64_t tail_cols = std::max<int64_t>(1, (k * pct + 99) / 100);
    const int64_t tail = std::min<int64_t>(k, (int64_t)align_up((size_t)tail_cols, (size_t)ksmall));
    it->kbig_end = ((k - tail) / KC) * KC;
    it->kbig = kbig;
    it->nbig = it->kbig_end > 0 ? (it->kbig_end + kbig - 1) / kbig : 0;
    it->ksmall = ksmall;
    it->nsmall = (k - it->kbig_end + ksmall - 1) / ksmall;
    it->batch = 1;
  }
  it->total = it->num_rb * it->nch();
  *grid = std::min<int64_t>(G_full, (it->total + it->batch - 1) / it->batch);
}

static bool fp32_split(int sms, int64_t m, int64_t k, int nt) {
  using Cfg = TmaCfg<float, 16>;
  Items it;
  int64_t G;
  make_items(sms, m, k, 4, Cfg::R, Cfg::KC, nt, current_tuning(), &it, &G);
  return it.nch() > 1;
}

template <typename T, int NT, int KIND, int RPT, int CW, int SB = 32768>
struct ConsumerFor {
  using type = FmaConsumer<T, NT, RPT, CW, SB>;
};
// DMMA geometries: 512-row blocks (RPT * CW == 16: 8 warps x 64 rows or 16 x 32) or 1024-row
// blocks (16 warps x 64 rows, RPT = 2); swizzled variants need 64 KB stages and 64 rows per warp
template <int RPT, int CW, int SB>
struct DmmaGeom {
  static constexpr int R = 32 * RPT * CW;
  // 1024-row blocks only with 64 KB stages (8 columns: two 4-column k-steps for the pipelined loop)
  static constexpr bool ok = (RPT * CW == 16 && (CW == 8 || CW == 16)) || (RPT * CW == 32 && CW == 16 && SB == 65536);
  static constexpr bool swz_ok = ok && R / CW == 64 && SB == 65536;
};
template <int NT, int RPT, int CW, int SB>
struct ConsumerFor<double, NT, kDmma, RPT, CW, SB> {
  using type = typename std::conditional<((NT == 8 || NT == 16) && DmmaGeom<RPT, CW, SB>::ok && (CW == 8 || CW == 16)),
                                         DmmaConsumer<(NT >= 8 ? NT : 8), (CW == 16 ? 16 : 8), false, SB, false,
                                                      DmmaGeom<RPT, CW, SB>::R>,
                                         FmaConsumer<double, NT, RPT, CW, SB>>::type;
};
template <int NT, int RPT, int CW, int SB>
struct ConsumerFor<double, NT, kDmmaP, RPT, CW, SB> {
  using type = typename std::conditional<((NT == 8 || NT == 16) && DmmaGeom<RPT, CW, SB>::ok && (CW == 8 || CW == 16)),
                                         DmmaConsumer<(NT >= 8 ? NT : 8), (CW == 16 ? 16 : 8), true, SB, false,
                                                      DmmaGeom<RPT, CW, SB>::R>,
                                         FmaConsumer<double, NT, RPT, CW, SB>>::type;
};
template <int NT, int RPT, int CW, int SB>
struct ConsumerFor<double, NT, kDmmaS, RPT, CW, SB> {
  using type = typename std::conditional<((NT == 8 || NT == 16) && DmmaGeom<RPT, CW, SB>::swz_ok && SB == 65536),
                                         DmmaConsumer<(NT >= 8 ? NT : 8), (CW == 16 ? 16 : 8), false, 65536, true,
                                                      DmmaGeom<RPT, CW, SB>::R>,
                                         FmaConsumer<double, NT, RPT, CW, SB>>::type;
};
template <int NT, int RPT, int CW, int SB>
struct ConsumerFor<double, NT, kDmmaPS, RPT, CW, SB> {
  using type = typename std::conditional<((NT == 8 || NT == 16) && DmmaGeom<RPT, CW, SB>::swz_ok && SB == 65536),
                                         DmmaConsumer<(NT >= 8 ? NT : 8), (CW == 16 ? 16 : 8), true, 65536, true,
                                                      DmmaGeom<RPT, CW, SB>::R>,
                                         FmaConsumer<double, NT, RPT, CW, SB>>::type;
};
template <typename T, int NT, int RPT, int CW, int SB>
struct ConsumerFor<T, NT, kNull, RPT, CW, SB> {
  using type = NullConsumer<T, NT, RPT, CW, SB>;
};
template <int NT, int RPT, int CW, int SB>
struct ConsumerFor<float, NT, kFfma2, RPT, CW, SB> {
  using type = typename std::conditional<(NT >= 2 && RPT == 4 && CW == 8 && SB == 32768), Ffma2Consumer<(NT >= 2 ? NT : 2)>,
                                         FmaConsumer<float, NT, RPT, CW, SB>>::type;
};

template <typename T, int NT, int KIND, int RPT, int CW, int SB = 32768>
static int launch_tma_kernel(const DynArgs<T>& a_in, const CUtensorMap& tmap_in, int64_t G, cudaStream_t s) {
  // inline B: the kernel is the call's first launch, so it must not start before the previous
  // work on the stream has finished (no programmatic serialization)
  using Cons = typename ConsumerFor<T, NT, KIND, RPT, CW, SB>::type;
  using Cfg = typename Cons::Cfg;
  static_assert(Cfg::R == TmaCfg<T, NT, RPT, CW, SB>::R && Cfg::KC == TmaCfg<T, NT, RPT, CW, SB>::KC,
                "consumer / plan geometry mismatch");
  auto kern = tsm2r_stream_tma<T, NT, Cons>;
  TSM2X_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  DynArgs<T> a = a_in;
  alignas(64) CUtensorMap tmap = tmap_in;
  // programmatic dependent launch: overlap this kernel's launch + prologue with prep_dyn
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.inline_b ? 0 : 1;
  TSM2X_CUDA(cudaLaunchKernelEx(&cfg, kern, a, tmap));
  return check_launch("tsm2r_stream_tma");
}

// TMA flavour, dynamic items (tsm2r_tma.cuh): item sizes from the per-CTA share of the work.
template <typename T, int NT, int RPT = Vec<T>::N, int CW = 8, int SB = 32768>
static int run_tsm2r_tma(const DevInfo& di, Workspace* ws, int64_t m, int64_t k, int w, const T* A, int64_t lda,
                         const T* B, int64_t ldb, T* C, int64_t ldc, bool c_is_zero, bool ordered,
                         cudaStream_t s) {
  using Cfg = TmaCfg<T, NT, RPT, CW, SB>;
  const size_t eb = sizeof(T);
  const Tuning tu = current_tuning();
  DynArgs<T> a;
  a.C = C;
  a.ldc = ldc;
  a.m = m;
  a.k = k;
  a.w = w;
  a.c_is_zero = c_is_zero ? 1 : 0;
  a.vec_c = aligned16(C) && (ldc % Vec<T>::N == 0);
  a.l2pol = l2_policy();
  Items& it = a.it;
  int64_t G;
  make_items(di.sms, m, k, eb, Cfg::R, Cfg::KC, NT, tu, &it, &G);
  const bool split = it.nch() > 1;
  const int64_t kpad = (int64_t)align_up((size_t)k, Cfg::KC);
  a.ldacc = (int64_t)it.num_rb * Cfg::R;
  a.ordered = ordered ? 1 : 0;
  const bool atomic_split = split && !a.ordered;
  // fp32 split row blocks combine in an fp64 accumulator + tsm2_finalize — except small calls
  // that read C (C += A*B, A <= 128 MB: a few column chunks per row block), which reduce in fp32
  // straight into C: no accumulator to zero, no finalize, and with the inline-B producer one
  // launch per call (fp32 512^2..4096^2 x 16 were launch-bound at three launches)
  const bool f32_direct = sizeof(T) == 4 && atomic_split && !c_is_zero && f32_direct_call(m, k);
  const bool f32_acc = sizeof(T) == 4 && atomic_split && !f32_direct;
  const size_t acc_bytes = f32_acc ? (size_t)a.ldacc * NT * sizeof(double) : 0;
  int kind = pick_consumer_rt(sizeof(T), NT, split, tu);
  // DMMA: the 512-row geometries (8 warps x 2 rows or 16 warps x 1 row); FFMA2: the default one
  if ((kind == kDmma || kind == kDmmaP) && !DmmaGeom<RPT, CW, SB>::ok) kind = kFma;
  if (kind == kFfma2 && (RPT != Vec<T>::N || CW != 8 || SB != 32768)) kind = kFma;
  if (kind == kTc) kind = (sizeof(T) == 4 && RPT == Vec<T>::N && CW == 8 && NT >= 2) ? kFfma2 : kFma;  // tc path not taken
  // the default DMMA geometry reads A through the swizzled layout when the leading dimension
  // allows it (bank-conflict-free fragment loads; DmmaConsumer)
  const bool swz = sizeof(T) == 8 && (kind == kDmma || kind == kDmmaP) && DmmaGeom<RPT, CW, SB>::swz_ok && SB == 65536 &&
                   (NT == 8 || NT == 16) && swz_layout_ok(A, m, k, lda);
  const size_t bt_bytes = align_up((size_t)kpad * NT * sizeof(T), 256);
  TSM2X_TRY(ws_reserve(ws, bt_bytes + acc_bytes, (size_t)it.num_rb + 8, s));
  a.tickets = reinterpret_cast<unsigned*>(ws->counters + 8);  // zero between launches
  a.Bt = reinterpret_cast<T*>(ws->buf);
  a.acc = acc_bytes ? reinterpret_cast<double*>(static_cast<char*>(ws->buf) + bt_bytes) : nullptr;
  a.queue = reinterpret_cast<unsigned long long*>(ws->counters);  // zero between launches
  // the zeroed accumulation target of split row blocks (C itself for fp64 under the zero-C
  // contract, the fp64 accumulator for fp32), if any
  double* zp = nullptr;
  int64_t zld = 0, zrows = 0;
  if (f32_acc) {
    zp = a.acc;
    zld = zrows = a.ldacc;
  } else if (atomic_split && c_is_zero) {
    zp = reinterpret_cast<double*>(C);
    zld = ldc;
    zrows = m;
  }
  // inline B (no prep kernel, the producer warp gathers each stage's Bt rows from B itself):
  // taken when there is nothing to zero and the call is small (A <= 256 MB: one launch per call
  // instead of two, BASELINE configs[0] 30.3 -> 28.6 us). Large calls keep prep_dyn: the
  // per-stage gather costs ~1 % of the stream kernel at n = 8 in burst runs (1.0365 vs 1.0288
  // ms per call, one box, profiles/inline_b_r02.json) and more at n = 16 / on 32 KB stages; only
  // deep in the power-capped regime (> 1 s back to back) is it ~2 % ahead at n = 3..8.
  // TSM2X_INLINE_B = 0 never, 1 always, unset = this rule.
  static const int inline_env = env_int("TSM2X_INLINE_B", -1);
  const bool want_inline = inline_env == 1 || (inline_env < 0 && small_call(m, k, eb));
  if (!zp && want_inline) {
    a.inline_b = 1;
    a.B = B;
    a.ldb = ldb;
  }
  if (!a.inline_b) {
    // one prep launch: Bt, plus the zeroed accumulation target
    const int64_t tot = kpad * NT + (zp ? zrows * w : 0);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, (int64_t)di.sms * 16));
    if constexpr (sizeof(T) == 8 && (NT == 8 || NT == 16)) {
      if (kind == kDmma || kind == kDmmaP) {
        prep_dyn<T, NT, true, double>
            <<<grid, 256, 0, s>>>(B, ldb, k, kpad, w, const_cast<T*>(a.Bt), zp, zld, zrows, w, swz ? 1 : 0);
        TSM2X_TRY(check_launch("prep_dyn"));
      } else {
        prep_dyn<T, NT, false, double><<<grid, 256, 0, s>>>(B, ldb, k, kpad, w, const_cast<T*>(a.Bt), zp, zld, zrows, w);
        TSM2X_TRY(check_launch("prep_dyn"));
      }
    } else {
      prep_dyn<T, NT, false, double><<<grid, 256, 0, s>>>(B, ldb, k, kpad, w, const_cast<T*>(a.Bt), zp, zld, zrows, w);
      TSM2X_TRY(check_launch("prep_dyn"));
    }
  }
#ifdef TSM2X_TC32_DIAG
  static unsigned long long* dbg = nullptr;
  const bool diag = getenv("TSM2X_TC_DIAG") != nullptr;
  constexpr int kDbg = 16 + 5 * 1024;  // counters + per-CTA timeline (tsm2r_stream_tma)
  if (diag) {
    if (!dbg) TSM2X_CUDA(cudaMalloc(&dbg, kDbg * sizeof(unsigned long long)));
    TSM2X_CUDA(cudaMemsetAsync(dbg, 0, kDbg * sizeof(unsigned long long), s));
    a.dbg = dbg;
    a.diag = atoi(getenv("TSM2X_TC_DIAG"));
  }
#endif
  alignas(64) CUtensorMap tmap;
  if (swz)
    TSM2X_TRY(encode_a_map_swz(&tmap, reinterpret_cast<const double*>(A), m, k, lda, Cfg::KC, Cfg::R));
  else
    TSM2X_TRY(encode_a_map(&tmap, A, m, k, lda, eb, Cfg::BOX, Cfg::KC));
  if (swz && kind == kDmma)
    TSM2X_TRY((launch_tma_kernel<T, NT, kDmmaS, RPT, CW, SB>(a, tmap, G, s)));
  else if (swz && kind == kDmmaP)
    TSM2X_TRY((launch_tma_kernel<T, NT, kDmmaPS, RPT, CW, SB>(a, tmap, G, s)));
  else if (kind == kDmma)
    TSM2X_TRY((launch_tma_kernel<T, NT, kDmma, RPT, CW, SB>(a, tmap, G, s)));
  else if (kind == kDmmaP)
    TSM2X_TRY((launch_tma_kernel<T, NT, kDmmaP, RPT, CW, SB>(a, tmap, G, s)));
  else if (kind == kFfma2)
    TSM2X_TRY((launch_tma_kernel<T, NT, kFfma2, RPT, CW, SB>(a, tmap, G, s)));
  else if (kind == kNull)
    TSM2X_TRY((launch_tma_kernel<T, NT, kNull, RPT, CW, SB>(a, tmap, G, s)));
  else
    TSM2X_TRY((launch_tma_kernel<T, NT, kFma, RPT, CW, SB>(a, tmap, G, s)));
#ifdef TSM2X_TC32_DIAG
  if (diag) {
    std::vector<unsigned long long> h(kDbg);
    TSM2X_CUDA(cudaMemcpyAsync(h.data(), dbg, kDbg * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    TSM2X_CUDA(cudaStreamSynchronize(s));
    const double ns = h[4] ? (double)h[4] : 1.0;
    // per-CTA timeline relative to the first CTA's entry: median / max of each event (us)
    unsigned long long t00 = ~0ull;
    for (int64_t c = 0; c < G; ++c) t00 = std::min(t00, h[16 + 5 * c]);
    double med[5], mx[5];
    for (int e = 0; e < 5; ++e) {
      std::vector<double> v;
      for (int64_t c = 0; c < G; ++c)
        if (h[16 + 5 * c + e]) v.push_back((h[16 + 5 * c + e] - t00) * 1e-3);
      std::sort(v.begin(), v.end());
      med[e] = v.empty() ? -1 : v[v.size() / 2];
      mx[e] = v.empty() ? -1 : v.back();
    }
    fprintf(stderr,
            "{\"tma_diag\": \"consumer %d\", \"stages\": %llu, \"wait_full\": %.0f, \"stage\": %.0f, \"finish\": %.0f, "
            "\"timeline_us\": {\"entry\": [%.2f, %.2f], \"first_tma\": [%.2f, %.2f], \"first_stage\": [%.2f, %.2f], "
            "\"producer_done\": [%.2f, %.2f], \"consumers_done\": [%.2f, %.2f]}, \"ctas\": %lld}\n",
            kind, h[4], h[0] / ns, h[1] / ns, h[2] / ns, med[0], mx[0], med[1], mx[1], med[2], mx[2], med[3], mx[3],
            med[4], mx[4], (long long)G);
  }
#endif
  if (f32_acc) {
    const int64_t tot = m * w;
    const unsigned grid = (unsigned)std::min<int64_t>((tot + 255) / 256, (int64_t)di.sms * 8);
    TSM2X_TRY(launch_finalize<T>(grid, a.acc, a.ldacc, C, ldc, m, w, a.c_is_zero, s));
  }
  return TSM2X_OK;
}

// fp32 on the tensor cores (tsm2r_tc32.cuh): split-precision tf32, one 16-column pass (w <= 16).
// Dynamic items as run_tsm2r_tma; split row blocks combine with fp64 reductions into the fp64
// accumulator (+ tsm2_finalize), single-chunk row blocks store C directly.
static bool tc32_ok(const float* A, int64_t m, int64_t k, int64_t lda) {
  return aligned16(A) && lda % 4 == 0 && lda >= (int64_t)align_up((size_t)m, 32) && m < (int64_t(1) << 31) &&
         k < (int64_t(1) << 31) && tail_in_allocation(A, m, k, lda, 4, 32);
}

static int run_tsm2r_tc32(const DevInfo& di, Workspace* ws, int64_t m, int64_t k, int w, const float* A, int64_t lda,
                          const float* B, int64_t ldb, float* C, int64_t ldc, bool c_is_zero, cudaStream_t s) {
  using Cfg = Tc32Cfg;
  const Tuning tu = current_tuning();
  DynArgs<float> a;
  a.C = C;
  a.ldc = ldc;
  a.m = m;
  a.k = k;
  a.w = w;
  a.c_is_zero = c_is_zero ? 1 : 0;
  a.vec_c = 0;
  a.l2pol = l2_policy();
  Items& it = a.it;
  int64_t G;
  make_items(di.sms, m, k, sizeof(float), Cfg::R, Cfg::KC, 16, tu, &it, &G);
  const bool split = it.nch() > 1;
  const int64_t nstages = (k + Cfg::KC - 1) / Cfg::KC;
  a.ldacc = (int64_t)it.num_rb * Cfg::R;
  a.ordered = 0;
  const size_t acc_bytes = split ? (size_t)a.ldacc * 16 * sizeof(double) : 0;
  const size_t bt_bytes = align_up((size_t)nstages * Cfg::B_BYTES, 256);
  TSM2X_TRY(ws_reserve(ws, bt_bytes + acc_bytes, (size_t)it.num_rb + 8, s));
  a.tickets = reinterpret_cast<unsigned*>(ws->counters + 8);
  a.Bt = reinterpret_cast<const float*>(ws->buf);
  a.acc = acc_bytes ? reinterpret_cast<double*>(static_cast<char*>(ws->buf) + bt_bytes) : nullptr;
  a.queue = reinterpret_cast<unsigned long long*>(ws->counters);
  {
    const int64_t tot = nstages * 512 + (a.acc ? a.ldacc * w : 0);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, (int64_t)di.sms * 16));
    prep_tc32<<<grid, 256, 0, s>>>(B, ldb, k, nstages, w, const_cast<float*>(a.Bt), a.acc, a.ldacc, a.ldacc, w);
    TSM2X_TRY(check_launch("prep_tc32"));
  }
#ifdef TSM2X_TC32_DIAG
  // diagnostics (TSM2X_TC_DIAG=<skip bits>, any value enables the cycle counters; printed to stderr)
  static const int env_diag = [] {
    const char* e = getenv("TSM2X_TC_DIAG");
    return e ? atoi(e) + 0x10000 : 0;
  }();
  static unsigned long long* dbg = nullptr;
  if (env_diag) {
    if (!dbg) TSM2X_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
    TSM2X_CUDA(cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), s));
    a.diag = env_diag & 0xffff;
    a.dbg = dbg;
  }
#else
  constexpr int env_diag = 0;
  unsigned long long* dbg = nullptr;
#endif
  alignas(64) CUtensorMap tmap;
  TSM2X_TRY(encode_a_map_tc32(&tmap, A, m, k, lda));
  auto kern = split ? tsm2r_stream_tc32<false> : tsm2r_stream_tc32<true>;
  TSM2X_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TSM2X_CUDA(cudaLaunchKernelEx(&cfg, kern, a, tmap));
  TSM2X_TRY(check_launch("tsm2r_stream_tc32"));
  if (env_diag) {
    unsigned long long h[16];
    TSM2X_CUDA(cudaMemcpyAsync(h, dbg, sizeof h, cudaMemcpyDeviceToHost, s));
    TSM2X_CUDA(cudaStreamSynchronize(s));
    const double ns = h[4] ? (double)h[4] : 1.0;
    fprintf(stderr,
            "{\"tc32_diag\": %d, \"stages\": %llu, \"mma_wait_full\": %.0f, \"mma_wait_lo\": %.0f, \"mma_issue\": %.0f, "
            "\"mma_wait_acc\": %.0f, \"conv_wait_full\": %.0f, \"conv_wait_lo_empty\": %.0f, \"conv_convert\": %.0f, "
            "\"conv_epilogue\": %.0f}\n",
            env_diag & 0xffff, h[4], h[0] / ns, h[1] / ns, h[2] / ns, h[3] / ns, h[8] / ns, h[9] / ns, h[10] / ns, h[11] / ns);
  }
  if (split) {
    const int64_t tot = m * w;
    const unsigned grid = (unsigned)std::min<int64_t>((tot + 255) / 256, (int64_t)di.sms * 8);
    TSM2X_TRY(launch_finalize<float>(grid, a.acc, a.ldacc, C, ldc, m, w, a.c_is_zero, s));
  }
  return TSM2X_OK;
}

// TMA flavour, static stream-K with fixed-order combine (tsm2r_tma_static.cuh): deterministic.
template <typename T, int NT>
static int run_tsm2r_tma_static(const DevInfo& di, Workspace* ws, int64_t m, int64_t k, int w, const T* A,
                                int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, bool c_is_zero,
                                cudaStream_t s) {
  using Cfg = TmaCfg<T, NT>;
  auto kern = tsm2r_static_tma<T, NT>;
  TSM2X_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int occ = occupancy(kern, Cfg::THREADS, Cfg::SMEM);
  StreamArgs<T> a;
  a.A = A;
  a.lda = lda;
  a.C = C;
  a.ldc = ldc;
  a.m = m;
  a.k = k;
  a.w = w;
  a.c_is_zero = c_is_zero ? 1 : 0;
  a.num_rb = (m + Cfg::R - 1) / Cfg::R;
  a.KC = Cfg::KC;
  const int64_t num_kb = (k + Cfg::KC - 1) / Cfg::KC;
  const int64_t units = a.num_rb * num_kb;
  const int64_t G = std::min<int64_t>(units, (int64_t)di.sms * occ);
  a.part.units = units;
  a.part.num_kb = num_kb;
  a.part.G = G;
  const int64_t max_contrib = (num_kb * G + units - 1) / units + 1;
  a.defer = (max_contrib > 24) ? 1 : 0;
  const size_t part_bytes = (size_t)G * 2 * NT * Cfg::R * sizeof(T);
  T* Bt;
  char* rest;
  TSM2X_TRY((stage_bt<T, NT>(ws, k, num_kb * Cfg::KC, w, B, ldb, part_bytes, (size_t)a.num_rb + 4, s, &Bt, &rest)));
  a.Bt = Bt;
  a.ws = reinterpret_cast<T*>(rest);
  a.counters = ws->counters + 4;
  alignas(64) CUtensorMap tmap;
  TSM2X_TRY(encode_a_map(&tmap, A, m, k, lda, sizeof(T), Cfg::BOX, Cfg::KC));
  void* args[] = {&a, &tmap};
  TSM2X_CUDA(cudaLaunchKernel((const void*)kern, dim3((unsigned)G), dim3(Cfg::THREADS), args, Cfg::SMEM, s));
  TSM2X_TRY(check_launch("tsm2r_static_tma"));
  if (a.defer) {
    dim3 grid((unsigned)((Cfg::R + 255) / 256), (unsigned)a.num_rb);
    reduce_partials<T, NT, Cfg::R><<<grid, 256, 0, s>>>(a);
    TSM2X_TRY(check_launch("reduce_partials"));
  }
  return TSM2X_OK;
}

// LDG flavour: static stream-K (any alignment; the fallback when TMA's 16-byte rules fail)
template <typename T, int NT>
static int run_tsm2r_ldg(const DevInfo& di, Workspace* ws, int64_t m, int64_t k, int w, const T* A, int64_t lda,
                         const T* B, int64_t ldb, T* C, int64_t ldc, bool c_is_zero, cudaStream_t s) {
  constexpr int THREADS = 256, P = 8, KC = 32;
  const bool vec = aligned16(A) && (lda % Vec<T>::N == 0);
  const int R = THREADS * (vec ? Vec<T>::N : 1);
  StreamArgs<T> a;
  a.A = A;
  a.lda = lda;
  a.C = C;
  a.ldc = ldc;
  a.m = m;
  a.k = k;
  a.w = w;
  a.c_is_zero = c_is_zero ? 1 : 0;
  a.num_rb = (m + R - 1) / R;
  a.KC = KC;
  const int64_t num_kb = (k + KC - 1) / KC;
  const int64_t units = a.num_rb * num_kb;
  const void* kfn;
  int occ;
  if (vec) {
    auto kern = tsm2r_stream_ldg<T, NT, THREADS, P, true>;
    occ = occupancy(kern, THREADS, 0);
    kfn = (const void*)kern;
  } else {
    auto kern = tsm2r_stream_ldg<T, NT, THREADS, P, false>;
    occ = occupancy(kern, THREADS, 0);
    kfn = (const void*)kern;
  }
  const int64_t G = std::min<int64_t>(units, (int64_t)di.sms * occ);
  a.part.units = units;
  a.part.num_kb = num_kb;
  a.part.G = G;
  const int64_t max_contrib = (num_kb * G + units - 1) / units + 1;
  a.defer = (max_contrib > 24) ? 1 : 0;
  const size_t part_bytes = (size_t)G * 2 * NT * R * sizeof(T);
  T* Bt;
  char* rest;
  TSM2X_TRY((stage_bt<T, NT>(ws, k, num_kb * KC, w, B, ldb, part_bytes, (size_t)a.num_rb + 4, s, &Bt, &rest)));
  a.Bt = Bt;
  a.ws = reinterpret_cast<T*>(rest);
  a.counters = ws->counters + 4;
  void* args[] = {&a};
  TSM2X_CUDA(cudaLaunchKernel(kfn, dim3((unsigned)G), dim3(THREADS), args, 0, s));
  TSM2X_TRY(check_launch("tsm2r_stream_ldg"));
  if (a.defer) {
    dim3 grid((unsigned)((R + 255) / 256), (unsigned)a.num_rb);
    if (R == 256)
      reduce_partials<T, NT, 256><<<grid, 256, 0, s>>>(a);
    else if (R == 512)
      reduce_partials<T, NT, 512><<<grid, 256, 0, s>>>(a);
    else
      reduce_partials<T, NT, 1024><<<grid, 256, 0, s>>>(a);
    TSM2X_TRY(check_launch("reduce_partials"));
  }
  return TSM2X_OK;
}

template <typename T, int NT>
static int run_tsm2r_pass(const DevInfo& di, Workspace* ws, int impl, int64_t m, int64_t k, int w, const T* A,
                          int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, bool c_is_zero, bool deterministic,
                          cudaStream_t s) {
  // TMA needs 16-byte aligned base and column stride; coordinates are int32
  const bool tma_ok = aligned16(A) && ((lda * (int64_t)sizeof(T)) % 16 == 0) && m < (int64_t(1) << 31) &&
                      k < (int64_t(1) << 31);
  const bool tma = (impl == TSM2X_IMPL_AUTO || impl == TSM2X_IMPL_STREAM_TMA) && tma_ok;
  // combine of split row blocks: fp64 atomics by default (fastest, sustained A/B in
  // profiles/abtest_r01.json); DETERMINISTIC (or tuning.combine = 1) selects the chunk-ordered
  // ticket combine — bitwise reproducible, same dynamic balance and DRAM order, 5-30 % slower;
  // tuning.combine = 3 the static stream-K split (reproducible too, kept for comparison)
  const int combine = current_tuning().combine;
  if (tma && combine == 3) return run_tsm2r_tma_static<T, NT>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, s);
  const bool ordered = combine == 1 || (combine == 0 && deterministic);
  if constexpr (sizeof(T) == 4 && (NT == 16 || NT == 8)) {
    // fp32: the tensor-core consumer when chosen (TSM2X_CONSUMER=tc / tuning consumer 4) and the
    // layout allows the 3-D TMA view; the deterministic (ordered) combine stays on FFMA2
    // small C += calls stay on FFMA2 with fp32 reductions into C: one launch instead of three
    if (tma && !ordered && pick_consumer_rt(4, NT, fp32_split(di.sms, m, k, NT), current_tuning()) == kTc &&
        !(f32_direct_call(m, k) && !c_is_zero && current_tuning().consumer != 4 && !env_forces_tc()) &&
        tc32_ok(reinterpret_cast<const float*>(A), m, k, lda))
      return run_tsm2r_tc32(di, ws, m, k, w, reinterpret_cast<const float*>(A), lda,
                            reinterpret_cast<const float*>(B), ldb, reinterpret_cast<float*>(C), ldc, c_is_zero, s);
  }
  if (tma) {
    // rows per consumer thread (row-block height R = 256 * rpt): TSM2X_RPT overrides for
    // experiments on fp64 8-column passes (1, 2, 4, 8); the default is one 16-byte vector's worth
    static const int env_rpt = [] {
      const char* e = getenv("TSM2X_RPT");
      return e ? atoi(e) : 0;
    }();
    static const int env_cw = [] {
      const char* e = getenv("TSM2X_CW");
      return e ? atoi(e) : 0;
    }();
    // fp64 8/16-column passes (DMMA): 64 KB stages x 3 by default — half the barrier round trips
    // and stage hand-offs per byte for a consumer bound by fragment-load latency (sustained
    // -0.6 % n=8, -1.2 % n=16, -1 to -3 % TSM2L; profiles/README.md); TSM2X_STAGE_KB=32 restores
    // 32 KB x 6
    static const int env_stage_kb = [] {
      const char* e = getenv("TSM2X_STAGE_KB");
      return e ? atoi(e) : 64;
    }();
    static const int env_rb = env_int("TSM2X_RB", 512);  // row-block height of the DMMA passes (experiment)
    if constexpr (sizeof(T) == 8 && (NT == 8 || NT == 16)) {
      if (env_stage_kb == 64 && env_cw == 0 && env_rpt == 0 && env_rb == 512)
        return run_tsm2r_tma<T, NT, 2, 8, 65536>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
      if (env_cw == 16 && env_rpt == 1)  // 16 consumer warps x 1 row: 512-row blocks (DMMA-capable)
        return run_tsm2r_tma<T, NT, 1, 16>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
      if (env_rb == 1024 && env_stage_kb == 64)  // 16 warps x 64 rows: 1024-row blocks, 8 columns per stage
        return run_tsm2r_tma<T, NT, 2, 16, 65536>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
    }
    if constexpr (sizeof(T) == 8 && NT == 8) {
      if (env_cw == 16) return run_tsm2r_tma<T, NT, 2, 16>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
      if (env_cw == 12) return run_tsm2r_tma<T, NT, 2, 12>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
      switch (env_rpt) {
        case 1: return run_tsm2r_tma<T, NT, 1>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
        case 4: return run_tsm2r_tma<T, NT, 4>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
        case 8: return run_tsm2r_tma<T, NT, 8>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
        default: break;
      }
    }
    return run_tsm2r_tma<T, NT>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, ordered, s);
  }
  return run_tsm2r_ldg<T, NT>(di, ws, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, s);
}

// ---- TSM2L pass ------------------------------------------------------------------------------
template <typename T, int NT>
static int run_tsm2l_pass(const DevInfo& di, int64_t m, int64_t k, int w, const T* A, int64_t lda, const T* B,
                          int64_t ldb, T* C, int64_t ldc, bool c_is_zero, cudaStream_t s) {
  constexpr int THREADS = 256;
  constexpr int KCH = 8;
  const bool vec = aligned16(A) && aligned16(C) && (lda % Vec<T>::N == 0) && (ldc % Vec<T>::N == 0);
  LArgs<T> a;
  a.A = A;
  a.lda = lda;
  a.B = B;
  a.ldb = ldb;
  a.C = C;
  a.ldc = ldc;
  a.m = m;
  a.k = (int)k;
  a.w = w;
  a.c_is_zero = c_is_zero ? 1 : 0;
  const int rpt = vec ? Vec<T>::N : 1;
  const int64_t groups = (m + rpt - 1) / rpt;
  const void* kfn;
  int occ;
  if (vec) {
    auto kern = tsm2l_kernel<T, NT, THREADS, KCH, true>;
    occ = occupancy(kern, THREADS, 0);
    kfn = (const void*)kern;
  } else {
    auto kern = tsm2l_kernel<T, NT, THREADS, KCH, false>;
    occ = occupancy(kern, THREADS, 0);
    kfn = (const void*)kern;
  }
  int64_t grid = std::min<int64_t>((groups + THREADS - 1) / THREADS, (int64_t)di.sms * occ);
  grid = std::max<int64_t>(grid, 1);
  void* args[] = {&a};
  TSM2X_CUDA(cudaLaunchKernel(kfn, dim3((unsigned)grid), dim3(THREADS), args, 0, s));
  TSM2X_TRY(check_launch("tsm2l"));
  return TSM2X_OK;
}

// TSM2L split-n (tsm2l_splitn.cuh): S lanes per row group, warp-shuffle combine. A/B candidate
// (TSM2X_IMPL_TSM2L_SPLITN), never chosen automatically: profiles/splitn_r02.json.
template <typename T, int NT>
static int run_tsm2l_splitn_pass(const DevInfo& di, int64_t m, int64_t k, int w, const T* A, int64_t lda, const T* B,
                                 int64_t ldb, T* C, int64_t ldc, bool c_is_zero, cudaStream_t s) {
  if constexpr (NT < 4) {
    return run_tsm2l_pass<T, NT>(di, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, s);  // too few columns to split
  } else {
    constexpr int THREADS = 256, S = 4, KCH = 4;
    const bool vec = aligned16(A) && aligned16(C) && (lda % Vec<T>::N == 0) && (ldc % Vec<T>::N == 0);
    if (!vec) return run_tsm2l_pass<T, NT>(di, m, k, w, A, lda, B, ldb, C, ldc, c_is_zero, s);
    LArgs<T> a;
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.C = C;
    a.ldc = ldc;
    a.m = m;
    a.k = (int)k;
    a.w = w;
    a.c_is_zero = c_is_zero ? 1 : 0;
    auto kern = tsm2l_splitn_kernel<T, NT, S, THREADS, KCH>;
    const int occ = occupancy(kern, THREADS, 0);
    const int64_t groups = (m + Vec<T>::N - 1) / Vec<T>::N;
    int64_t grid = std::min<int64_t>((groups + THREADS / S - 1) / (THREADS / S), (int64_t)di.sms * occ);
    grid = std::max<int64_t>(grid, 1);
    kern<<<(unsigned)grid, THREADS, 0, s>>>(a);
    TSM2X_TRY(check_launch("tsm2l_splitn"));
    return TSM2X_OK;
  }
}

template <typename T>
__global__ void nonzero_check(const T* __restrict__ C, int64_t m, int64_t n, int64_t ldc, int* flag) {
  int64_t tot = m * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = i / m, r = i - j * m;
    if (C[r + j * ldc] != T(0)) {
      atomicOr(flag, 1);
      return;
    }
  }
}

// ---- one full device-resident call ----------------------------------------------------------
template <typename T>
static int run_passes(int variant, int64_t m, int64_t k, int64_t n, const T* A, int64_t lda, const T* B,
                      int64_t ldb, T* C, int64_t ldc, const tsm2x_params* params, uint32_t flags, int impl,
                      bool c_is_zero, const DevInfo& di, Workspace* ws, cudaStream_t s);
template <typename T>
static int run_device(int variant, int64_t m, int64_t k, int64_t n, const T* A, int64_t lda, const T* B, int64_t ldb,
                      T* C, int64_t ldc, const tsm2x_params* params, uint32_t flags, int impl, cudaStream_t s) {
  int dev;
  TSM2X_CUDA(cudaGetDevice(&dev));
  DevInfo di;
  TSM2X_TRY(device_info(dev, &di));
  if (lda < m || ldb < k || ldc < m)
    return fail(TSM2X_EINVAL, "leading dimensions too small: lda=%lld (m=%lld) ldb=%lld (k=%lld) ldc=%lld",
                (long long)lda, (long long)m, (long long)ldb, (long long)k, (long long)ldc);
  if (!A || !B || !C) return fail(TSM2X_EINVAL, "null matrix pointer");
  // C is written while A and B are read (A streamed, B gathered per stage): C must not overlap
  // either (the reference's Matrix inputs are distinct immutable arrays)
  {
    auto span = [](const void* p, int64_t rows, int64_t cols, int64_t ld) {
      const uintptr_t b = reinterpret_cast<uintptr_t>(p);
      return std::make_pair(b, b + (uintptr_t)(((cols - 1) * ld + rows) * (int64_t)sizeof(T)));
    };
    const auto c = span(C, m, n, ldc), a = span(A, m, k, lda), b = span(B, k, n, ldb);
    if ((c.first < a.second && a.first < c.second) || (c.first < b.second && b.first < c.second))
      return fail(TSM2X_EINVAL, "C overlaps A or B in memory: C is written while A and B are read");
  }
  Workspace* ws = workspace_for(dev, s);
  std::lock_guard<std::mutex> lk(ws->mu);
  bool c_is_zero = (flags & TSM2X_FLAG_C_IS_ZERO) != 0;
  if (variant == TSM2X_L_OPT2 && (flags & TSM2X_FLAG_CHECK_ZERO_C) && !c_is_zero) {
    TSM2X_TRY(ws_reserve(ws, 0, 0, s));
    TSM2X_CUDA(cudaMemsetAsync(ws->flag, 0, sizeof(int), s));
    nonzero_check<T><<<di.sms * 4, 256, 0, s>>>(C, m, n, ldc, ws->flag);
    TSM2X_TRY(check_launch("nonzero_check"));
    int h = 0;
    TSM2X_CUDA(cudaMemcpyAsync(&h, ws->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    TSM2X_CUDA(cudaStreamSynchronize(s));
    if (h) return fail(TSM2X_EINVAL, "L_OPT2 stores partial sums to C and requires a zeroed C");
    c_is_zero = true;
  }
  // tsm2x_set_kernel_events: the two events bracket the whole call — its first launch (prep_dyn
  // when there is one) to its last (tsm2_finalize for fp32 split passes) — so they sit outside
  // the programmatic-dependent-launch chain between those kernels instead of cutting it
  const cudaEvent_t ev0 = t_ev_start, ev1 = t_ev_stop;
  t_ev_start = t_ev_stop = nullptr;
  const bool timed = ev0 && ev1;
  if (timed) TSM2X_CUDA(record_kernel_event(ev0, s));
  TSM2X_TRY(run_passes<T>(variant, m, k, n, A, lda, B, ldb, C, ldc, params, flags, impl, c_is_zero, di, ws, s));
  if (timed) TSM2X_CUDA(record_kernel_event(ev1, s));
  return TSM2X_OK;
}

template <typename T>
static int run_passes(int variant, int64_t m, int64_t k, int64_t n, const T* A, int64_t lda, const T* B,
                      int64_t ldb, T* C, int64_t ldc, const tsm2x_params* params, uint32_t flags, int impl,
                      bool c_is_zero, const DevInfo& di, Workspace* ws, cudaStream_t s) {
  if (impl == TSM2X_IMPL_ABLATION) {
    if (variant > TSM2X_V2) impl = TSM2X_IMPL_AUTO;
    else return run_ablation<T>(variant, m, k, n, A, lda, B, ldb, C, ldc, params, c_is_zero, s);
  }
  const bool determ = (flags & TSM2X_FLAG_DETERMINISTIC) != 0;
  // the TMA stream kernel also covers TSM2L shapes (single-chunk row blocks); the LDG TSM2L
  // kernel is the fallback for layouts TMA cannot describe, or on request
  const bool tma_layout = aligned16(A) && ((lda * (int64_t)sizeof(T)) % 16 == 0);
  const bool splitn = impl == TSM2X_IMPL_TSM2L_SPLITN;
  const bool use_l = (impl == TSM2X_IMPL_TSM2L) || splitn || (impl == TSM2X_IMPL_AUTO && k <= TSM2L_KMAX && !tma_layout);
  if (use_l && k > TSM2L_KMAX) return fail(TSM2X_EINVAL, "TSM2L kernel needs k <= %d, got %lld", TSM2L_KMAX, (long long)k);
  for (int64_t p = 0; p < n; p += 16) {
    const int w = (int)std::min<int64_t>(16, n - p);
    int nt = nt_for(w);
    if (sizeof(T) == 8 && nt == 4 && !use_l && tma_layout && (impl == TSM2X_IMPL_AUTO || impl == TSM2X_IMPL_STREAM_TMA) &&
        n4_on_dmma(current_tuning()))
      nt = 8;
    const T* Bp = B + p * ldb;
    T* Cp = C + p * ldc;
    int rc;
#define TSM2X_PASS(NTV)                                                                                     \
  case NTV:                                                                                                 \
    rc = splitn  ? run_tsm2l_splitn_pass<T, NTV>(di, m, k, w, A, lda, Bp, ldb, Cp, ldc, c_is_zero, s)        \
         : use_l ? run_tsm2l_pass<T, NTV>(di, m, k, w, A, lda, Bp, ldb, Cp, ldc, c_is_zero, s)                \
               : run_tsm2r_pass<T, NTV>(di, ws, impl, m, k, w, A, lda, Bp, ldb, Cp, ldc, c_is_zero, determ, s); \
    break;
    switch (nt) {
      TSM2X_PASS(1)
      TSM2X_PASS(2)
      TSM2X_PASS(4)
      TSM2X_PASS(8)
      TSM2X_PASS(16)
      default: return fail(TSM2X_EUNSUPPORTED, "bad pass width");
    }
#undef TSM2X_PASS
    TSM2X_TRY(rc);
  }
  return TSM2X_OK;
}

static int run_device_any(int variant, int precision, int64_t m, int64_t k, int64_t n, const void* A, int64_t lda,
                          const void* B, int64_t ldb, void* C, int64_t ldc, const tsm2x_params* p, uint32_t flags,
                          int impl, cudaStream_t s) {
  if (precision == TSM2X_DOUBLE)
    return run_device<double>(variant, m, k, n, (const double*)A, lda, (const double*)B, ldb, (double*)C, ldc, p, flags,
                              impl, s);
  return run_device<float>(variant, m, k, n, (const float*)A, lda, (const float*)B, ldb, (float*)C, ldc, p, flags,
                           impl, s);
}

// ------------------------------------------------------------------------------------------
// host-buffer path: H2D of A pipelined with the kernels.
//   TSM2R (k > TSM2L_KMAX): column slabs of A; kernel j computes C += A[:, slab j] * B[slab j, :]
//   TSM2L: row slabs of A and C; H2D (A, C) / kernel / D2H (C) on three streams.
struct PinnedPool {
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> bufs;
};
static PinnedPool g_pinned;

static bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// host threads for the pageable staging copies and the zero-C scan
// Persistent host worker pool for the host path's parallel copies and scans: a pageable 7.55 GB
// A is staged as ~240 slabs of 32 MB, and spawning + joining 15 threads per slab (~0.3 ms) cost as
// much as the copy itself. One parallel region at a time; a caller that finds the pool busy
// (another device's host thread, tsm2x_run_host_multi) runs its region on fresh threads. The
// pool is never destroyed (its workers are detached and live until the process exits).
class HostPool {
 public:
  static HostPool& get() {
    static std::once_flag once;
    std::call_once(once, [] {
      instance() = new HostPool();
      // a forked child has none of the parent's workers (and may inherit a locked mutex): it
      // starts from a fresh pool (the old one is leaked)
      pthread_atfork(nullptr, nullptr, [] { instance() = new HostPool(); });
    });
    return *instance();
  }
  // fn(t) for t in [0, nt): t = 0 on the calling thread, the others on the pool's workers
  void run(unsigned nt, const std::function<void(unsigned)>& fn) {
    std::unique_lock<std::mutex> busy(region_mu_, std::try_to_lock);
    if (!busy.owns_lock() || nt > kMax) {
      std::vector<std::thread> th;
      for (unsigned t = 1; t < nt; ++t) th.emplace_back(fn, t);
      fn(0);
      for (auto& x : th) x.join();
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      while (workers_ + 1 < nt) {
        std::thread(&HostPool::worker, this, workers_ + 1).detach();
        ++workers_;
      }
      fn_ = &fn;
      nt_ = nt;
      pending_ = nt - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  static constexpr unsigned kMax = 64;
  static HostPool*& instance() {
    static HostPool* p = nullptr;
    return p;
  }
  void worker(unsigned id) {
    unsigned long long seen = 0;
    {
      std::lock_guard<std::mutex> lk(mu_);
      seen = gen_ - 1;  // a region may already be waiting for this new worker
    }
    for (;;) {
      const std::function<void(unsigned)>* fn;
      unsigned nt;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        fn = fn_;
        nt = nt_;
      }
      if (fn && id < nt) {
        (*fn)(id);
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::mutex region_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(unsigned)>* fn_ = nullptr;
  unsigned nt_ = 0, pending_ = 0, workers_ = 0;
  unsigned long long gen_ = 0;
};

static unsigned host_threads(size_t bytes) {
  if (bytes < (8u << 20)) return 1;
  return std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
}

// reference kernels.py:366-368 (_require_zero_c): L_OPT2 requires an all-zero C — a parallel scan
// of the host copy with early exit, before any device work (so a CPU-only caller gets the
// ValueError too)
template <typename T>
static bool host_all_zero(const T* C, int64_t m, int64_t n, int64_t ldc) {
  const unsigned nt = host_threads((size_t)m * n * sizeof(T));
  std::atomic<bool> nonzero{false};
  auto scan = [&](unsigned t) {
    const int64_t j0 = n * t / nt, j1 = n * (t + 1) / nt;
    if (n >= nt || nt == 1) {
      for (int64_t j = j0; j < j1 && !nonzero.load(std::memory_order_relaxed); ++j)
        for (int64_t i = 0; i < m; ++i)
          if (C[i + j * ldc] != T(0)) {
            nonzero = true;
            return;
          }
    } else {  // few columns: split the rows instead
      const int64_t i0 = m * t / nt, i1 = m * (t + 1) / nt;
      for (int64_t j = 0; j < n && !nonzero.load(std::memory_order_relaxed); ++j)
        for (int64_t i = i0; i < i1; ++i)
          if (C[i + j * ldc] != T(0)) {
            nonzero = true;
            return;
          }
    }
  };
  HostPool::get().run(nt, scan);
  return !nonzero.load();
}

// parallel memcpy (pageable -> pinned staging); 2-D with pitches
static void par_copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height) {
  const size_t total = width * height;
  const unsigned nt = host_threads(total);
  auto work = [&](unsigned t) {
    if (width == dpitch && width == spitch) {
      size_t lo = total * t / nt, hi = total * (t + 1) / nt;
      memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
    } else {
      size_t lo = height * t / nt, hi = height * (t + 1) / nt;
      for (size_t r = lo; r < hi; ++r)
        memcpy(static_cast<char*>(dst) + r * dpitch, static_cast<const char*>(src) + r * spitch, width);
    }
  };
  if (nt == 1) {
    work(0);
    return;
  }
  HostPool::get().run(nt, work);
}

// Per-device resources of the host path, kept across calls (allocation and stream creation
// would otherwise cost more than the copies): three streams, named device / pinned buffers that
// only grow, and an event pool. One call at a time per device (mutex).
struct HostCtx {
  std::mutex mu;
  int dev = -1;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  std::map<std::string, std::pair<void*, size_t>> dbufs, hbufs;
  std::vector<cudaEvent_t> events;
  size_t ev_next = 0;
  int init(int device) {
    if (h2d) return TSM2X_OK;
    dev = device;
    TSM2X_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    TSM2X_CUDA(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking));
    TSM2X_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    return TSM2X_OK;
  }
  int dbuf(const std::string& name, size_t bytes, void** p) {
    auto& e = dbufs[name];
    if (e.second < bytes) {
      if (e.first) TSM2X_CUDA(cudaFree(e.first));
      e = {nullptr, 0};
      if (cudaMalloc(&e.first, bytes) != cudaSuccess) {
        cudaGetLastError();
        e.first = nullptr;
        return fail(TSM2X_ENOMEM, "device allocation of %zu bytes failed", bytes);
      }
      e.second = bytes;
    }
    *p = e.first;
    return TSM2X_OK;
  }
  int hbuf(const std::string& name, size_t bytes, void** p) {
    auto& e = hbufs[name];
    if (e.second < bytes) {
      if (e.first) TSM2X_CUDA(cudaFreeHost(e.first));
      e = {nullptr, 0};
      if (cudaMallocHost(&e.first, bytes) != cudaSuccess) {
        cudaGetLastError();
        e.first = nullptr;
        return fail(TSM2X_ENOMEM, "pinned allocation of %zu bytes failed", bytes);
      }
      e.second = bytes;
    }
    *p = e.first;
    return TSM2X_OK;
  }
  int event(cudaEvent_t* e) {
    if (ev_next == events.size()) {
      cudaEvent_t x;
      TSM2X_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      events.push_back(x);
    }
    *e = events[ev_next++];
    return TSM2X_OK;
  }
  void begin() { ev_next = 0; }
  // frees every cached buffer, event and stream (tsm2x_release_cached); the context re-initialises
  // on its next use
  void release() {
    drain();
    for (auto& e : dbufs)
      if (e.second.first) cudaFree(e.second.first);
    for (auto& e : hbufs)
      if (e.second.first) cudaFreeHost(e.second.first);
    dbufs.clear();
    hbufs.clear();
    for (auto e : events) cudaEventDestroy(e);
    events.clear();
    ev_next = 0;
    for (cudaStream_t* st : {&h2d, &comp, &d2h})
      if (*st) {
        cudaStreamDestroy(*st);
        *st = nullptr;
      }
  }
  void drain() {
    cudaStreamSynchronize(h2d);
    cudaStreamSynchronize(comp);
    cudaStreamSynchronize(d2h);
  }
};
static std::mutex g_host_mu;
static std::map<int, std::unique_ptr<HostCtx>> g_host;

static HostCtx* host_ctx(int dev) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  auto& slot = g_host[dev];
  if (!slot) slot.reset(new HostCtx());
  return slot.get();
}

// copy a 2-D host block (width bytes x height rows, host pitch) to the device, via pinned
// staging (filled by host threads) when the source is pageable. Ordered on `st`.
struct Stager {
  HostCtx* hc = nullptr;
  bool pinned_src = true;
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2];
  bool used[2] = {false, false};
  int next = 0;
  int init(HostCtx* h, bool pinned, size_t max_block, const char* tag) {
    hc = h;
    pinned_src = pinned;
    if (pinned) return TSM2X_OK;
    for (int i = 0; i < 2; ++i) {
      TSM2X_TRY(hc->hbuf(std::string(tag) + char('0' + i), max_block, &stage[i]));
      TSM2X_TRY(hc->event(&done[i]));
    }
    return TSM2X_OK;
  }
  int copy(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height, cudaStream_t st) {
    if (pinned_src) {
      TSM2X_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, st));
      return TSM2X_OK;
    }
    const int i = next;
    next ^= 1;
    if (used[i]) TSM2X_CUDA(cudaEventSynchronize(done[i]));  // staging buffer i free again
    par_copy2d(stage[i], width, src, spitch, width, height);
    TSM2X_CUDA(cudaMemcpy2DAsync(dst, dpitch, stage[i], width, width, height, cudaMemcpyHostToDevice, st));
    TSM2X_CUDA(cudaEventRecord(done[i], st));
    used[i] = true;
    return TSM2X_OK;
  }
};

template <typename T>
static int run_host_t(int variant, int64_t m, int64_t k, int64_t n, const T* A, int64_t lda, const T* B, int64_t ldb,
                      const T* Cin, T* Cout, int64_t ldc, const tsm2x_params* params, uint32_t flags, int device) {
  TSM2X_CUDA(cudaSetDevice(device));
  DevInfo di;
  TSM2X_TRY(device_info(device, &di));
  if (lda < m || ldb < k || ldc < m) return fail(TSM2X_EINVAL, "leading dimensions too small");
  bool c_is_zero = (flags & TSM2X_FLAG_C_IS_ZERO) != 0;
  if (variant == TSM2X_L_OPT2) c_is_zero = true;  // tsm2x_run_host checked C == 0 on the host
  HostCtx* hc = host_ctx(device);
  std::lock_guard<std::mutex> lk(hc->mu);
  TSM2X_TRY(hc->init(device));
  hc->begin();
  struct Drain {
    HostCtx* h;
    ~Drain() { h->drain(); }
  } drain_on_exit{hc};
  const size_t eb = sizeof(T);
  const int64_t ldd = (int64_t)align_up((size_t)m, 32);  // padded device leading dimension
  const bool pinnedA = is_pinned(A);
  const bool use_l = k <= TSM2L_KMAX;
  const int dev_variant = (variant == TSM2X_L_OPT2) ? TSM2X_L_OPT1 : variant;  // zero-C handled by flags

  T* dB;
  TSM2X_TRY(hc->dbuf("B", (size_t)k * n * eb, (void**)&dB));
  TSM2X_CUDA(cudaMemcpy2DAsync(dB, k * eb, B, ldb * eb, k * eb, n, cudaMemcpyHostToDevice, hc->h2d));
  cudaEvent_t b_ready;
  TSM2X_TRY(hc->event(&b_ready));
  TSM2X_CUDA(cudaEventRecord(b_ready, hc->h2d));
  TSM2X_CUDA(cudaStreamWaitEvent(hc->comp, b_ready, 0));

  // pinned sources: 256 MB slabs (few, long DMAs); pageable: 32 MB, so the host threads' copy of
  // slab j+1 into pinned staging overlaps the DMA of slab j even for a 134 MB A
  const size_t slab_target = pinnedA ? (size_t)256 << 20 : (size_t)32 << 20;
  if (!use_l) {
    // ---- TSM2R: column slabs of A stream in while earlier slabs are multiplied; C stays on
    // the device (C += A[:, slab] * B[slab, :] per slab)
    T* dC;
    TSM2X_TRY(hc->dbuf("C", (size_t)ldd * n * eb, (void**)&dC));
    if (!c_is_zero) {
      TSM2X_CUDA(cudaMemcpy2DAsync(dC, ldd * eb, Cin, ldc * eb, m * eb, n, cudaMemcpyHostToDevice, hc->h2d));
      TSM2X_CUDA(cudaEventRecord(b_ready, hc->h2d));
      TSM2X_CUDA(cudaStreamWaitEvent(hc->comp, b_ready, 0));
    }
    int64_t sw = std::max<int64_t>(1, (int64_t)(slab_target / ((size_t)ldd * eb)));
    sw = std::min<int64_t>(sw, k);
    const int64_t nslab = (k + sw - 1) / sw;
    const int nbuf = (int)std::min<int64_t>(3, nslab);
    T* dA[3];
    cudaEvent_t loaded[3], consumed[3];
    for (int i = 0; i < nbuf; ++i) {
      TSM2X_TRY(hc->dbuf(std::string("A") + char('0' + i), (size_t)ldd * sw * eb, (void**)&dA[i]));
      TSM2X_TRY(hc->event(&loaded[i]));
      TSM2X_TRY(hc->event(&consumed[i]));
    }
    Stager stg;
    TSM2X_TRY(stg.init(hc, pinnedA, (size_t)m * eb * sw, "stageA"));
    for (int64_t j = 0; j < nslab; ++j) {
      const int b = (int)(j % nbuf);
      const int64_t c0 = j * sw, cw = std::min(sw, k - c0);
      if (j >= nbuf) TSM2X_CUDA(cudaStreamWaitEvent(hc->h2d, consumed[b], 0));
      TSM2X_TRY(stg.copy(dA[b], ldd * eb, A + c0 * lda, lda * eb, m * eb, cw, hc->h2d));
      TSM2X_CUDA(cudaEventRecord(loaded[b], hc->h2d));
      TSM2X_CUDA(cudaStreamWaitEvent(hc->comp, loaded[b], 0));
      const uint32_t f = ((c_is_zero && j == 0) ? TSM2X_FLAG_C_IS_ZERO : 0) | (flags & TSM2X_FLAG_DETERMINISTIC);
      TSM2X_TRY(run_device<T>(dev_variant, m, cw, n, dA[b], ldd, dB + c0, k, dC, ldd, params, f, TSM2X_IMPL_AUTO,
                              hc->comp));
      TSM2X_CUDA(cudaEventRecord(consumed[b], hc->comp));
    }
    TSM2X_CUDA(cudaMemcpy2DAsync(Cout, ldc * eb, dC, ldd * eb, m * eb, n, cudaMemcpyDeviceToHost, hc->comp));
    TSM2X_CUDA(cudaStreamSynchronize(hc->comp));
    return TSM2X_OK;
  }

  // ---- TSM2L: row slabs of A (and C); H2D / kernel / D2H on three streams
  const size_t row_bytes = (size_t)(k + (c_is_zero ? 0 : n)) * eb;
  int64_t rs = std::max<int64_t>(1024, (int64_t)(slab_target / std::max<size_t>(row_bytes, 1)));
  rs = (int64_t)align_up((size_t)std::min<int64_t>(rs, m), 32);
  const int64_t nslab = (m + rs - 1) / rs;
  const int nbuf = (int)std::min<int64_t>(3, nslab);
  T *dA[3], *dC[3];
  cudaEvent_t loaded[3], computed[3], drained[3];
  for (int i = 0; i < nbuf; ++i) {
    TSM2X_TRY(hc->dbuf(std::string("LA") + char('0' + i), (size_t)rs * k * eb, (void**)&dA[i]));
    TSM2X_TRY(hc->dbuf(std::string("LC") + char('0' + i), (size_t)rs * n * eb, (void**)&dC[i]));
    TSM2X_TRY(hc->event(&loaded[i]));
    TSM2X_TRY(hc->event(&computed[i]));
    TSM2X_TRY(hc->event(&drained[i]));
  }
  Stager stgA, stgC;
  TSM2X_TRY(stgA.init(hc, pinnedA, (size_t)rs * k * eb, "stageLA"));
  if (!c_is_zero) TSM2X_TRY(stgC.init(hc, is_pinned(Cin), (size_t)rs * n * eb, "stageLC"));
  const bool pinnedOut = is_pinned(Cout);
  T* out_stage[2] = {nullptr, nullptr};
  cudaEvent_t out_done[2];
  if (!pinnedOut) {
    for (int i = 0; i < 2; ++i) {
      TSM2X_TRY(hc->hbuf(std::string("outL") + char('0' + i), (size_t)rs * n * eb, (void**)&out_stage[i]));
      TSM2X_TRY(hc->event(&out_done[i]));
    }
  }
  // pageable output: slab j's staged result is copied out while slab j+1 is in flight
  int64_t pend_r0 = -1, pend_rw = 0;
  int pend_i = 0;
  auto flush_out = [&]() -> int {
    if (pend_r0 < 0) return TSM2X_OK;
    TSM2X_CUDA(cudaEventSynchronize(out_done[pend_i]));
    par_copy2d(Cout + pend_r0, ldc * eb, out_stage[pend_i], pend_rw * eb, pend_rw * eb, n);
    pend_r0 = -1;
    return TSM2X_OK;
  };
  for (int64_t j = 0; j < nslab; ++j) {
    const int b = (int)(j % nbuf);
    const int64_t r0 = j * rs, rw = std::min(rs, m - r0);
    if (j >= nbuf) TSM2X_CUDA(cudaStreamWaitEvent(hc->h2d, drained[b], 0));
    TSM2X_TRY(stgA.copy(dA[b], rs * eb, A + r0, lda * eb, rw * eb, k, hc->h2d));
    if (!c_is_zero) TSM2X_TRY(stgC.copy(dC[b], rs * eb, Cin + r0, ldc * eb, rw * eb, n, hc->h2d));
    TSM2X_CUDA(cudaEventRecord(loaded[b], hc->h2d));
    TSM2X_CUDA(cudaStreamWaitEvent(hc->comp, loaded[b], 0));
    TSM2X_TRY(run_device<T>(dev_variant, rw, k, n, dA[b], rs, dB, k, dC[b], rs, params,
                            (c_is_zero ? TSM2X_FLAG_C_IS_ZERO : 0) | (flags & TSM2X_FLAG_DETERMINISTIC),
                            TSM2X_IMPL_AUTO, hc->comp));
    TSM2X_CUDA(cudaEventRecord(computed[b], hc->comp));
    TSM2X_CUDA(cudaStreamWaitEvent(hc->d2h, computed[b], 0));
    if (pinnedOut) {
      TSM2X_CUDA(cudaMemcpy2DAsync(Cout + r0, ldc * eb, dC[b], rs * eb, rw * eb, n, cudaMemcpyDeviceToHost, hc->d2h));
      TSM2X_CUDA(cudaEventRecord(drained[b], hc->d2h));
    } else {
      const int oi = (int)(j % 2);
      TSM2X_CUDA(cudaMemcpy2DAsync(out_stage[oi], rw * eb, dC[b], rs * eb, rw * eb, n, cudaMemcpyDeviceToHost, hc->d2h));
      TSM2X_CUDA(cudaEventRecord(drained[b], hc->d2h));
      TSM2X_CUDA(cudaEventRecord(out_done[oi], hc->d2h));
      TSM2X_TRY(flush_out());
      pend_r0 = r0;
      pend_rw = rw;
      pend_i = oi;
    }
  }
  TSM2X_TRY(flush_out());
  TSM2X_CUDA(cudaStreamSynchronize(hc->d2h));
  TSM2X_CUDA(cudaStreamSynchronize(hc->comp));
  return TSM2X_OK;
}

// counter-based uniform generator (see tsm2x.h tsm2x_fill_uniform)
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
template <typename T>
__global__ void fill_uniform(T* p, int64_t rows, int64_t cols, int64_t ld, int64_t r0, int64_t c0, uint64_t seed) {
  const int64_t tot = rows * cols;
  const uint64_t base = seed * 0x9E3779B97F4A7C15ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / rows, r = i - j * rows;
    const uint64_t key = ((uint64_t)(c0 + j) << 32) | (uint64_t)(r0 + r);
    const double u = (double)(splitmix64(base + key) >> 11) * 0x1.0p-53;
    p[r + j * ld] = (T)u;
  }
}

// tsm2x_run_multi: per-(device, stream) copies of B and peer access between the shard devices
struct BCopy {
  void* p = nullptr;
  size_t cap = 0;
};
static std::mutex g_bcopy_mu;
static std::map<std::pair<int, cudaStream_t>, BCopy> g_bcopy;

static int bcopy_reserve(int dev, cudaStream_t s, size_t bytes, void** out) {
  std::lock_guard<std::mutex> lk(g_bcopy_mu);
  BCopy& b = g_bcopy[{dev, s}];
  if (bytes > b.cap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TSM2X_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(TSM2X_EUNSUPPORTED, "B copy buffer must grow during a CUDA graph capture: make one eager call first");
    if (b.p) TSM2X_CUDA(cudaFreeAsync(b.p, s));
    b.p = nullptr;
    b.cap = 0;
    if (cudaMallocAsync(&b.p, bytes, s) != cudaSuccess) {
      cudaGetLastError();
      return fail(TSM2X_ENOMEM, "B copy allocation of %zu bytes failed", bytes);
    }
    b.cap = bytes;
  }
  *out = b.p;
  return TSM2X_OK;
}

static void bcopy_release(int device) {
  std::lock_guard<std::mutex> lk(g_bcopy_mu);
  for (auto it = g_bcopy.begin(); it != g_bcopy.end();) {
    if (device < 0 || it->first.first == device) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(it->first.first);
      cudaDeviceSynchronize();
      if (it->second.p) cudaFreeAsync(it->second.p, 0);  // stream-ordered allocation (bcopy_reserve)
      cudaSetDevice(prev);
      it = g_bcopy.erase(it);
    } else {
      ++it;
    }
  }
}

// enable access from `dev` (current device) to `peer` once; devices without a peer path fall back
// to the driver's staged copy (cudaMemcpy3DPeerAsync handles both)
static int peer_enable(int dev, int peer) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, bool> done;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, peer);
  if (done.count(key)) return TSM2X_OK;
  int can = 0;
  TSM2X_CUDA(cudaDeviceCanAccessPeer(&can, dev, peer));
  if (can) {
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return fail(TSM2X_ECUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", dev, peer, cudaGetErrorString(e));
    cudaGetLastError();
  }
  done[key] = true;
  return TSM2X_OK;
}

}  // namespace tsm2x

// ============================================================================================
// C ABI
using namespace tsm2x;

extern "C" {

int tsm2x_validate(int variant, int64_t m, int64_t k, int64_t n, const tsm2x_params* params) {
  return validate(variant, TSM2X_DOUBLE, m, k, n, params);
}

int tsm2x_run_ex(int variant, int precision, int64_t m, int64_t k, int64_t n, const void* A, int64_t lda,
                 const void* B, int64_t ldb, void* C, int64_t ldc, const tsm2x_params* params, uint32_t flags,
                 int impl, void* stream) {
  TSM2X_TRY(validate(variant, precision, m, k, n, params));
  if (impl < TSM2X_IMPL_AUTO || impl > TSM2X_IMPL_TSM2L_SPLITN) return fail(TSM2X_EINVAL, "unknown impl %d", impl);
  return run_device_any(variant, precision, m, k, n, A, lda, B, ldb, C, ldc, params, flags, impl,
                        reinterpret_cast<cudaStream_t>(stream));
}

int tsm2x_run(int variant, int precision, int64_t m, int64_t k, int64_t n, const void* A, int64_t lda, const void* B,
              int64_t ldb, void* C, int64_t ldc, const tsm2x_params* params, uint32_t flags, void* stream) {
  return tsm2x_run_ex(variant, precision, m, k, n, A, lda, B, ldb, C, ldc, params, flags, TSM2X_IMPL_AUTO, stream);
}

int tsm2x_run_host(int variant, int precision, int64_t m, int64_t k, int64_t n, const void* A, int64_t lda,
                   const void* B, int64_t ldb, const void* C_in, void* C_out, int64_t ldc,
                   const tsm2x_params* params, uint32_t flags, int device) {
  TSM2X_TRY(validate(variant, precision, m, k, n, params));
  if (!A || !B || !C_out || (!C_in && !(flags & TSM2X_FLAG_C_IS_ZERO))) return fail(TSM2X_EINVAL, "null host pointer");
  if (ldc < m) return fail(TSM2X_EINVAL, "leading dimensions too small");
  if (variant == TSM2X_L_OPT2 && !(flags & TSM2X_FLAG_C_IS_ZERO)) {
    const bool zero = precision == TSM2X_DOUBLE ? host_all_zero((const double*)C_in, m, n, ldc)
                                                : host_all_zero((const float*)C_in, m, n, ldc);
    if (!zero) return fail(TSM2X_EINVAL, "L_OPT2 stores partial sums to C and requires a zeroed C");
    flags |= TSM2X_FLAG_C_IS_ZERO;
  }
  if (precision == TSM2X_DOUBLE)
    return run_host_t<double>(variant, m, k, n, (const double*)A, lda, (const double*)B, ldb, (const double*)C_in,
                              (double*)C_out, ldc, params, flags, device);
  return run_host_t<float>(variant, m, k, n, (const float*)A, lda, (const float*)B, ldb, (const float*)C_in,
                           (float*)C_out, ldc, params, flags, device);
}

int tsm2x_run_host_multi(int variant, int precision, int64_t m, int64_t k, int64_t n, const void* A, int64_t lda,
                         const void* B, int64_t ldb, const void* C_in, void* C_out, int64_t ldc,
                         const tsm2x_params* params, uint32_t flags, int ndev, const int* devices) {
  TSM2X_TRY(validate(variant, precision, m, k, n, params));
  if (ndev < 1 || !devices) return fail(TSM2X_EINVAL, "need at least one device");
  if (!A || !B || !C_out || (!C_in && !(flags & TSM2X_FLAG_C_IS_ZERO))) return fail(TSM2X_EINVAL, "null host pointer");
  const size_t eb = precision == TSM2X_DOUBLE ? 8 : 4;
  // contiguous row shards in 32-row units (paper_2002_03258_b200.multi.row_partition)
  const int64_t blocks = (m + 31) / 32;
  std::vector<int> rc(ndev, TSM2X_OK);
  std::vector<std::string> msg(ndev);
  std::vector<std::thread> th;
  for (int d = 0; d < ndev; ++d) {
    const int64_t r0 = std::min<int64_t>(m, blocks * d / ndev * 32);
    const int64_t r1 = std::min<int64_t>(m, blocks * (d + 1) / ndev * 32);
    if (r1 <= r0) continue;
    th.emplace_back([=, &rc, &msg] {
      const char* a = static_cast<const char*>(A) + r0 * eb;
      const char* ci = C_in ? static_cast<const char*>(C_in) + r0 * eb : nullptr;
      char* co = static_cast<char*>(C_out) + r0 * eb;
      rc[d] = tsm2x_run_host(variant, precision, r1 - r0, k, n, a, lda, B, ldb, ci, co, ldc, params, flags,
                             devices[d]);
      if (rc[d] != TSM2X_OK) msg[d] = t_err;
    });
  }
  for (auto& x : th) x.join();
  for (int d = 0; d < ndev; ++d)
    if (rc[d] != TSM2X_OK) return fail(rc[d], "device %d: %s", devices[d], msg[d].c_str());
  return TSM2X_OK;
}

void tsm2x_row_range(int64_t m, int ndev, int g, int64_t* r0, int64_t* r1) {
  // contiguous row shards in 32-row units (paper_2002_03258_b200.multi.row_partition)
  const int64_t blocks = (m + 31) / 32;
  if (ndev < 1 || g < 0 || g >= ndev || m < 0) {
    *r0 = *r1 = 0;
    return;
  }
  *r0 = std::min<int64_t>(m, blocks * g / ndev * 32);
  *r1 = std::min<int64_t>(m, blocks * (g + 1) / ndev * 32);
}

int tsm2x_run_multi(int variant, int precision, int64_t m, int64_t k, int64_t n, int ndev, const int* devices,
                    const void* const* A, const int64_t* lda, const void* B, int64_t ldb, void* const* C,
                    const int64_t* ldc, const tsm2x_params* params, uint32_t flags, void* const* streams) {
  TSM2X_TRY(validate(variant, precision, m, k, n, params));
  if (ndev < 1 || !devices) return fail(TSM2X_EINVAL, "need at least one device");
  if (!A || !lda || !B || !C || !ldc) return fail(TSM2X_EINVAL, "null shard array or pointer");
  const size_t eb = precision == TSM2X_DOUBLE ? 8 : 4;
  int prev = 0;
  TSM2X_CUDA(cudaGetDevice(&prev));
  struct Restore {
    int dev;
    ~Restore() { cudaSetDevice(dev); }
  } restore{prev};
  auto stream_of = [&](int g) { return streams ? reinterpret_cast<cudaStream_t>(streams[g]) : (cudaStream_t)0; };
  // B is ready on devices[0]'s stream: every shard's stream waits for it before reading or copying it
  TSM2X_CUDA(cudaSetDevice(devices[0]));
  cudaEvent_t b_ready;
  TSM2X_CUDA(cudaEventCreateWithFlags(&b_ready, cudaEventDisableTiming));
  struct EvDestroy {
    cudaEvent_t e;
    ~EvDestroy() { cudaEventDestroy(e); }  // safe once enqueued: released when the waits complete
  } evd{b_ready};
  TSM2X_CUDA(cudaEventRecord(b_ready, stream_of(0)));
  for (int g = 0; g < ndev; ++g) {
    int64_t r0, r1;
    tsm2x_row_range(m, ndev, g, &r0, &r1);
    if (r1 <= r0) continue;
    const int dev = devices[g];
    cudaStream_t sg = stream_of(g);
    TSM2X_CUDA(cudaSetDevice(dev));
    TSM2X_CUDA(cudaStreamWaitEvent(sg, b_ready, 0));
    const void* Bg = B;
    int64_t ldbg = ldb;
    if (dev != devices[0]) {
      // B (k x n) to this device once per call, over NVLink when the devices are peers (the 4 MB
      // at configs[4] take microseconds); the copy lives in a per-(device, stream) buffer, so
      // stream order makes its reuse by the next call on this stream safe
      TSM2X_TRY(peer_enable(dev, devices[0]));
      void* dst = nullptr;
      TSM2X_TRY(bcopy_reserve(dev, sg, (size_t)k * n * eb, &dst));
      cudaMemcpy3DPeerParms cp = {};
      cp.srcPtr = make_cudaPitchedPtr(const_cast<void*>(B), (size_t)ldb * eb, (size_t)k * eb, (size_t)n);
      cp.srcDevice = devices[0];
      cp.dstPtr = make_cudaPitchedPtr(dst, (size_t)k * eb, (size_t)k * eb, (size_t)n);
      cp.dstDevice = dev;
      cp.extent = make_cudaExtent((size_t)k * eb, (size_t)n, 1);
      TSM2X_CUDA(cudaMemcpy3DPeerAsync(&cp, sg));
      Bg = dst;
      ldbg = k;
    }
    const int rc = run_device_any(variant, precision, r1 - r0, k, n, A[g], lda[g], Bg, ldbg, C[g], ldc[g], params,
                                  flags, TSM2X_IMPL_AUTO, sg);
    if (rc != TSM2X_OK) return fail(rc, "shard %d (device %d): %s", g, dev, t_err);
  }
  return TSM2X_OK;
}

int tsm2x_fill_uniform(int precision, int64_t rows, int64_t cols, void* ptr, int64_t ld, int64_t row_offset,
                       int64_t col_offset, uint64_t seed, void* stream) {
  if (rows < 1 || cols < 1 || ld < rows || !ptr || row_offset < 0 || col_offset < 0 ||
      row_offset + rows > (int64_t(1) << 32))
    return fail(TSM2X_EINVAL, "bad fill_uniform arguments");
  int dev;
  TSM2X_CUDA(cudaGetDevice(&dev));
  DevInfo di;
  TSM2X_TRY(device_info(dev, &di));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned grid = (unsigned)std::min<int64_t>((rows * cols + 255) / 256, (int64_t)di.sms * 16);
  if (precision == TSM2X_DOUBLE)
    fill_uniform<double><<<grid, 256, 0, s>>>((double*)ptr, rows, cols, ld, row_offset, col_offset, seed);
  else
    fill_uniform<float><<<grid, 256, 0, s>>>((float*)ptr, rows, cols, ld, row_offset, col_offset, seed);
  return check_launch("fill_uniform");
}

int tsm2x_set_tuning(const tsm2x_tuning* t) {
  Tuning nt;
  if (t) {
    if (t->consumer < 0 || t->consumer > 5 || t->small_kb < 0 || t->big_kb < 0 || t->tail_pct < 0 ||
        t->tail_pct > 100 || t->batch_kb < 0 || t->combine < 0 || t->combine > 3)
      return fail(TSM2X_EINVAL, "bad tuning values");
    nt.combine = t->combine;
    nt.consumer = t->consumer;
    nt.small_kb = t->small_kb;
    nt.big_kb = t->big_kb;
    nt.tail_pct = t->tail_pct;
    nt.batch_kb = t->batch_kb;
  }
  std::lock_guard<std::mutex> lk(g_tune_mu);
  g_tune = nt;
  return TSM2X_OK;
}

int tsm2x_get_tuning(tsm2x_tuning* out) {
  if (!out) return fail(TSM2X_EINVAL, "null output");
  const Tuning t = current_tuning();
  out->consumer = t.consumer;
  out->small_kb = t.small_kb;
  out->big_kb = t.big_kb;
  out->tail_pct = t.tail_pct;
  out->batch_kb = t.batch_kb;
  out->combine = t.combine;
  return TSM2X_OK;
}

int tsm2x_plan_for(int precision, int64_t m, int64_t k, int64_t n, int64_t lda, int a_aligned16, uint32_t flags,
                   int impl, tsm2x_plan* out) {
  if (!out) return fail(TSM2X_EINVAL, "null output");
  if (precision != TSM2X_SINGLE && precision != TSM2X_DOUBLE) return fail(TSM2X_EINVAL, "bad precision");
  if (m < 1 || k < 1 || n < 1 || lda < m) return fail(TSM2X_EINVAL, "bad dimensions");
  memset(out, 0, sizeof(*out));
  const size_t eb = precision == TSM2X_DOUBLE ? 8 : 4;
  const int w = (int)std::min<int64_t>(16, n);
  int nt = nt_for(w);
  out->cols_per_pass = nt;
  out->passes = (int)((n + 15) / 16);
  int sms = 148;
  int dev;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    DevInfo di;
    if (device_info(dev, &di) == TSM2X_OK) sms = di.sms;
  }
  cudaGetLastError();
  const bool tma_layout = a_aligned16 && ((lda * (int64_t)eb) % 16 == 0) && m < (int64_t(1) << 31);
  const bool determ = (flags & TSM2X_FLAG_DETERMINISTIC) != 0;
  if (impl == TSM2X_IMPL_TSM2L_SPLITN) {
    out->impl = TSM2X_IMPL_TSM2L_SPLITN;
    out->rows_per_block = 256 / 4 * (int)(16 / eb);  // 64 row groups of one 16-byte vector per CTA
    out->cols_per_pass = nt;
    return TSM2X_OK;
  }
  if (impl == TSM2X_IMPL_ABLATION || impl == TSM2X_IMPL_TSM2L ||
      (impl == TSM2X_IMPL_AUTO && k <= TSM2L_KMAX && !tma_layout)) {
    out->impl = impl == TSM2X_IMPL_ABLATION ? TSM2X_IMPL_ABLATION : TSM2X_IMPL_TSM2L;
    out->rows_per_block = 256 * (a_aligned16 ? (int)(16 / eb) : 1);
    return TSM2X_OK;
  }
  const bool tma = (impl == TSM2X_IMPL_AUTO || impl == TSM2X_IMPL_STREAM_TMA) && tma_layout;
  if (!tma) {
    out->impl = TSM2X_IMPL_STREAM_LDG;
    out->rows_per_block = 256 * (a_aligned16 && lda % (16 / eb) == 0 ? (int)(16 / eb) : 1);
    out->cols_per_stage = 32;
    out->deterministic = 1;
    return TSM2X_OK;
  }
  out->impl = TSM2X_IMPL_STREAM_TMA;
  if (eb == 8 && nt == 4 && n4_on_dmma(current_tuning())) out->cols_per_pass = nt = 8;  // as run_device
  const int R = 256 * (int)(16 / eb);
  out->rows_per_block = R;
  const bool stage64 = eb == 8 && (nt == 8 || nt == 16) && getenv("TSM2X_STAGE_KB") == nullptr;
  out->cols_per_stage = stage64 ? TmaCfg<double, 8, 2, 8, 65536>::KC : TmaCfg<double, 1>::KC;
  out->stages = stage64 ? TmaCfg<double, 8, 2, 8, 65536>::STAGES : TmaCfg<double, 1>::STAGES;
  const Tuning tu0 = current_tuning();
  if (tu0.combine == 3) {
    out->cols_per_stage = TmaCfg<double, 1>::KC;  // the static kernel keeps 32 KB stages
    out->stages = TmaCfg<double, 1>::STAGES;
    out->deterministic = 1;
    out->consumer = 1;
    const int64_t units = ((m + R - 1) / R) * ((k + 7) / 8);
    out->grid = std::min<int64_t>(units, sms);
    return TSM2X_OK;
  }
  const Tuning tu = current_tuning();
  Items it;
  int64_t G;
  if (eb == 4 && nt == 16 && !determ && tu.combine != 1 && pick_consumer_rt(4, nt, fp32_split(sms, m, k, nt), tu) == kTc &&
      !(f32_direct_call(m, k) && !(flags & TSM2X_FLAG_C_IS_ZERO) && tu.consumer != 4 && !env_forces_tc()) &&
      a_aligned16 && lda % 4 == 0 && lda >= (int64_t)align_up((size_t)m, 32) && k < (int64_t(1) << 31)) {
    // fp32 16-column passes on the tensor cores (run_tsm2r_tc32)
    out->rows_per_block = Tc32Cfg::R;
    out->cols_per_stage = Tc32Cfg::KC;
    out->stages = Tc32Cfg::STAGES;
    make_items(sms, m, k, eb, Tc32Cfg::R, Tc32Cfg::KC, nt, tu, &it, &G);
    out->grid = G;
    out->items = it.total;
    out->nbig = it.nbig;
    out->kbig = it.kbig;
    out->nsmall = it.nsmall;
    out->ksmall = it.ksmall;
    out->batch = it.batch;
    out->consumer = 1 + kTc;
    out->deterministic = it.nch() == 1 ? 1 : 0;
    return TSM2X_OK;
  }
  make_items(sms, m, k, eb, R, out->cols_per_stage, nt, tu, &it, &G);
  out->grid = G;
  out->items = it.total;
  out->nbig = it.nbig;
  out->kbig = it.kbig;
  out->nsmall = it.nsmall;
  out->ksmall = it.ksmall;
  out->batch = it.batch;
  out->consumer = 1 + pick_consumer_rt(eb, nt, it.nch() > 1, tu);
  if (out->consumer == 1 + kTc) out->consumer = 1 + (nt >= 2 ? kFfma2 : kFma);  // tc path not taken
  out->deterministic = (it.nch() == 1 || tu.combine == 1 || (tu.combine == 0 && determ)) ? 1 : 0;
  return TSM2X_OK;
}

int tsm2x_release_cached(int device) {
  bcopy_release(device);  // tsm2x_run_multi's per-(device, stream) copies of B
  // per-(device, stream) workspaces: every stream that ever called the library on `device` (-1 =
  // all devices) — synchronised, then freed; the next call on a stream allocates afresh
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
      if (device >= 0 && it->first.first != device) {
        ++it;
        continue;
      }
      {
        Workspace* w = it->second.get();
        std::lock_guard<std::mutex> wl(w->mu);  // released before the workspace is destroyed below
        TSM2X_CUDA(cudaSetDevice(it->first.first));
        TSM2X_CUDA(cudaDeviceSynchronize());  // the stream itself may already be destroyed
        // stream-ordered allocations (ws_reserve): freed on the legacy stream after the device sync
        if (w->buf) TSM2X_CUDA(cudaFreeAsync(w->buf, 0));
        if (w->counters) TSM2X_CUDA(cudaFreeAsync(w->counters, 0));
        w->buf = nullptr;
        w->counters = nullptr;
        w->cap = w->ccap = 0;
        w->flag = nullptr;
      }
      it = g_ws.erase(it);
    }
  }
  // return the freed blocks of the default memory pools to the driver
  {
    int ndev = 0;
    TSM2X_CUDA(cudaGetDeviceCount(&ndev));
    for (int d = 0; d < ndev; ++d) {
      if (device >= 0 && d != device) continue;
      cudaMemPool_t pool;
      TSM2X_CUDA(cudaSetDevice(d));
      TSM2X_CUDA(cudaDeviceSynchronize());
      TSM2X_CUDA(cudaDeviceGetDefaultMemPool(&pool, d));
      TSM2X_CUDA(cudaMemPoolTrimTo(pool, 0));
    }
  }
  // host-path contexts: device / pinned staging buffers, events, streams
  std::lock_guard<std::mutex> lk(g_host_mu);
  for (auto& e : g_host) {
    if (device >= 0 && e.first != device) continue;
    std::lock_guard<std::mutex> hl(e.second->mu);
    TSM2X_CUDA(cudaSetDevice(e.first));
    e.second->release();
  }
  return TSM2X_OK;
}

int tsm2x_set_kernel_events(void* start_event, void* stop_event) {
  t_ev_start = reinterpret_cast<cudaEvent_t>(start_event);
  t_ev_stop = reinterpret_cast<cudaEvent_t>(stop_event);
  return TSM2X_OK;
}

const char* tsm2x_last_error(void) { return t_err.c_str(); }
int tsm2x_version(void) { return 100; }
const char* tsm2x_build_target(void) { return "sm_100a"; }
int64_t tsm2x_launch_count(void) { return g_launches.load(); }

}  // extern "C"
