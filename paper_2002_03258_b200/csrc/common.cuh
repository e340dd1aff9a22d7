// Shared device helpers for the TSM2X sm_100a kernels: vector types, streaming loads,
// mbarrier / bulk-copy PTX wrappers, and the stream-K partition arithmetic.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tsm2x {

// ------------------------------------------------------------------------------------------
// Element traits: the 16-byte vector each thread moves per A column, RPT = rows per vector.
template <typename T> struct Vec;
template <> struct Vec<double> { using type = double2; static constexpr int N = 2; };
template <> struct Vec<float>  { using type = float4;  static constexpr int N = 4; };

template <typename T> __device__ __forceinline__ T vget(const typename Vec<T>::type& v, int i);
template <> __device__ __forceinline__ double vget<double>(const double2& v, int i) { return i == 0 ? v.x : v.y; }
template <> __device__ __forceinline__ float vget<float>(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

template <typename T> __device__ __forceinline__ typename Vec<T>::type vmake(const T* o);
template <> __device__ __forceinline__ double2 vmake<double>(const double* o) { return make_double2(o[0], o[1]); }
template <> __device__ __forceinline__ float4 vmake<float>(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }

// Streaming 128-bit load that does not allocate in L1 (A is touched exactly once).
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

// One RPT-row slice of an A column: vector load when the whole vector is inside [0, m),
// element loads for the ragged tail, zeros past m.
template <typename T, bool VEC>
struct AFrag {
  static constexpr int RPT = VEC ? Vec<T>::N : 1;
  T v[RPT];
  __device__ __forceinline__ void load(const T* __restrict__ col, int64_t row0, int64_t m) {
    if constexpr (VEC) {
      using V = typename Vec<T>::type;
      if (row0 + RPT <= m) {
        V x = ld_stream(reinterpret_cast<const V*>(col + row0));
#pragma unroll
        for (int r = 0; r < RPT; ++r) v[r] = vget<T>(x, r);
      } else {
#pragma unroll
        for (int r = 0; r < RPT; ++r) v[r] = (row0 + r < m) ? ld_stream(col + row0 + r) : T(0);
      }
    } else {
      v[0] = (row0 < m) ? ld_stream(col + row0) : T(0);
    }
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < RPT; ++r) v[r] = T(0);
  }
};

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// ------------------------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine, 1-D form) wrappers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// expect-tx without an arrival (the stage's one arrival comes later, after other lanes' writes)
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
#ifndef TSM2X_WAIT_BACKOFF_NS
#define TSM2X_WAIT_BACKOFF_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if TSM2X_WAIT_BACKOFF_NS > 0
  while (!mbar_try_wait(bar, parity)) __nanosleep(TSM2X_WAIT_BACKOFF_NS);
#else
  asm volatile(
      "{\n .reg .pred p;\n"
      "TSM2X_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TSM2X_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
// Wait with a short sleep between polls: fewer issue slots (and watts) spent by warps that
// mostly wait — the tensor-core fp32 kernel, whose converter / MMA warps idle behind the tensor
// pipe, is 2 % faster sustained with it; the DMMA kernels are indifferent (profiles/README.md).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, unsigned ns = 64) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(ns);
}
// Warp release of a ring stage: the warp's lanes read the stage, __syncwarp, lane 0 arrives
// (release; the barrier orders the other lanes' reads before it). compute-sanitizer racecheck does
// not follow that __syncwarp edge and reports the producer's next write as a hazard
// (tools/racecheck_probe.cu shows it on a minimal correct kernel), so the racecheck build
// (-DTSM2X_RACECHECK, `make racecheck`) has every lane arrive and the barriers count lanes.
#ifdef TSM2X_RACECHECK
constexpr int kArrivalsPerWarp = 32;
__device__ __forceinline__ void warp_release(uint64_t* bar) { mbar_arrive(bar); }
#else
constexpr int kArrivalsPerWarp = 1;
__device__ __forceinline__ void warp_release(uint64_t* bar) {
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
#endif

// global -> shared bulk copy completing on an mbarrier; bytes % 16 == 0, both addresses 16B-aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                     uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// L2 policy for the streamed A (TSM2X_L2POL experiments): 0 evict_first (default),
// 1 evict_normal, 2 evict_unchanged, 3 evict_last
__device__ __forceinline__ uint64_t policy_for(int which) {
  uint64_t p;
  if (which == 1)
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else if (which == 2)
    asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  else if (which == 3)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Programmatic dependent launch (griddepcontrol): see prep_dyn / tsm2r_stream_tma.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------------------------------
// Stream-K partition of U = num_rb * num_kb work units (row block major, k block minor) over G
// CTAs: CTA g owns units [start(g), start(g+1)), start(g) = floor(g*U/G). Every CTA gets
// floor(U/G) or ceil(U/G) units, so one wave finishes together for any (m, k).
struct Partition {
  int64_t units;   // num_rb * num_kb
  int64_t num_kb;  // k blocks per row block
  int64_t G;       // CTAs
  __host__ __device__ int64_t start(int64_t g) const { return (g * units) / G; }
  // the CTA whose range contains unit u (largest g with start(g) <= u)
  __host__ __device__ int64_t owner(int64_t u) const { return ((u + 1) * G - 1) / units; }
};

}  // namespace tsm2x
