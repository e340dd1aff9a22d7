// Does compute-sanitizer racecheck model mbarrier synchronisation? A minimal, correct
// producer/consumer handoff through an mbarrier (arrive = release, try_wait = acquire, PTX
// defaults): if racecheck reports a hazard here, its reports on the TMA/mbarrier ring of the
// stream kernels are of the same (false-positive) class. Also a cp.async.bulk variant.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/racecheck_probe tools/racecheck_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_parity(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(s32(bar)),
      "r"(ph)
      : "memory");
}

// The ring's release pattern: a consumer warp reads the buffer, __syncwarp, lane 0 arrives on the
// "empty" barrier; the producer waits on it and overwrites the buffer (st.shared, or bulk copy).
__global__ void release(const double* g, double* out, int bulk) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) uint64_t empty, full;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&empty)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 256; ++i) buf[i] = 1.0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) {
    out[threadIdx.x] = buf[threadIdx.x % 256];
    __syncwarp();
    if (threadIdx.x == 32) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty)) : "memory");
  } else if (threadIdx.x == 0) {
    wait_parity(&empty, 0);
    if (bulk) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full)), "r"(2048) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];" ::"r"(
                       s32(buf)),
                   "l"(g), "r"(s32(&full))
                   : "memory");
      wait_parity(&full, 0);
    } else {
      for (int i = 0; i < 256; ++i) buf[i] = 2.0;
    }
  }
}

__global__ void handoff(const double* g, double* out, int bulk) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) uint64_t full;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (bulk) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full)), "r"(2048) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];" ::"r"(
                       s32(buf)),
                   "l"(g), "r"(s32(&full))
                   : "memory");
    } else {
      for (int i = 0; i < 256; ++i) buf[i] = g[i];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&full)) : "memory");
    }
  } else if (threadIdx.x >= 32) {
    wait_parity(&full, 0);
    out[threadIdx.x] = buf[threadIdx.x % 256];
  }
}

int main() {
  double *g, *o;
  cudaMalloc(&g, 2048);
  cudaMalloc(&o, 64 * 8);
  cudaMemset(g, 0, 2048);
  for (int bulk = 0; bulk < 2; ++bulk) {
    handoff<<<1, 64>>>(g, o, bulk);
    cudaError_t e = cudaDeviceSynchronize();
    printf("handoff (%s): %s\n", bulk ? "cp.async.bulk" : "st.shared", cudaGetErrorString(e));
  }
  for (int bulk = 0; bulk < 2; ++bulk) {
    release<<<1, 64>>>(g, o, bulk);
    cudaError_t e = cudaDeviceSynchronize();
    printf("release via __syncwarp + lane-0 arrive (%s): %s\n", bulk ? "cp.async.bulk" : "st.shared", cudaGetErrorString(e));
  }
  return 0;
}
