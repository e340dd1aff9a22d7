// The paper's baseline TSM2R algorithms, compiled as written (one thread per row of A, block
// size t1, grid ceil(m/t1)), so the V0 -> V1 -> V2 -> V3 ablation of PAPER.md:867 can be
// measured on B200. Production calls never use these.
//   V0  Alg 1, reference kernels.py:86-100   inner product, C updated in global memory
//   V1  Alg 2, reference kernels.py:103-121  outer product, t2 register accumulators per pass,
//                                            B read straight from global memory
//   V2  Alg 3, reference kernels.py:242-261 (no-prefetch branch 211-220): + t1 x t2 B tile in
//                                            shared memory, column-major (conflict-free), two
//                                            barriers per t1-row step
#pragma once
#include <atomic>

#include "common.cuh"

namespace tsm2x {

template <typename T>
__global__ void ablation_v0(const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, int64_t m, int64_t k,
                            int64_t n, int c_is_zero) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  for (int64_t i = 0; i < n; ++i) {
    if (c_is_zero) C[row + i * ldc] = T(0);
    for (int64_t j = 0; j < k; ++j) C[row + i * ldc] += A[row + j * lda] * B[j + i * ldb];  // aliasing: RMW per j
  }
}

template <typename T, int NT>
__global__ void ablation_v1(const T* __restrict__ A, int64_t lda, const T* __restrict__ B, int64_t ldb,
                            T* __restrict__ C, int64_t ldc, int64_t m, int64_t k, int64_t n, int t2, int c_is_zero) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  for (int64_t p = 0; p < n; p += t2) {
    const int w = (int)min64(t2, n - p);
    T regs[NT];
#pragma unroll
    for (int c = 0; c < NT; ++c) regs[c] = (c < w && !c_is_zero) ? C[row + (p + c) * ldc] : T(0);
    for (int64_t i = 0; i < k; ++i) {
      const T av = A[row + i * lda];
#pragma unroll
      for (int c = 0; c < NT; ++c)
        if (c < w) regs[c] = fma(av, B[i + (p + c) * ldb], regs[c]);
    }
#pragma unroll
    for (int c = 0; c < NT; ++c)
      if (c < w) C[row + (p + c) * ldc] = regs[c];
  }
}

template <typename T, int NT>
__global__ void ablation_v2(const T* __restrict__ A, int64_t lda, const T* __restrict__ B, int64_t ldb,
                            T* __restrict__ C, int64_t ldc, int64_t m, int64_t k, int64_t n, int t2, int t3,
                            int c_is_zero) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);  // t1 x NT, column-major: tile[r + c*t1]
  const int t1 = blockDim.x;
  const int ltid = threadIdx.x;
  const int64_t row = (int64_t)blockIdx.x * t1 + ltid;
  const bool live = row < m;
  for (int64_t p = 0; p < n; p += t2) {
    const int w = (int)min64(t2, n - p);
    T regs[NT];
#pragma unroll
    for (int c = 0; c < NT; ++c) regs[c] = (live && c < w && !c_is_zero) ? C[row + (p + c) * ldc] : T(0);
    for (int64_t j = 0; j < k; j += t1) {
      __syncthreads();
      const int64_t brow = j + ltid;
#pragma unroll
      for (int c = 0; c < NT; ++c) tile[ltid + c * t1] = (brow < k && c < w) ? B[brow + (p + c) * ldb] : T(0);
      __syncthreads();
      const int lim = (int)min64(t1, k - j);
      for (int l = 0; l < lim; l += t3) {
        const int hi = min(l + t3, lim);
        for (int e = l; e < hi; ++e) {
          const T av = live ? A[row + (j + e) * lda] : T(0);
#pragma unroll
          for (int c = 0; c < NT; ++c) regs[c] = fma(av, tile[e + c * t1], regs[c]);
        }
      }
    }
    if (live) {
#pragma unroll
      for (int c = 0; c < NT; ++c)
        if (c < w) C[row + (p + c) * ldc] = regs[c];
    }
  }
}

}  // namespace tsm2x
