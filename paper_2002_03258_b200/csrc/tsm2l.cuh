// TSM2L kernel: C[m x w] (+)= A[m x k] * B[k x w] with A tall-and-skinny (k <= KMAX) and B
// small. Re-derives TSM2L-Opt1/Opt2 (reference kernels.py:264-344) for
// sm_100a: the whole of B lives in shared memory for the life of the CTA (the paper reloads
// the B tile once per row tile, tcf times per thread), CTAs walk row groups grid-stride (the
// tcf "row tiles per thread" analogue, chosen so one wave covers the GPU), and when the caller
// guarantees a zero C (the Opt2 contract, kernels.py:366-368) C is written without being read.
#pragma once
#include "common.cuh"

namespace tsm2x {

template <typename T>
struct LArgs {
  const T* A;
  int64_t lda;
  const T* B;
  int64_t ldb;
  T* C;
  int64_t ldc;
  int64_t m;
  int k;          // <= KMAX
  int w;          // valid columns (<= NT)
  int c_is_zero;
};

constexpr int TSM2L_KMAX = 64;

template <typename T, int NT, int THREADS, int KCH, bool VEC>
__global__ void __launch_bounds__(THREADS) tsm2l_kernel(const LArgs<T> a) {
  using F = AFrag<T, VEC>;
  constexpr int RPT = F::RPT;
  __shared__ __align__(16) T sB[TSM2L_KMAX * NT];  // row-major: sB[l*NT + j] = B[l, j]
  for (int i = threadIdx.x; i < a.k * NT; i += THREADS) {
    int l = i / NT, j = i % NT;
    sB[i] = j < a.w ? a.B[l + (int64_t)j * a.ldb] : T(0);
  }
  __syncthreads();

  const int64_t groups = (a.m + RPT - 1) / RPT;
  for (int64_t gi = (int64_t)blockIdx.x * THREADS + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * THREADS) {
    const int64_t row0 = gi * RPT;
    T acc[RPT][NT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[r][j] = T(0);

    for (int l0 = 0; l0 < a.k; l0 += KCH) {
      F f[KCH];
#pragma unroll
      for (int p = 0; p < KCH; ++p) {
        if (l0 + p < a.k) f[p].load(a.A + (int64_t)(l0 + p) * a.lda, row0, a.m);
        else f[p].zero();
      }
#pragma unroll
      for (int p = 0; p < KCH; ++p) {
        if (l0 + p < a.k) {
          const T* br = sB + (l0 + p) * NT;
          T b[NT];
          if constexpr (NT * sizeof(T) >= 16) {
            using V = typename Vec<T>::type;
            constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
            for (int i = 0; i < NT / PER; ++i) {
              V v = reinterpret_cast<const V*>(br)[i];
#pragma unroll
              for (int e = 0; e < PER; ++e) b[i * PER + e] = vget<T>(v, e);
            }
          } else {
#pragma unroll
            for (int i = 0; i < NT; ++i) b[i] = br[i];
          }
#pragma unroll
          for (int r = 0; r < RPT; ++r)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[r][j] = fma(f[p].v[r], b[j], acc[r][j]);
        }
      }
    }

    // epilogue: all reads of C first (one round trip), then the stores; whole vectors in range
    // use one 128-bit access per column.
    T old[RPT][NT];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int r = 0; r < RPT; ++r) old[r][j] = T(0);
    const bool full_vec = VEC && (row0 + RPT <= a.m);
    if (!a.c_is_zero) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        if (j >= a.w) continue;
        const T* cj = a.C + (int64_t)j * a.ldc;
        if constexpr (VEC) {
          if (full_vec) {
            using V = typename Vec<T>::type;
            const V v = __ldcs(reinterpret_cast<const V*>(cj + row0));
#pragma unroll
            for (int r = 0; r < RPT; ++r) old[r][j] = vget<T>(v, r);
            continue;
          }
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r)
          if (row0 + r < a.m) old[r][j] = cj[row0 + r];
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j >= a.w) continue;
      T* cj = a.C + (int64_t)j * a.ldc;
      T out[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) out[r] = old[r][j] + acc[r][j];
      if constexpr (VEC) {
        if (full_vec) {
          using V = typename Vec<T>::type;
          __stcs(reinterpret_cast<V*>(cj + row0), vmake<T>(out));
          continue;
        }
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (row0 + r < a.m) cj[row0 + r] = out[r];
    }
  }
}

}  // namespace tsm2x
