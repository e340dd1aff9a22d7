// TSM2L split-n kernel: the warp-shuffle variant named in BASELINE.json's north_star, built as an
// A/B candidate against the production TSM2L path (the TMA stream kernel's single-chunk row
// blocks). C[m x w] (+)= A[m x k] * B[k x w], k <= TSM2L_KMAX, A and C 16-byte aligned.
//
// S lanes share one group of RPT rows (one 16-byte vector of A per column: 2 fp64 / 4 fp32 rows):
// lane s of the group takes the inner indices l in [s*KS, (s+1)*KS), KS = ceil(k / S), so each
// lane issues k/S vector loads per row group instead of k (more row groups in flight per SM for
// the same registers), and accumulates partial sums of all NT outputs of its rows. The S partial
// sums are combined by recursive halving over warp shuffles (log2 S steps; at step h a lane keeps
// half of its current columns, sends the other half to lane s ^ h and adds what it receives),
// so lane s ends with the full sums of output columns [s*NT/S, (s+1)*NT/S) and stores them as
// 16-byte vectors — (1 - 1/S) * RPT * NT shuffles per lane per row group. B lives in shared
// memory for the CTA's life with rows padded by one vector, so the S rows the lanes of a group
// read at once fall in different banks. Reference algorithm: TSM2L-Opt1/Opt2 (PAPER.md:537-613,
// reference kernels.py:264-344); zero-C contract (kernels.py:366-368): C never read.
#pragma once
#include "common.cuh"
#include "tsm2l.cuh"

namespace tsm2x {

template <typename T, int NT, int S, int THREADS, int KCH>
__global__ void __launch_bounds__(THREADS) tsm2l_splitn_kernel(const LArgs<T> a) {
  static_assert(S >= 2 && (S & (S - 1)) == 0 && NT % S == 0 && THREADS % 32 == 0, "split geometry");
  using V = typename Vec<T>::type;
  constexpr int RPT = Vec<T>::N;
  constexpr int PAD = 16 / (int)sizeof(T);
  constexpr int NTP = NT + PAD;  // padded B row: the S rows read together start in different banks
  constexpr int OWN = NT / S;    // output columns per lane after the reduction
  __shared__ __align__(16) T sB[TSM2L_KMAX * NTP];
  for (int i = threadIdx.x; i < a.k * NTP; i += THREADS) {
    const int l = i / NTP, j = i % NTP;
    sB[i] = j < a.w ? a.B[l + (int64_t)j * a.ldb] : T(0);
  }
  __syncthreads();

  const int s = threadIdx.x % S;
  const int KS = (a.k + S - 1) / S;
  const int l_begin = s * KS, l_end = min(a.k, l_begin + KS);
  const int64_t groups = (a.m + RPT - 1) / RPT;
  const int64_t stride = (int64_t)gridDim.x * (THREADS / S);
  // warp-uniform loop (every lane takes part in the shuffles); groups past the end have row0 >= m,
  // so their loads read zeros and their stores are skipped
  const int64_t warp_g0 = (int64_t)blockIdx.x * (THREADS / S) + (threadIdx.x / 32) * (32 / S);
  for (int64_t g0 = warp_g0; g0 < groups; g0 += stride) {
    const int64_t gi = g0 + (threadIdx.x % 32) / S;
    const int64_t row0 = gi * RPT;
    const bool full = row0 + RPT <= a.m;
    T acc[RPT][NT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[r][j] = T(0);
    for (int l0 = l_begin; l0 < l_end; l0 += KCH) {
      T av[KCH][RPT];
#pragma unroll
      for (int p = 0; p < KCH; ++p) {
        const int l = l0 + p;
        const T* col = a.A + (int64_t)l * a.lda;
        if (l < l_end && full) {
          const V x = ld_stream(reinterpret_cast<const V*>(col + row0));
#pragma unroll
          for (int r = 0; r < RPT; ++r) av[p][r] = vget<T>(x, r);
        } else {
#pragma unroll
          for (int r = 0; r < RPT; ++r) av[p][r] = (l < l_end && row0 + r < a.m) ? ld_stream(col + row0 + r) : T(0);
        }
      }
#pragma unroll
      for (int p = 0; p < KCH; ++p) {
        if (l0 + p >= l_end) break;
        const V* br = reinterpret_cast<const V*>(sB + (l0 + p) * NTP);
#pragma unroll
        for (int i = 0; i < NT / PAD; ++i) {
          const V bv = br[i];
#pragma unroll
          for (int e = 0; e < PAD; ++e)
#pragma unroll
            for (int r = 0; r < RPT; ++r) acc[r][i * PAD + e] = fma(av[p][r], vget<T>(bv, e), acc[r][i * PAD + e]);
        }
      }
    }
    // recursive halving over the S lanes of the group: after the step with mask h a lane holds
    // the group-wide partial sums of half the columns it held before, in acc[.][0 .. W/2)
    constexpr int LOG2S = S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : 4;
#pragma unroll
    for (int step = 0; step < LOG2S; ++step) {
      const int h = S >> (step + 1), W = NT >> step;  // compile-time after unrolling
      const bool upper = (s & h) != 0;
#pragma unroll
      for (int j = 0; j < W / 2; ++j)
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const T lo = acc[r][j], hi = acc[r][j + W / 2];
          const T recv = __shfl_xor_sync(0xffffffffu, upper ? lo : hi, h);
          acc[r][j] = (upper ? hi : lo) + recv;
        }
    }
    // lane s owns columns [s*OWN, (s+1)*OWN): column offset of the kept halves
    const int c0 = s * OWN;
#pragma unroll
    for (int j = 0; j < OWN; ++j) {
      const int col = c0 + j;
      if (col >= a.w) continue;
      T* cj = a.C + (int64_t)col * a.ldc;
      T out[RPT];
      if (full) {
        if (!a.c_is_zero) {
          const V old = __ldcs(reinterpret_cast<const V*>(cj + row0));
#pragma unroll
          for (int r = 0; r < RPT; ++r) out[r] = vget<T>(old, r) + acc[r][j];
        } else {
#pragma unroll
          for (int r = 0; r < RPT; ++r) out[r] = acc[r][j];
        }
        __stcs(reinterpret_cast<V*>(cj + row0), vmake<T>(out));
      } else {
#pragma unroll
        for (int r = 0; r < RPT; ++r)
          if (row0 + r < a.m) cj[row0 + r] = (a.c_is_zero ? T(0) : cj[row0 + r]) + acc[r][j];
      }
    }
  }
}

}  // namespace tsm2x
