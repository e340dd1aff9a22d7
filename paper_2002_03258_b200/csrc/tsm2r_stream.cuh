// TSM2R stream kernels: C[m x w] (+)= A[m x k] * B[k x w], A large, w <= NT <= 16 (reference
// naming). Re-derives the paper's three-level tiling (Alg 4, PAPER.md:290-333;
// reference routine kernels.py:187-261) for sm_100a:
//   t1 -> rows per CTA tile R = THREADS * RPT, RPT rows per 128-bit A vector (2 fp64 / 4 fp32)
//   t2 -> NT, all skinny columns in one pass held in registers (A is streamed exactly once)
//   t3 -> the A prefetch depth P (columns in flight per thread, register double buffer)
// The reduction dimension k is split stream-K style across a single wave of CTAs; row blocks
// whose k range is split are combined by the last-arriving CTA in a fixed CTA order, so the
// result is deterministic run to run.
#pragma once
#include "common.cuh"

namespace tsm2x {

template <typename T>
struct StreamArgs {
  const T* A;
  int64_t lda;
  const T* Bt;  // k x NT row-major copy of this pass of B, columns >= w zero
  T* C;
  int64_t ldc;
  int64_t m, k;
  int w;          // valid columns in this pass (<= NT)
  int c_is_zero;  // C is not read
  int64_t num_rb;
  int KC;         // columns per work unit
  Partition part;
  T* ws;          // partials [G][2][NT][R]
  int* counters;  // [num_rb], zero between launches
  int defer;      // 1: only write partials; reduce_partials combines them (many-way splits)
};

// NT consecutive values of one Bt row, loaded with the widest aligned uniform loads.
template <typename T, int NT>
__device__ __forceinline__ void load_brow(const T* __restrict__ p, T (&b)[NT]) {
  constexpr int BYTES = NT * (int)sizeof(T);
  if constexpr (BYTES >= 16) {
    using V = typename Vec<T>::type;
    constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
    for (int i = 0; i < NT / PER; ++i) {
      V v = __ldg(reinterpret_cast<const V*>(p) + i);
#pragma unroll
      for (int e = 0; e < PER; ++e) b[i * PER + e] = vget<T>(v, e);
    }
  } else {
#pragma unroll
    for (int i = 0; i < NT; ++i) b[i] = __ldg(p + i);
  }
}

// Epilogue helpers shared by the LDG and TMA stream kernels. acc[r][j] holds rows row0+r.
template <typename T, int NT, int RPT>
__device__ __forceinline__ void store_c(const StreamArgs<T>& a, int64_t row0, const T (&acc)[RPT][NT]) {
  T old[RPT][NT];  // all reads of C first: one round trip instead of NT*RPT dependent ones
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int64_t row = row0 + r;
      old[r][j] = (!a.c_is_zero && j < a.w && row < a.m) ? a.C[j * a.ldc + row] : T(0);
    }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < a.w) {
      T* cj = a.C + j * a.ldc;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int64_t row = row0 + r;
        if (row < a.m) cj[row] = old[r][j] + acc[r][j];
      }
    }
  }
}

// Partial-segment protocol: write this CTA's partial, count arrivals, the last arriver sums
// all partials of the row block in CTA order and applies the epilogue. Returns nothing;
// must be called by all threads of the CTA (contains __syncthreads).
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

template <typename T, int NT, int RPT, int R, typename Sync = CtaSync>
__device__ __forceinline__ void finish_partial(const StreamArgs<T>& a, int64_t g, int64_t rb, int lrow,
                                               const T (&acc)[RPT][NT], int* s_flag, bool leader = threadIdx.x == 0,
                                               Sync sync = Sync()) {
  const int64_t u0 = rb * a.part.num_kb;
  const int s = (a.part.start(g) >= u0) ? 0 : 1;
  T* mine = a.ws + ((g * 2 + s) * NT) * (int64_t)R;
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int r = 0; r < RPT; ++r) mine[j * R + lrow + r] = acc[r][j];
  if (a.defer) return;
  __threadfence();
  sync();
  const int64_t g_lo = a.part.owner(u0);
  const int64_t g_hi = a.part.owner(u0 + a.part.num_kb - 1);
  if (leader) {
    int prev = atomicAdd(a.counters + rb, 1);
    *s_flag = (prev == (int)(g_hi - g_lo));
  }
  sync();
  if (*s_flag) {
    __threadfence();
    T tot[RPT][NT];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int r = 0; r < RPT; ++r) tot[r][j] = T(0);
    for (int64_t gg = g_lo; gg <= g_hi; ++gg) {
      const int ss = (a.part.start(gg) >= u0) ? 0 : 1;
      const T* p = a.ws + ((gg * 2 + ss) * NT) * (int64_t)R;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int r = 0; r < RPT; ++r) tot[r][j] += __ldcg(p + j * R + lrow + r);
    }
    store_c<T, NT, RPT>(a, rb * R + lrow, tot);
    if (leader) a.counters[rb] = 0;  // ready for the next launch on this workspace
  }
  sync();  // s_flag reuse
}

// ------------------------------------------------------------------------------------------
// LDG flavour: every thread streams its own RPT rows with register double-buffered 128-bit
// loads (the paper's currA/nextA prefetch, Alg 4 lines 6-16), Bt rows via uniform L1 loads.
template <typename T, int NT, int THREADS, int P, bool VEC>
__global__ void __launch_bounds__(THREADS) tsm2r_stream_ldg(const StreamArgs<T> a) {
  using F = AFrag<T, VEC>;
  constexpr int RPT = F::RPT;
  constexpr int R = THREADS * RPT;
  __shared__ int s_flag;
  const int lrow = threadIdx.x * RPT;
  const int64_t g = blockIdx.x;
  int64_t u = a.part.start(g);
  const int64_t u_end = a.part.start(g + 1);
  while (u < u_end) {
    const int64_t rb = u / a.part.num_kb;
    const int64_t u0 = rb * a.part.num_kb;
    const int64_t seg_end = min64(u_end, u0 + a.part.num_kb);
    const int64_t c0 = (u - u0) * a.KC;
    const int64_t c1 = min64(a.k, (seg_end - u0) * (int64_t)a.KC);
    const int64_t row0 = rb * R + lrow;
    T acc[RPT][NT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[r][j] = T(0);

    F cur[P], nxt[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (c0 + p < c1) cur[p].load(a.A + (c0 + p) * a.lda, row0, a.m);
      else cur[p].zero();
    }
    for (int64_t c = c0; c < c1; c += P) {
      const bool more = c + P < c1;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (more && c + P + p < c1) nxt[p].load(a.A + (c + P + p) * a.lda, row0, a.m);
        else nxt[p].zero();
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (c + p < c1) {
          T b[NT];
          load_brow<T, NT>(a.Bt + (c + p) * NT, b);
#pragma unroll
          for (int r = 0; r < RPT; ++r)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[r][j] = fma(cur[p].v[r], b[j], acc[r][j]);
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) cur[p] = nxt[p];
    }

    const bool whole = (u == u0) && (seg_end == u0 + a.part.num_kb);
    if (whole) {
      store_c<T, NT, RPT>(a, row0, acc);
    } else {
      finish_partial<T, NT, RPT, R>(a, g, rb, lrow, acc, &s_flag);
    }
    u = seg_end;
  }
}

// Deferred combine for row blocks split many ways (few row blocks, long k): one thread per
// (row, column), partials summed in the same fixed CTA order as finish_partial.
template <typename T, int NT, int R>
__global__ void reduce_partials(const StreamArgs<T> a) {
  const int lrow = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rb = blockIdx.y;
  if (lrow >= R) return;
  const int64_t u0 = rb * a.part.num_kb;
  const int64_t g_lo = a.part.owner(u0);
  const int64_t g_hi = a.part.owner(u0 + a.part.num_kb - 1);
  if (g_lo == g_hi) return;  // written directly by its only CTA
  const int64_t row = rb * R + lrow;
  if (row >= a.m) return;
  for (int j = 0; j < a.w; ++j) {
    T tot = T(0);
    for (int64_t gg = g_lo; gg <= g_hi; ++gg) {
      const int ss = (a.part.start(gg) >= u0) ? 0 : 1;
      tot += a.ws[((gg * 2 + ss) * NT + j) * (int64_t)R + lrow];
    }
    T* c = a.C + row + j * a.ldc;
    *c = a.c_is_zero ? tot : *c + tot;
  }
}

// Bt[c][j] = B[c + j*ldb] for c < k and j < w; 0 for padding rows k <= c < kpad and
// columns w <= j < NT (B pass slab -> row-major, zero padded to whole stages).
template <typename T, int NT>
__global__ void prep_bt(const T* __restrict__ B, int64_t ldb, int64_t k, int64_t kpad, int w, T* __restrict__ Bt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kpad * NT) {
    int64_t c = i / NT;
    int j = (int)(i - c * NT);
    Bt[i] = (j < w && c < k) ? B[c + j * ldb] : T(0);
  }
}

}  // namespace tsm2x
