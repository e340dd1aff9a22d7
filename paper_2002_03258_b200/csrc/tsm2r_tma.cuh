// TSM2R stream kernel, TMA flavour (the production path on sm_100a).
//
// Work decomposition. A (m x k, column-major) is cut into items = (row block of R rows,
// column chunk of KCH columns). Items are handed out dynamically (one atomicAdd per item on a
// global queue) in row-block-major order, so every SM keeps streaming until the queue is empty
// whatever bandwidth it happens to get (per-SM DRAM bandwidth on B200 varies by ~+-10%, which a
// static split turns straight into tail time — measured, profiles/README). Each item's partial
// sum starts from zero and is written to its own slot; the last item of a row block to finish
// adds the slots in chunk order plus C and writes C, then discards the slots from L2. The
// result therefore does not depend on which CTA ran which item: the kernel is deterministic.
//
// Per CTA: warp 0 is the producer — one elected lane takes items off the queue and, per stage
// of KC columns, issues 2-D TMA tensor loads of the A tile (R rows x KC columns as R/256 boxes
// of 256 rows; rows >= m and columns >= k arrive zero-filled) plus a 1-D bulk copy of the KC
// matching rows of Bt, completing on the stage's "full" mbarrier, and tags the stage with its
// item id. Warps 1..CW are consumers: each thread owns RPT consecutive rows, reads its A vector
// with one conflict-free LDS.128 per column and the Bt row as broadcast LDS.128s, and keeps the
// NT outputs per row in registers; one lane per warp releases the stage on its "empty" mbarrier.
// A STAGES-deep ring keeps ~(STAGES-1) * 32 KB of A in flight per SM independent of register
// pressure — the B200 replacement for the paper's register double buffer (Alg 4).
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "tsm2r_stream.cuh"

namespace tsm2x {

template <typename T, int NT>
struct TmaCfg {
  static constexpr int CW = 8;                        // consumer warps
  static constexpr int THREADS = 32 * (CW + 1);       // + producer warp
  static constexpr int RPT = Vec<T>::N;               // rows per consumer thread
  static constexpr int R = CW * 32 * RPT;             // rows per row block (512 fp64 / 1024 fp32)
  static constexpr int BOX = 256;                     // rows per TMA box (box dim limit)
  static constexpr int NBOX = R / BOX;
  static constexpr int KC = 8;                        // columns per stage
  static constexpr int STAGES = 6;
  static constexpr int A_ELEMS = R * KC;
  static constexpr int B_ELEMS = KC * NT;
  static constexpr int A_BYTES = A_ELEMS * (int)sizeof(T);
  static constexpr int B_BYTES = B_ELEMS * (int)sizeof(T);
  static constexpr int B_BYTES_PAD = (B_BYTES + 127) / 128 * 128;
  static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES_PAD) + 2 * STAGES * 8 + STAGES * 8 + 16;
};

template <typename T>
struct DynArgs {
  const T* Bt;      // kpad x NT row-major copy of this pass of B, zero padded
  T* C;
  int64_t ldc;
  int64_t m, k;
  int w;            // valid columns in this pass (<= NT)
  int c_is_zero;
  int64_t num_rb;
  int64_t nch;      // column chunks per row block
  int64_t kch;      // columns per chunk (multiple of KC)
  int64_t items;    // num_rb * nch
  int defer;        // 1: leave partials for reduce_items (very many chunks per row block)
  T* ws;            // partial slots [items][NT][R]
  int* counters;    // [num_rb] arrivals, zero between launches
  int* queue;       // [0] next item, [1] producers finished; zero between launches
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

struct ConsumerSync {
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync 1, %0;" ::"r"(TmaCfg<double, 1>::CW * 32) : "memory");
  }
};

// Epilogue of one item (all consumer threads): direct C update when the row block is a single
// chunk, else partial slot + arrival count; the last arrival combines the row block.
template <typename T, int NT, int RPT, int R>
__device__ __forceinline__ void finish_item(const DynArgs<T>& a, int64_t item, int ct, T (&acc)[RPT][NT],
                                            int* s_flag) {
  const int64_t rb = item / a.nch;
  const int lrow = ct * RPT;
  const int64_t row0 = rb * R + lrow;
  auto store = [&](const T (&v)[RPT][NT]) {
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j < a.w) {
        T* cj = a.C + j * a.ldc;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int64_t row = row0 + r;
          if (row < a.m) cj[row] = a.c_is_zero ? v[r][j] : cj[row] + v[r][j];
        }
      }
    }
  };
  if (a.nch == 1) {
    store(acc);
    return;
  }
  using V = typename Vec<T>::type;
  T* slot = a.ws + item * (int64_t)(NT * R);
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    T tmp[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) tmp[r] = acc[r][j];
    *reinterpret_cast<V*>(slot + j * R + lrow) = vmake<T>(tmp);
  }
  if (a.defer) return;
  __threadfence();
  ConsumerSync()();
  if (ct == 0) {
    const int prev = atomicAdd(a.counters + rb, 1);
    *s_flag = (prev == (int)(a.nch - 1));
  }
  ConsumerSync()();
  if (*s_flag) {
    __threadfence();
    T tot[RPT][NT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < NT; ++j) tot[r][j] = T(0);
    const T* base = a.ws + rb * a.nch * (int64_t)(NT * R);
    for (int64_t c = 0; c < a.nch; ++c) {
      const T* p = base + c * (NT * R);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const V v = __ldcg(reinterpret_cast<const V*>(p + j * R + lrow));
#pragma unroll
        for (int r = 0; r < RPT; ++r) tot[r][j] += vget<T>(v, r);
      }
    }
    store(tot);
    ConsumerSync()();  // everyone has read the slots
    // the slots are dead: drop them from L2 without a DRAM write-back
    const int64_t lines = a.nch * (int64_t)(NT * R * sizeof(T)) / 128;
    const char* b = reinterpret_cast<const char*>(base);
    for (int64_t l = ct; l < lines; l += TmaCfg<T, NT>::CW * 32) discard_l2_line(b + l * 128);
    if (ct == 0) a.counters[rb] = 0;  // ready for the next launch on this workspace
  }
  ConsumerSync()();  // s_flag reuse
}

template <typename T, int NT>
__global__ void __launch_bounds__(TmaCfg<T, NT>::THREADS, 1)
    tsm2r_stream_tma(const DynArgs<T> a, const __grid_constant__ CUtensorMap tmA) {
  using Cfg = TmaCfg<T, NT>;
  using V = typename Vec<T>::type;
  constexpr int RPT = Cfg::RPT, R = Cfg::R, KC = Cfg::KC, STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* sA = reinterpret_cast<T*>(smem);
  T* sB = reinterpret_cast<T*>(smem + STAGES * Cfg::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (Cfg::A_BYTES + Cfg::B_BYTES_PAD));
  uint64_t* empty = full + STAGES;
  int64_t* meta = reinterpret_cast<int64_t*>(empty + STAGES);  // item id of each stage, -1 = end
  int* s_flag = reinterpret_cast<int*>(meta + STAGES);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::CW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      const uint64_t pol = policy_evict_first();
      int it = 0;
      for (;;) {
        const int64_t item = atomicAdd(reinterpret_cast<unsigned long long*>(a.queue), 1ull);
        if (item >= a.items) break;
        const int64_t rb = item / a.nch;
        const int64_t col0 = (item - rb * a.nch) * a.kch;
        const int64_t col1 = min64(a.k, col0 + a.kch);
        const int64_t row_base = rb * R;
        const int nbox = (int)min64(Cfg::NBOX, (a.m - row_base + Cfg::BOX - 1) / Cfg::BOX);
        const uint32_t tx = (uint32_t)(nbox * Cfg::BOX * KC * (int)sizeof(T) + Cfg::B_BYTES);
        for (int64_t col = col0; col < col1; col += KC, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          meta[s] = item;
          mbar_arrive_expect_tx(&full[s], tx);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(sA + (size_t)s * Cfg::A_ELEMS + b * (Cfg::BOX * KC), &tmA, (int)(row_base + b * Cfg::BOX),
                        (int)col, &full[s], pol);
          bulk_g2s(sB + (size_t)s * (Cfg::B_BYTES_PAD / sizeof(T)), a.Bt + col * NT, Cfg::B_BYTES, &full[s]);
        }
      }
      // end-of-work marker for the consumers
      const int s = it % STAGES;
      mbar_wait(&empty[s], ((uint32_t)(it / STAGES) & 1u) ^ 1u);
      meta[s] = -1;
      mbar_arrive(&full[s]);
      // the last producer out resets the queue for the next launch on this workspace
      __threadfence();
      const unsigned prev = atomicAdd(reinterpret_cast<unsigned*>(a.queue) + 2, 1u);
      if (prev == gridDim.x - 1) {
        *reinterpret_cast<unsigned long long*>(a.queue) = 0ull;
        reinterpret_cast<unsigned*>(a.queue)[2] = 0u;
        __threadfence();
      }
    }
    return;
  }

  // ---------------- consumers
  const int ct = threadIdx.x - 32;
  const int lrow = ct * RPT;
  const int box = lrow / Cfg::BOX, rin = lrow % Cfg::BOX;
  T acc[RPT][NT];
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[r][j] = T(0);
  int64_t cur = -1;
  for (int it = 0;; ++it) {
    const int s = it % STAGES;
    const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
    mbar_wait(&full[s], ph);
    const int64_t item = meta[s];
    if (item != cur) {
      if (cur >= 0) {
        finish_item<T, NT, RPT, R>(a, cur, ct, acc, s_flag);
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[r][j] = T(0);
      }
      if (item < 0) break;
      cur = item;
    }
    const T* As = sA + (size_t)s * Cfg::A_ELEMS + box * (Cfg::BOX * KC) + rin;
    const T* Bs = sB + (size_t)s * (Cfg::B_BYTES_PAD / sizeof(T));
#pragma unroll
    for (int cc = 0; cc < KC; ++cc) {
      const V av = *reinterpret_cast<const V*>(As + cc * Cfg::BOX);
      T b[NT];
      if constexpr (NT * sizeof(T) >= 16) {
        constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
        for (int i = 0; i < NT / PER; ++i) {
          const V bv = reinterpret_cast<const V*>(Bs + cc * NT)[i];
#pragma unroll
          for (int e = 0; e < PER; ++e) b[i * PER + e] = vget<T>(bv, e);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NT; ++i) b[i] = Bs[cc * NT + i];
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const T ar = vget<T>(av, r);
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[r][j] = fma(ar, b[j], acc[r][j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// Combine for row blocks split into very many chunks (defer mode): one thread per (row, column),
// slots summed in chunk order — the same order as finish_item, so the same bits.
template <typename T, int NT, int R>
__global__ void reduce_items(const DynArgs<T> a) {
  const int lrow = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rb = blockIdx.y;
  const int64_t row = rb * R + lrow;
  if (lrow >= R || row >= a.m) return;
  const T* base = a.ws + rb * a.nch * (int64_t)(NT * R);
  for (int j = 0; j < a.w; ++j) {
    T tot = T(0);
    for (int64_t c = 0; c < a.nch; ++c) tot += base[c * (NT * R) + j * R + lrow];
    T* cp = a.C + row + j * a.ldc;
    *cp = a.c_is_zero ? tot : *cp + tot;
  }
}

}  // namespace tsm2x
