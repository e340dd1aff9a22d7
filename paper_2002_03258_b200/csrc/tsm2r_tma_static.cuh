// TSM2R stream kernel, TMA flavour, STATIC stream-K split — the deterministic mode
// (TSM2X_FLAG_DETERMINISTIC). Same producer / consumer structure as tsm2r_tma.cuh, but each CTA
// owns a contiguous range of (row block, 8-column stage) units fixed by (m, k, grid) alone, and
// row blocks split between CTAs are combined by the last-arriving CTA in CTA order, so every
// launch produces the same bits. Costs the per-SM bandwidth spread as tail time.
#pragma once
#include "tsm2r_tma.cuh"

namespace tsm2x {

template <typename T, int NT>
__global__ void __launch_bounds__(TmaCfg<T, NT>::THREADS, 1)
    tsm2r_static_tma(const StreamArgs<T> a, const __grid_constant__ CUtensorMap tmA) {
  using Cfg = TmaCfg<T, NT>;
  using V = typename Vec<T>::type;
  constexpr int RPT = Cfg::RPT, R = Cfg::R, KC = Cfg::KC, STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* sA = reinterpret_cast<T*>(smem);
  T* sB = reinterpret_cast<T*>(smem + STAGES * Cfg::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (Cfg::A_BYTES + Cfg::B_BYTES_PAD));
  uint64_t* empty = full + STAGES;
  int* s_flag = reinterpret_cast<int*>(empty + STAGES);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::CW * kArrivalsPerWarp);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t g = blockIdx.x;
  const int64_t u_begin = a.part.start(g), u_end = a.part.start(g + 1);

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      const uint64_t pol = policy_evict_first();
      int it = 0;
      for (int64_t u = u_begin; u < u_end;) {
        const int64_t rb = u / a.part.num_kb;
        const int64_t u0 = rb * a.part.num_kb;
        const int64_t seg_end = min64(u_end, u0 + a.part.num_kb);
        const int64_t row_base = rb * R;
        int nbox = (int)min64(Cfg::NBOX, (a.m - row_base + Cfg::BOX - 1) / Cfg::BOX);
        const uint32_t tx = (uint32_t)(nbox * Cfg::BOX * KC * (int)sizeof(T) + Cfg::B_BYTES);
        for (int64_t uu = u; uu < seg_end; ++uu, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full[s], tx);
          const int col = (int)((uu - u0) * KC);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(sA + (size_t)s * Cfg::A_ELEMS + b * (Cfg::BOX * KC), &tmA, (int)(row_base + b * Cfg::BOX), col,
                        &full[s], pol);
          bulk_g2s(sB + (size_t)s * (Cfg::B_BYTES_PAD / sizeof(T)), a.Bt + (int64_t)col * NT, Cfg::B_BYTES, &full[s]);
        }
        u = seg_end;
      }
    }
    return;
  }

  // ---------------- consumers
  const int ct = threadIdx.x - 32;
  const int lrow = ct * RPT;
  const int box = lrow / Cfg::BOX, rin = lrow % Cfg::BOX;
  const bool leader = (ct == 0);
  int it = 0;
  for (int64_t u = u_begin; u < u_end;) {
    const int64_t rb = u / a.part.num_kb;
    const int64_t u0 = rb * a.part.num_kb;
    const int64_t seg_end = min64(u_end, u0 + a.part.num_kb);
    T acc[RPT][NT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[r][j] = T(0);

    for (int64_t uu = u; uu < seg_end; ++uu, ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
      mbar_wait(&full[s], ph);
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
      warp_release(&empty[s]);
    }

    const int64_t row0 = rb * R + lrow;
    const bool whole = (u == u0) && (seg_end == u0 + a.part.num_kb);
    if (whole) {
      store_c<T, NT, RPT>(a, row0, acc);
    } else {
      finish_partial<T, NT, RPT, R, ConsumerSync>(a, g, rb, lrow, acc, s_flag, leader, ConsumerSync());
    }
    u = seg_end;
  }
}

}  // namespace tsm2x
