// fp32 TSM2R / TSM2L on the 5th-generation tensor cores: split-precision tf32 (tcgen05.mma
// kind::tf32, accumulators in tensor memory) — the production fp32 path for 16-column passes.
//
// Why. At n = 16 the packed-FFMA2 consumer needs ~60 TFLOP/s of FP32 to keep up with HBM, ~80 %
// of the FP32 pipe at full clock and more than it has once the part sits at its 1000 W cap
// (profiles/README.md). Moving the products onto the tensor core leaves the SM one subtraction
// per element of A.
//
// Arithmetic. The tensor core reads fp32 operands as tf32 by truncating the 13 low mantissa bits
// (measured: tools/tc_probe.cu). With hi(x) = x & ~0x1fff and lo(x) = x - hi(x) (exact in fp32),
//   a*b ~= hi(a)hi(b) + hi(a)lo(b) + lo(a)hi(b)        (the dropped lo(a)lo(b) is < 2^-22 |ab|)
// computed as two MMAs per 8-column k-step and 128-row tile into one accumulator D[128 x 32]:
//   D          += A     x [B | lo(B)]   A straight from the TMA-written stage (the tensor core
//                                        truncates it to hi(A) itself), B operand from smem
//   D[:, 0:16] += lo(A) x B             lo(A) written to tensor memory by the converter warps
// and C = D[:, 0:16] + D[:, 16:32] in the epilogue. Measured error of the split product:
// 3e-7 relative (tc_probe). Accumulation: fp32 in TMEM over a segment of SEG stages (128
// columns), then round-to-nearest fp32 in the converter warps' registers over an item's
// segments, fp64 across split row blocks.
//
// Layouts. A (column-major, rows contiguous) is MN-major: a 3-D TMA box {32 rows, 16 columns,
// 16 row chunks} with the 128B/32B-atom swizzle lands as [chunk][column][32 rows] — the UMMA
// SWIZZLE_128B_BASE32B canonical layout (LBO = 2 KB between 32-row chunks, SBO = 512 B between
// 4-column groups). B and lo(B) are prepared K-major (SWIZZLE_64B, 32 N-rows x 16 K) by
// prep_tc32, one 2 KB block per stage, bulk-copied next to the A stage. lo(A) sits in TMEM as
// 128 lanes (rows) x 16 columns (K) per tile.
//
// Roles (576 threads, one CTA per SM): warp 0 producer (same dynamic item queue and order as
// tsm2r_stream_tma), warp 1 TMEM allocator + MMA issuer (one lane), warps 2-17 converters and
// epilogue. Converter warp w handles TMEM lane quarter w % 4 (the only lanes it may touch) of
// tile (w - 2) / 4 (with -DTSM2X_TC32_CW=8: 320 threads, warps 2-9, tiles {2h, 2h + 1}). Pipelines: full/empty (TMA <-> MMA, empty released by
// tcgen05.commit), lo_full (converters -> MMA, 4 TMEM slots: the converters run up to four stages
// ahead of the tensor core; a slot is reused once the stage four back has released its smem
// stage), acc_full/acc_empty (MMA <-> converters, 2 accumulator buffers alternating per segment;
// a segment is drained one segment late, so the drain never waits on MMAs still in flight).
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "tsm2r_tma.cuh"

// Diagnostic build (nvcc -DTSM2X_TC32_DIAG; tools/tc32_diag.sh): per-stage cycle counters of the
// MMA and converter loops and skip bits (TSM2X_TC_DIAG) that drop pieces of the pipeline.
#ifdef TSM2X_TC32_DIAG
#define TC32_DIAG(...) __VA_ARGS__
#define TC32_SKIP(bit) (a.diag & (bit))
#else
#define TC32_DIAG(...)
#define TC32_SKIP(bit) false
#endif

namespace tsm2x {

struct Tc32Cfg {
  static constexpr int R = 512;            // rows per row block (4 MMA tiles of 128)
  static constexpr int TILES = R / 128;
  static constexpr int KC = 16;            // columns per stage: 512 x 16 x 4 B = 32 KB
  static constexpr int STAGES = 6;
  static constexpr int A_BYTES = R * KC * 4;
  static constexpr int B_BYTES = 32 * KC * 4;  // [B | lo(B)] K-major, 2 KB
  // converter warps: 16 (one 128-row tile per warp; default: -0.45 % burst, -0.6 % sustained at
  // configs[3] vs 8 warps of two tiles, profiles/tc32_cw_r02.json) or 8 (-DTSM2X_TC32_CW=8)
#ifndef TSM2X_TC32_CW
#define TSM2X_TC32_CW 16
#endif
  static constexpr int CONV_WARPS = TSM2X_TC32_CW;
  static constexpr int TPW = TILES * 4 / CONV_WARPS;  // tiles per converter warp (a warp owns one TMEM lane quarter)
  static_assert(TPW >= 1 && TPW * CONV_WARPS == TILES * 4, "converter warps cover every (tile, lane quarter)");
  // accumulation segment: the tensor core's fp32 accumulation (not round-to-nearest: 2048-column
  // chains measured 2.5e-5 relative at K = 32768) is drained into fp64 every SEG stages
  static constexpr int SEG = 8;
  static constexpr int THREADS = 32 * (2 + CONV_WARPS);
  // TMEM columns: 2 accumulator buffers x 4 tiles x 32, then LO_SLOTS lo(A) slots x 4 tiles x 16
  static constexpr int ACC_COLS = 32;
  static constexpr int BUF_COLS = TILES * ACC_COLS;  // 128
  static constexpr int LO_BASE = 2 * BUF_COLS;       // 256
  static constexpr int LO_COLS = TILES * KC;         // 64 per slot
  static constexpr int LO_SLOTS = 4;
  static constexpr int TMEM_COLS = 512;
  static_assert(LO_BASE + LO_SLOTS * LO_COLS <= TMEM_COLS, "TMEM budget");
  // smem: A stages, B stages, barriers (full, empty per stage; lo_full per slot;
  // acc_full, acc_empty x 2), meta per stage, TMEM base address
  static constexpr int BAR_OFF = STAGES * (A_BYTES + B_BYTES);
  static constexpr int NBARS = 2 * STAGES + LO_SLOTS + 4;
  static_assert(LO_SLOTS < STAGES, "a TMEM slot is recycled through the smem stage's empty barrier");
  static constexpr int META_OFF = BAR_OFF + NBARS * 8;
  static constexpr int TMEM_OFF = META_OFF + STAGES * 16;
  static constexpr int SMEM = TMEM_OFF + 16 + 1024;  // + slack to align the stages to 1 KB
};

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)(layout & 7) << 61);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, majors (1 = MN), N, M
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem desc] x B[smem desc]
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] x B[smem desc]
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}


__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}" : "=r"(p));
  return p != 0;
}

// lo(x) = x - hi(x), hi(x) = x with the 13 low mantissa bits cleared (what the tensor core reads).
// Non-finite x: lo = 0 (hi keeps the inf / NaN, so non-finite inputs give non-finite outputs;
// an infinity can surface as NaN through inf * 0 in the cross terms — DESIGN.md §4).
__device__ __forceinline__ float tf32_lo(float a) {
  const uint32_t u = __float_as_uint(a);
  return (u & 0x7F800000u) == 0x7F800000u ? 0.0f : a - __uint_as_float(u & 0xFFFFE000u);
}

// 16 columns of one TMEM lane quarter (tcgen05.st 32x32b.x16), and the matching loads
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&d)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
        "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
      : "r"(addr)
      : "memory");
}
// tcgen05.wait::ld, with the loaded registers tied to it so no use is scheduled above the wait
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&a)[16], uint32_t (&b)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(a[j]), "+r"(b[j])::"memory");
}

// DEFER: single-chunk row blocks (TSM2L) — an item's epilogue runs after the next item's first
// stage is converted (see finish_item); split row blocks (TSM2R) use the plain order.
template <bool DEFER>
__global__ void __launch_bounds__(Tc32Cfg::THREADS, 1)
    tsm2r_stream_tc32(const DynArgs<float> a, const __grid_constant__ CUtensorMap tmA) {
  using Cfg = Tc32Cfg;
  constexpr int STAGES = Cfg::STAGES, KC = Cfg::KC, R = Cfg::R;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KB-aligned stages (the swizzle atoms are address based); offset arithmetic on the shared
  // array keeps every access an LDS/STS (an integer round trip would turn them into generic LDs)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = smem;                                  // STAGES x 32 KB
  unsigned char* sB = smem + STAGES * Cfg::A_BYTES;           // STAGES x 2 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* lo_full = empty + STAGES;              // [LO_SLOTS]
  uint64_t* acc_full = lo_full + Cfg::LO_SLOTS;    // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  longlong2* meta = reinterpret_cast<longlong2*>(smem + Cfg::META_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::TMEM_OFF);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int j = 0; j < Cfg::LO_SLOTS; ++j) mbar_init(&lo_full[j], Cfg::CONV_WARPS * kArrivalsPerWarp);
    for (int j = 0; j < 2; ++j) {
      mbar_init(&acc_full[j], 1);
      mbar_init(&acc_empty[j], Cfg::CONV_WARPS * kArrivalsPerWarp);
    }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch_dependents();  // only tsm2_finalize is launched as a programmatic dependent
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch as in tsm2r_stream_tma: the producer fills the ring with A
  // before waiting for the prep kernel (Bcat, zeroed accumulator); the other warps wait at once.

  if (warp == 0) {
    // ---------------- producer: same queue, item order and stage tagging as tsm2r_stream_tma
    if (lane == 0) {
      const uint64_t pol = policy_for(a.l2pol);
      int it = 0;
      bool prep_done = false;
      int npend = 0;
      int pend_s[STAGES];
      int64_t pend_col[STAGES];
      auto flush_bt = [&]() {
        pdl_wait();
        prep_done = true;
        for (int i = 0; i < npend; ++i)
          bulk_g2s(sB + (size_t)pend_s[i] * Cfg::B_BYTES,
                   reinterpret_cast<const unsigned char*>(a.Bt) + (pend_col[i] / KC) * Cfg::B_BYTES, Cfg::B_BYTES,
                   &full[pend_s[i]]);
        npend = 0;
      };
      bool first_grab = true;  // static first grab, as tsm2r_stream_tma
      for (;;) {
        const int64_t first =
            first_grab ? (int64_t)blockIdx.x * a.it.batch
                       : (int64_t)gridDim.x * a.it.batch + (int64_t)atomicAdd(a.queue, (unsigned long long)a.it.batch);
        first_grab = false;
        if (first >= a.it.total) break;
        const int64_t last = min64(first + a.it.batch, a.it.total);
        for (int64_t item = first; item < last; ++item) {
          int64_t rb, col0, col1;
          a.it.decode(item, a.k, &rb, &col0, &col1);
          const uint32_t tx = (uint32_t)(Cfg::A_BYTES + Cfg::B_BYTES);  // OOB rows/columns are zero-filled
          const int64_t nst = (col1 - col0 + KC - 1) / KC;
          for (int64_t col = col0; col < col1; col += KC, ++it) {
            const int s = it % STAGES;
            const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
            mbar_wait_sleep(&empty[s], ph ^ 1u);
            meta[s] = make_longlong2(rb | (nst << 32), item);  // read by the consumers once per item
            mbar_arrive_expect_tx(&full[s], tx);
            tma_load_3d(sA + (size_t)s * Cfg::A_BYTES, &tmA, 0, (int)col, (int)(rb * (R / 32)), &full[s], pol);
            if (prep_done) {
              bulk_g2s(sB + (size_t)s * Cfg::B_BYTES, reinterpret_cast<const unsigned char*>(a.Bt) + (col / KC) * Cfg::B_BYTES,
                       Cfg::B_BYTES, &full[s]);
            } else {
              pend_s[npend] = s;
              pend_col[npend] = col;
              if (++npend == STAGES) flush_bt();
            }
          }
        }
      }
      if (!prep_done) flush_bt();
      const int s = it % STAGES;
      mbar_wait_sleep(&empty[s], ((uint32_t)(it / STAGES) & 1u) ^ 1u);
      meta[s] = make_longlong2(-1, -1);
      mbar_arrive(&full[s]);
      __threadfence();
      const unsigned prev = atomicAdd(reinterpret_cast<unsigned*>(a.queue + 1), 1u);
      if (prev == gridDim.x - 1) {
        a.queue[0] = 0ull;
        a.queue[1] = 0ull;
        __threadfence();
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    // ---------------- MMA issuer: the whole warp walks the pipeline, one elected lane issues.
    // The issue path is a single dependent instruction stream sharing its SM sub-partition with
    // two converter warps, so it is kept short: descriptors are built once per stage and the
    // per-MMA variants are 32-bit adds on the start-address field; one commit per stage (the
    // converters reuse a TMEM slot after the stage that last used it has released its smem).
    constexpr uint32_t ID1 = umma_idesc_tf32(128, 32, 1, 0);  // A MN-major (smem), B K-major, N = 32
    constexpr uint32_t ID2 = umma_idesc_tf32(128, 16, 0, 0);  // A from TMEM, N = 16 (B rows 0-15)
    // descriptor high words: SBO = 512 B, version 1, layout (SW128_BASE32B = 1 for A, SW64 = 4 for B)
    constexpr uint32_t A_HI = (512u >> 4) | (1u << 14) | (1u << 29);
    constexpr uint32_t B_HI = (512u >> 4) | (1u << 14) | (4u << 29);
    constexpr uint32_t A_LBO = (2048u >> 4) << 16;  // between 32-row chunks
    int64_t cur = -1;
    int left = 0;           // stages of the current item still to come
    int seg = -1, sin = 0;  // segment (accumulator buffer seg & 1) and stages issued into it
    uint32_t acc0 = 1;
    TC32_DIAG(unsigned long long c_full = 0, c_lo = 0, c_issue = 0, c_acc = 0, n_st = 0;)
    for (int it = 0;; ++it) {
      const int s = it % STAGES;
      TC32_DIAG(const unsigned long long t0c = clock64();)
      mbar_wait_sleep(&full[s], (uint32_t)(it / STAGES) & 1u);
      TC32_DIAG(const unsigned long long t1c = clock64(); c_full += t1c - t0c;)
      if (left == 0 || sin == Cfg::SEG) {
        // new item, or SEG stages into the current segment: close the segment (its accumulators
        // go to the converters, which fold them into fp64) and start the next one from zero
        if (cur >= 0 && elect_one()) tc_commit(&acc_full[seg & 1]);
        __syncwarp();
        if (left == 0) {
          // read by lane 0 (the lane elect_one picks in this converged warp, which also commits
          // the stage's release) and broadcast: the read is then ordered before that release
          // by program order rather than by the warp's convergence
          longlong2 md = make_longlong2(0, 0);
          if (lane == 0) md = meta[s];
          md.x = __shfl_sync(0xffffffffu, md.x, 0);
          md.y = __shfl_sync(0xffffffffu, md.y, 0);
          if (md.y < 0) break;
          cur = md.y;
          left = (int)(md.x >> 32);
        }
        ++seg;
        sin = 0;
        TC32_DIAG(const unsigned long long ta = clock64();)
        mbar_wait_sleep(&acc_empty[seg & 1], ((uint32_t)(seg >> 1) & 1u) ^ 1u);
        TC32_DIAG(c_acc += clock64() - ta;)
        acc0 = 0;
      }
      ++sin;
      --left;
      const int slot = it % Cfg::LO_SLOTS;
      TC32_DIAG(const unsigned long long t2c = clock64();)
      mbar_wait_sleep(&lo_full[slot], (uint32_t)(it / Cfg::LO_SLOTS) & 1u);
      TC32_DIAG(const unsigned long long t3c = clock64(); c_lo += t3c - t2c;)
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a_lo = (smem_u32(sA + (size_t)s * Cfg::A_BYTES) >> 4) | A_LBO;
        const uint32_t b_lo = smem_u32(sB + (size_t)s * Cfg::B_BYTES) >> 4;
        const uint32_t acc_col = tmem + (uint32_t)((seg & 1) * Cfg::BUF_COLS);
        const uint32_t lo_col = tmem + (uint32_t)(Cfg::LO_BASE + slot * Cfg::LO_COLS);
#pragma unroll
        for (int t = 0; t < Cfg::TILES; ++t)
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {
            const uint64_t da = ((uint64_t)A_HI << 32) | (a_lo + t * 512 + ks * 64);  // + t*8 KB + ks*1 KB
            const uint64_t db = ((uint64_t)B_HI << 32) | (b_lo + ks * 2);             // + ks*32 B
#ifdef TSM2X_TC32_DIAG
            if (!(a.diag & 2)) umma_ss(acc_col + t * Cfg::ACC_COLS, da, db, ID1, ks == 0 ? acc0 : 1u);
            if (!(a.diag & 1))
              umma_ts(acc_col + t * Cfg::ACC_COLS, lo_col + t * KC + ks * 8, db, ID2,
                      (a.diag & 2) ? (ks == 0 ? acc0 : 1u) : 1u);
#else
            umma_ss(acc_col + t * Cfg::ACC_COLS, da, db, ID1, ks == 0 ? acc0 : 1u);
            umma_ts(acc_col + t * Cfg::ACC_COLS, lo_col + t * KC + ks * 8, db, ID2, 1u);  // after ID1: accumulate
#endif
          }
        tc_commit(&empty[s]);
      }
      __syncwarp();
      acc0 = 1;
      TC32_DIAG(c_issue += clock64() - t3c; ++n_st;)
    }
    TC32_DIAG(if (a.dbg && lane == 0) {
      atomicAdd(a.dbg + 0, c_full);
      atomicAdd(a.dbg + 1, c_lo);
      atomicAdd(a.dbg + 2, c_issue);
      atomicAdd(a.dbg + 3, c_acc);
      atomicAdd(a.dbg + 4, n_st);
    })
  } else {
    // ---------------- converters + epilogue
    pdl_wait();
    const int cw = warp - 2;        // 0..7
    const int q = warp & 3;         // TMEM lane quarter this warp may access
    const int t0 = Cfg::TPW * (cw >> 2);  // tiles t0 .. t0 + TPW - 1
    const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
    int64_t cur = -1, cur_rb = 0;
    int left = 0;                      // stages of the current item still to come
    int seg = -1, pend = -1, sin = 0;  // current segment, segment awaiting its drain, stages in segment
    // this thread's row of tiles t0, t0 + 1: running sums of the drained segments (fp32 with
    // round-to-nearest over ~16 segment values; fp64 would not fit the 168-register budget)
    float sum[Cfg::TPW][16];
#pragma unroll
    for (int tt = 0; tt < Cfg::TPW; ++tt)
#pragma unroll
      for (int j = 0; j < 16; ++j) sum[tt][j] = 0.f;
    TC32_DIAG(unsigned long long c_full = 0, c_loe = 0, c_conv = 0, c_epi = 0;)
    // fold segment g's accumulators (buffer g & 1) into the fp64 sums and hand the buffer back
    auto drain = [&](int g) {
      mbar_wait_sleep(&acc_full[g & 1], (uint32_t)(g >> 1) & 1u);
      tc_fence_after();
#pragma unroll
      for (int tt = 0; tt < Cfg::TPW; ++tt) {
        const uint32_t base = tmem + lane_addr + (uint32_t)((g & 1) * Cfg::BUF_COLS + (t0 + tt) * Cfg::ACC_COLS);
        uint32_t dh[16], dl[16];
        tmem_ld16(base, dh);       // A x B + lo(A) x B
        tmem_ld16(base + 16, dl);  // A x lo(B)
        tmem_ld_wait(dh, dl);
#pragma unroll
        for (int j = 0; j < 16; ++j) sum[tt][j] += __uint_as_float(dh[j]) + __uint_as_float(dl[j]);
      }
      tc_fence_before();
      __syncwarp();
      warp_release(&acc_empty[g & 1]);
    };
    // An item's epilogue is deferred until the converters have prepared the next item's first
    // stage: by then the tensor core has finished the item's last MMAs, so the drain does not
    // stall (TSM2L's single-stage items otherwise serialised convert -> MMA -> drain -> store)
    bool fin_pending = false;
    int64_t fin_rb = 0;
    int fin_pend = -1, fin_seg = 0;
    auto finish_item = [&]() {
      if (!fin_pending) return;
      fin_pending = false;
      if (fin_pend >= 0) drain(fin_pend);
      drain(fin_seg);
      const int64_t nch = a.it.nch();
#pragma unroll
      for (int tt = 0; tt < Cfg::TPW; ++tt) {
        const int64_t row = fin_rb * R + (t0 + tt) * 128 + 32 * q + lane;
        if (row < a.m) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j >= a.w) break;
            if (nch == 1) {
              float* cp = a.C + j * a.ldc + row;
              __stcs(cp, a.c_is_zero ? sum[tt][j] : __ldcs(cp) + sum[tt][j]);
            } else {
              red_add(a.acc + j * a.ldacc + row, (double)sum[tt][j]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) sum[tt][j] = 0.f;
      }
    };
    for (int it = 0;; ++it) {
      const int s = it % STAGES;
      TC32_DIAG(const unsigned long long t0c = clock64();)
      mbar_wait_sleep(&full[s], (uint32_t)(it / STAGES) & 1u);
      TC32_DIAG(const unsigned long long t1c = clock64(); c_full += t1c - t0c;)
      if (left == 0) {
        const longlong2 md = meta[s];
        if (cur >= 0) {  // item done: drain its older pending segment now (its MMAs finished
                         // long ago; the tensor core wants that buffer next), the last segment
                         // and the write-out after this stage's conversion
          if (pend >= 0) drain(pend);
          fin_pending = true;
          fin_rb = cur_rb;
          fin_pend = -1;
          fin_seg = seg;
          pend = -1;
        }
        // split row blocks (long items) finish at once; single-chunk ones (TSM2L: one or two
        // stages per item) after the next stage's conversion — sustained A/B: deferring gains
        // 9 % on TSM2L fp32 and cost 3-5 % on TSM2R fp32 n=16 (hence the two instantiations)
        if (md.y < 0 || !DEFER) finish_item();
        TC32_DIAG(c_epi += clock64() - t1c;)
        if (md.y < 0) break;
        cur = md.y;
        cur_rb = md.x & 0xffffffffll;
        left = (int)(md.x >> 32);
        ++seg;
        sin = 0;
      } else if (sin == Cfg::SEG) {
        // segment boundary inside the item: drain the segment before last (its buffer is the one
        // the tensor core needs next), keep the last one pending so this never waits on MMAs
        // still in flight
        if (pend >= 0) drain(pend);
        pend = seg;
        ++seg;
        sin = 0;
      }
      ++sin;
      --left;
      const int slot = it % Cfg::LO_SLOTS;
      TC32_DIAG(const unsigned long long t2c = clock64();)
      if (it >= Cfg::LO_SLOTS) {  // the slot's previous stage (it - LO_SLOTS) has finished its MMAs
        const int pj = it - Cfg::LO_SLOTS;
        mbar_wait_sleep(&empty[pj % STAGES], (uint32_t)(pj / STAGES) & 1u);
      }
      TC32_DIAG(const unsigned long long t3c = clock64(); c_loe += t3c - t2c;)
      tc_fence_after();
      const unsigned char* st = sA + (size_t)s * Cfg::A_BYTES;
#pragma unroll
      for (int tt = 0; tt < Cfg::TPW; ++tt) {
        const int t = t0 + tt;
        // row 128t + 32q + lane lives in 32-row chunk 4t + q; column k at (k/4)*512 + (k%4)*128,
        // 32-byte unit (lane/8) ^ (k%4), word lane%8
        const unsigned char* cbase = st + (4 * t + q) * 2048 + (lane & 7) * 4;
        uint32_t v[16];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const float x = TC32_SKIP(4) ? 1.0f + k : *reinterpret_cast<const float*>(cbase + (k >> 2) * 512 + (k & 3) * 128 + (((lane >> 3) ^ (k & 3)) * 32));
          v[k] = __float_as_uint(tf32_lo(x));
        }
        if (!TC32_SKIP(8)) tmem_st16(tmem + lane_addr + (uint32_t)(Cfg::LO_BASE + slot * Cfg::LO_COLS + t * KC), v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      warp_release(&lo_full[slot]);
      TC32_DIAG(const unsigned long long t4c = clock64(); c_conv += t4c - t3c;)
      if constexpr (DEFER) finish_item();  // the previous item's epilogue, if one is pending
      TC32_DIAG(c_epi += clock64() - t4c;)
    }
    TC32_DIAG(if (a.dbg && cw == 0 && lane == 0) {
      atomicAdd(a.dbg + 8, c_full);
      atomicAdd(a.dbg + 9, c_loe);
      atomicAdd(a.dbg + 10, c_conv);
      atomicAdd(a.dbg + 11, c_epi);
    })
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::TMEM_COLS) : "memory");
}

// [B | lo(B)] per stage of 16 B rows: 32 N-rows x 16 K, K-major, SWIZZLE_64B (16-byte unit
// (k/4) ^ ((n/2) % 4) of the 64-byte row n), one 2 KB block per stage; rows >= k and columns >= w
// are zero. Also zeroes the split-combine target (fp64 accumulator) like prep_dyn.
__global__ void prep_tc32(const float* __restrict__ B, int64_t ldb, int64_t k, int64_t nstages, int w,
                          float* __restrict__ Bt, double* __restrict__ zp, int64_t zld, int64_t zrows, int zcols) {
  pdl_launch_dependents();
  const int64_t nb = nstages * 512, nz = zp ? zrows * zcols : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb + nz; i += stride) {
    if (i < nb) {
      const int64_t st = i / 512;
      const int e = (int)(i % 512), n = e / 16, kk = e % 16;
      const int64_t row = st * 16 + kk;
      const int col = n & 15;
      const float b = (row < k && col < w) ? B[row + col * ldb] : 0.f;
      const float v = n < 16 ? b : tf32_lo(b);
      const int off = n * 16 + (((kk >> 2) ^ ((n >> 1) & 3)) * 4) + (kk & 3);  // in floats
      Bt[st * 512 + off] = v;
    } else {
      const int64_t z = i - nb, col = z / zrows, row = z - col * zrows;
      zp[row + col * zld] = 0.0;
    }
  }
}

}  // namespace tsm2x
