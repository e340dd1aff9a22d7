// TSM2R / TSM2L stream kernel, TMA flavour — the production path on sm_100a.
//
// Work decomposition. A (m x k, column-major) is cut into items = (row block of R rows, column
// chunk). Items are handed out dynamically (atomicAdd on a global queue), so every SM keeps
// streaming until the queue is empty whatever DRAM bandwidth it happens to get: per-SM
// bandwidth on B200 varies by ~10 %, which a static split turns straight into tail time
// (profiles/README.md). Item sizes shrink towards the end of the queue — "big" chunks cover the
// first ~80 % of every row block's columns and are dispatched first, "small" chunks the rest —
// so the last items finish within ~10 us of each other. Row blocks split into several chunks
// are combined by fire-and-forget fp64 reductions (red.global.add.f64) into C (fp64) or into
// an fp64 accumulator (fp32, converted by tsm2_finalize). A row block that is a single chunk
// (TSM2L shapes: k small) is written with plain vector stores — and, under the zero-C
// contract, C is never read.
//
// Per CTA: warp 0 is the producer — one elected lane takes items off the queue and, per stage
// of KC columns, issues 2-D TMA tensor loads of the A tile (R rows x KC columns as R/256 boxes
// of 256 rows; rows >= m and columns >= k arrive zero-filled) plus a 1-D bulk copy of the KC
// matching rows of Bt, completing on the stage's "full" mbarrier, and tags the stage with its
// item. Warps 1..CW are consumers: thread ct owns rows ct + 256*r (one per TMA box), reads them
// with conflict-free LDS (32 consecutive elements per warp) and the Bt row as broadcast
// LDS.128s, and keeps the NT outputs per row in registers; one lane per warp releases the stage on its "empty"
// mbarrier. A STAGES-deep ring keeps ~(STAGES-1) * 32 KB of A in flight per SM independent of
// register pressure — the B200 replacement for the paper's register double buffer (Alg 4,
// PAPER.md:290-333) and of its t1 x t2 shared B tile (Alg 3).
#pragma once
#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "tsm2r_stream.cuh"

// Diagnostic build (nvcc -DTSM2X_TC32_DIAG, `make diag`): per-stage cycle counters.
#ifdef TSM2X_TC32_DIAG
#define KDIAG(...) __VA_ARGS__
#else
#define KDIAG(...)
#endif

namespace tsm2x {

template <typename T, int NT, int RPT_ = Vec<T>::N, int CW_ = 8, int SB_ = 32768>
struct TmaCfg {
  static constexpr int CW = CW_;                      // consumer warps
  static constexpr int CT = 32 * CW;                  // consumer threads
  static constexpr int THREADS = 32 * (CW + 1);       // + producer warp
  static constexpr int RPT = RPT_;                    // rows per consumer thread (one per TMA box)
  static constexpr int R = CT * RPT;                  // rows per row block (512 fp64 / 1024 fp32)
  static constexpr int BOX = 256;                     // rows per TMA box (box dim limit)
  static constexpr int NBOX = R / BOX;
  static constexpr int SB = SB_;                      // A bytes per stage (32 KB; 64 KB experiment)
  static constexpr int KC = SB / (R * (int)sizeof(T));  // columns per stage (8 by default)
  static_assert(KC >= 1 && (KC * NT * (int)sizeof(T)) % 16 == 0, "bulk-copy granularity");
  static constexpr int STAGES = 196608 / SB;           // 192 KB of A in the ring
  static constexpr int A_ELEMS = R * KC;
  static constexpr int B_ELEMS = KC * NT;
  static constexpr int A_BYTES = A_ELEMS * (int)sizeof(T);
  static constexpr int B_BYTES = B_ELEMS * (int)sizeof(T);
  static constexpr int B_BYTES_PAD = (B_BYTES + 127) / 128 * 128;
  static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES_PAD) + 2 * STAGES * 8 + STAGES * 16 + 16;
};

// Item geometry: per row block, nbig chunks of kbig columns over [0, kbig_end), then nsmall
// chunks of ksmall columns over [kbig_end, k). Ids: all big items, then all small items, each
// class COLUMN-CHUNK major (row block fastest): the CTAs in flight work on the same columns of
// neighbouring row blocks, so DRAM sees each column (contiguous in memory) read end to end at
// about the same time — row-buffer friendly. Row-block-major order read scattered 4 KB pieces
// and cost ~150 W more at the same bandwidth, which the 1000 W cap turned into SM clock
// (profiles/README.md). batch > 1 (single-chunk row blocks only) hands out that many
// consecutive items per queue access.
struct Items {
  int64_t num_rb;
  int64_t nbig, kbig, kbig_end;
  int64_t nsmall, ksmall;
  int64_t total;
  int64_t batch;
  __host__ __device__ int64_t nch() const { return nbig + nsmall; }
  // column-chunk index (0 .. nch-1, increasing with the columns) of an item
  __device__ int64_t chunk(int64_t id) const {
    const int64_t n_big_items = num_rb * nbig;
    return id < n_big_items ? id / num_rb : nbig + (id - n_big_items) / num_rb;
  }
  __device__ void decode(int64_t id, int64_t k, int64_t* rb, int64_t* c0, int64_t* c1) const {
    const int64_t n_big_items = num_rb * nbig;
    if (id < n_big_items) {
      const int64_t c = id / num_rb;
      *rb = id - c * num_rb;
      *c0 = c * kbig;
      *c1 = min64(*c0 + kbig, kbig_end);
    } else {
      const int64_t j = id - n_big_items;
      const int64_t c = j / num_rb;
      *rb = j - c * num_rb;
      *c0 = kbig_end + c * ksmall;
      *c1 = min64(*c0 + ksmall, k);
    }
  }
};

template <typename T>
struct DynArgs {
  const T* Bt;      // kpad x NT row-major copy of this pass of B, zero padded
  T* C;
  int64_t ldc;
  int64_t m, k;
  int w;            // valid columns in this pass (<= NT)
  int c_is_zero;    // single-chunk row blocks: C is written, never read
  int vec_c;        // C columns 16-B aligned (vector stores allowed)
  double* acc;      // reduction combine, fp32: fp64 accumulator [NT][ldacc] (zeroed); fp64: null (C)
  int64_t ldacc;
  int ordered;      // split row blocks: 1 = chunk-ordered combine through per-row-block tickets
                    // (deterministic), 0 = fp64 atomic reductions
  unsigned* tickets;  // [num_rb] next chunk allowed to update the row block; zero between launches
  Items it;
  unsigned long long* queue;  // [0] next item, [1] low 32 bits: producers finished
  const T* B = nullptr;  // inline_b: the pass's B (k x w, column-major, ldb) — no prep kernel
  int64_t ldb = 0;
  int inline_b = 0;      // 1: the producer warp builds each stage's Bt rows from B itself
  int l2pol = 0;                      // L2 policy of the A stream (policy_for; TSM2X_L2POL)
  int diag = 0;                       // tsm2r_stream_tc32 diagnostics (TSM2X_TC_DIAG): skip bits
  unsigned long long* dbg = nullptr;  // tsm2r_stream_tc32 diagnostics: cycle counters (or null)
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Consumers that take A in the swizzled layout (DmmaConsumer<..., SWZ = true>) declare kSwz.
template <typename C, typename = void>
struct SwzOf : std::false_type {};
template <typename C>
struct SwzOf<C, std::void_t<decltype(C::kSwz)>> : std::integral_constant<bool, C::kSwz> {};

// Element i of Bt (the per-pass copy of B the stage ring reads): row-major kpad x NT (FMA /
// FFMA2 consumers) or, FRAG, DMMA fragment order — for each group of 4 B rows (kg) and N tile
// (nt) the 32 values in lane order, lane (g = lane/4, t = lane%4) holding B[row][8nt + g] with
// row = 4kg + t, or on the swizzled A layout row = 8(kg/2) + 2t + kg%2 (k-step kg takes columns
// {0,2,4,6} / {1,3,5,7} of an 8-column group). Zero outside k x w. Used by prep_dyn and by the
// stream kernel's inline-B producer.
template <typename T, int NT, bool FRAG>
__device__ __forceinline__ T bt_elem(const T* __restrict__ B, int64_t ldb, int64_t k, int w, bool swz, int64_t i) {
  if constexpr (FRAG) {
    const int lane = (int)(i % 32);
    const int64_t tile = i / 32;
    const int nt = (int)(tile % (NT / 8));
    const int64_t kg = tile / (NT / 8);
    const int64_t row = swz ? 8 * (kg >> 1) + 2 * (lane & 3) + (kg & 1) : 4 * kg + (lane & 3);
    const int col = 8 * nt + (lane >> 2);
    return (row < k && col < w) ? __ldg(B + row + col * ldb) : T(0);
  } else {
    const int64_t c = i / NT;
    const int j = (int)(i - c * NT);
    return (j < w && c < k) ? __ldg(B + c + j * ldb) : T(0);
  }
}

// Inverse of bt_elem: the Bt index of B[row][col] (row < kpad, col < NT).
template <int NT, bool FRAG>
__device__ __forceinline__ int64_t bt_index(int64_t row, int col, bool swz) {
  if constexpr (FRAG) {
    const int nt = col >> 3, g = col & 7;
    int64_t kg;
    int t;
    if (swz) {
      const int within = (int)(row & 7);
      kg = 2 * (row >> 3) + (within & 1);
      t = within >> 1;
    } else {
      kg = row >> 2;
      t = (int)(row & 3);
    }
    return (kg * (NT / 8) + nt) * 32 + g * 4 + t;
  } else {
    return row * NT + col;
  }
}

// Inline-B producer: a stage's "full" barrier completes on the TMA bytes plus the producer warp's
// arrival after its B stores — lane 0's after __syncwarp in the production build; every lane's in
// the racecheck build (compute-sanitizer racecheck does not follow the __syncwarp edge, see
// common.cuh warp_release), whose barriers then count 32 arrivals.
#ifdef TSM2X_RACECHECK
constexpr int kInlineFullArrivals = 32;
__device__ __forceinline__ void inline_publish(uint64_t* bar) { mbar_arrive(bar); }
#else
constexpr int kInlineFullArrivals = 1;
__device__ __forceinline__ void inline_publish(uint64_t* bar) {
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
#endif

// Consumers that read B in DMMA fragment order (every DmmaConsumer, which declares kSwz).
template <typename C, typename = void>
struct FragOf : std::false_type {};
template <typename C>
struct FragOf<C, std::void_t<decltype(C::kSwz)>> : std::true_type {};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

struct ConsumerSync {  // named barrier over the consumer warps (every warp but the producer)
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x - 32) : "memory");
  }
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Ordered combine of split row blocks: chunk c of row block rb may update C only after chunks
// 0..c-1 did (ticket == c), so C's rows receive their partial sums in column order whatever
// CTA ran which item — bitwise reproducible. Column-chunk-major dispatch hands chunk c of a row
// block out ~one round of items before chunk c+1, so the wait is rarely long; the pause costs
// 2-30 % (profiles/abtest_r01b.json), which is why it is opt-in (deterministic=True).
// Called by all consumer threads; the leader spins, the named barrier publishes its acquire.
__device__ __forceinline__ void ticket_wait(const unsigned* tick, unsigned chunk, bool leader) {
  if (leader)
    while (ld_acquire(tick) != chunk) __nanosleep(128);
  ConsumerSync()();
}
// All consumers' C stores precede the barrier; the leader's release store hands the row block on.
__device__ __forceinline__ void ticket_pass(unsigned* tick, unsigned next, bool leader) {
  ConsumerSync()();
  if (leader) st_release(tick, next);
}

// Epilogue of one item. Consumer thread ct owns rows ct + 256*r (r < RPT) of the row block, so
// every warp-wide access below touches 32 consecutive elements of a C column: coalesced stores
// for single-chunk row blocks (C (+)= acc), coalesced fp64 reductions for split row blocks
// (into C for fp64, into the fp64 accumulator for fp32).
template <typename T, int NT, int RPT, int R, int CT = 256>
__device__ __forceinline__ void finish_item(const DynArgs<T>& a, int64_t rb, int64_t item, int ct,
                                            const T (&acc)[RPT][NT]) {
  const int64_t row_base = rb * R + ct;
  const int64_t nch = a.it.nch();
  const int64_t c = nch == 1 ? 0 : a.it.chunk(item);
  if (nch == 1 || a.ordered) {
    if (nch > 1) ticket_wait(a.tickets + rb, (unsigned)c, ct == 0);
    // the first chunk starts from C's input (or from zero under the zero-C contract)
    const bool read_c = c > 0 || !a.c_is_zero;
    if (!read_c) {
      // zero-C single-chunk row blocks (TSM2L): plain streaming stores, C never read
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        if (j >= a.w) continue;
        T* cj = a.C + j * a.ldc;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int64_t row = row_base + r * CT;
          if (row < a.m) __stcs(cj + row, acc[r][j]);
        }
      }
    } else {
      // loads of a group of columns first (one round trip per group, not per element), then
      // their stores; groups of 4 columns bound the live registers (a whole 16-column tile of
      // loaded C spilled at RPT = 4)
      constexpr int G = NT < 4 ? NT : 4;
#pragma unroll
      for (int j0 = 0; j0 < NT; j0 += G) {
        T old[RPT][G];
#pragma unroll
        for (int jj = 0; jj < G; ++jj)
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int64_t row = row_base + r * CT;
            old[r][jj] = (j0 + jj < a.w && row < a.m) ? __ldcg(a.C + (j0 + jj) * a.ldc + row) : T(0);
          }
#pragma unroll
        for (int jj = 0; jj < G; ++jj) {
          if (j0 + jj >= a.w) continue;
          T* cj = a.C + (j0 + jj) * a.ldc;
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int64_t row = row_base + r * CT;
            if (row < a.m) {
              if (nch == 1)
                __stcs(cj + row, old[r][jj] + acc[r][j0 + jj]);
              else
                __stcg(cj + row, old[r][jj] + acc[r][j0 + jj]);
            }
          }
        }
      }
    }
    if (nch > 1) ticket_pass(a.tickets + rb, c + 1 == nch ? 0u : (unsigned)(c + 1), ct == 0);
    return;
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j >= a.w) continue;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int64_t row = row_base + r * CT;
      if constexpr (sizeof(T) == 8) {
        if (row < a.m) red_add(reinterpret_cast<double*>(a.C) + j * a.ldc + row, (double)acc[r][j]);
      } else {
        if (a.acc)
          red_add(a.acc + j * a.ldacc + row, (double)acc[r][j]);  // accumulator padded to whole row blocks
        else if (row < a.m)  // small fp32 calls: fp32 reductions straight into C (one launch per call)
          red_add(reinterpret_cast<float*>(a.C) + j * a.ldc + row, (float)acc[r][j]);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// Consumer policies: how one stage (R rows x KC columns of A in smem, the matching Bt rows) is
// folded into the per-thread accumulators, and how an item's accumulators leave the CTA.

// FMA: thread ct owns rows ct + 256*r; one scalar LDS per row per column (32 consecutive
// elements per warp, conflict-free), Bt row as broadcast LDS.128s, NT FMAs per row per column.
template <typename T, int NT, int RPT_ = Vec<T>::N, int CW_ = 8, int SB_ = 32768>
struct FmaConsumer {
  using Cfg = TmaCfg<T, NT, RPT_, CW_, SB_>;
  using V = typename Vec<T>::type;
  static constexpr int RPT = Cfg::RPT;
  static constexpr bool kFragB = false;
  static constexpr bool kPipelined = false;
  T acc[RPT][NT];
  int ct;
  __device__ __forceinline__ void init(int consumer_thread) {
    ct = consumer_thread;
    zero();
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[r][j] = T(0);
  }
  __device__ __forceinline__ void stage(const T* sA, const T* sB) {
#pragma unroll
    for (int cc = 0; cc < Cfg::KC; ++cc) {
      T av[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int row = ct + r * Cfg::CT;  // row in the block -> (TMA box, offset in the box)
        av[r] = sA[(row / Cfg::BOX) * (Cfg::BOX * Cfg::KC) + cc * Cfg::BOX + row % Cfg::BOX];
      }
      T b[NT];
      if constexpr (NT * sizeof(T) >= 16) {
        constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
        for (int i = 0; i < NT / PER; ++i) {
          const V bv = reinterpret_cast<const V*>(sB + cc * NT)[i];
#pragma unroll
          for (int e = 0; e < PER; ++e) b[i * PER + e] = vget<T>(bv, e);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NT; ++i) b[i] = sB[cc * NT + i];
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[r][j] = fma(av[r], b[j], acc[r][j]);
    }
  }
  __device__ __forceinline__ void finish(const DynArgs<T>& a, int64_t rb, int64_t item) const {
    finish_item<T, NT, RPT, Cfg::R, Cfg::CT>(a, rb, item, ct, acc);
  }
};

// FFMA2 (fp32): as FmaConsumer, but output columns are processed in pairs with the packed
// fma.rn.f32x2 (one issue slot per two FMAs; the FP32 pipe, not issue, bounds n = 16).
template <int NT>
struct Ffma2Consumer {
  using Cfg = TmaCfg<float, NT>;
  static constexpr int RPT = Cfg::RPT;
  static constexpr bool kFragB = false;
  static constexpr bool kPipelined = false;
  static_assert(NT % 2 == 0, "pairs of columns");
  unsigned long long acc[RPT][NT / 2];  // packed (col 2p, col 2p+1)
  int ct;
  __device__ __forceinline__ void init(int consumer_thread) {
    ct = consumer_thread;
    zero();
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int p = 0; p < NT / 2; ++p) acc[r][p] = 0ull;
  }
  __device__ __forceinline__ void stage(const float* sA, const float* sB) {
    const float* As = sA + ct;
#pragma unroll
    for (int cc = 0; cc < Cfg::KC; ++cc) {
      unsigned long long a2[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const float av = As[r * (Cfg::BOX * Cfg::KC) + cc * Cfg::BOX];
        asm("mov.b64 %0, {%1, %1};" : "=l"(a2[r]) : "f"(av));
      }
      unsigned long long b2[NT / 2];
      const unsigned long long* bp = reinterpret_cast<const unsigned long long*>(sB + cc * NT);
#pragma unroll
      for (int p = 0; p < NT / 2; ++p) b2[p] = bp[p];
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int p = 0; p < NT / 2; ++p) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[r][p]) : "l"(a2[r]), "l"(b2[p]));
    }
  }
  __device__ __forceinline__ void finish(const DynArgs<float>& a, int64_t rb, int64_t item) const {
    float out[RPT][NT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int p = 0; p < NT / 2; ++p) asm("mov.b64 {%0, %1}, %2;" : "=f"(out[r][2 * p]), "=f"(out[r][2 * p + 1]) : "l"(acc[r][p]));
    finish_item<float, NT, RPT, Cfg::R>(a, rb, item, ct, out);
  }
};

// DMMA (fp64, NT in {8, 16}): the FP64 tensor-core MMA m8n8k4 (DMMA.8x8x4). Warp w owns rows
// [64w, 64w+64) of the row block as four 16-row groups; one LDS.128 per lane loads rows
// (2g, 2g+1) of column t of a group — two A fragments (M tiles of the even and the odd rows) for
// 8 lanes x 4 columns (4 wavefronts when conflict-free: see SWZ below). Bt is staged in fragment order (prep_bfrag)
// so each B fragment is one LDS.64 per lane. 32 DMMAs per warp per stage replace 256 DFMAs and
// 64 LDS.128 of the FMA consumer; the FP64 datapath is shared (measured), so this buys issue
// slots and power, not peak.
//
// SWZ (the default geometry): A arrives as one 3-D TMA box {16 rows, KC columns, 32 row chunks}
// with the 128-byte swizzle, i.e. smem [chunk][column][16 rows] where the 16-byte piece p of
// column c sits at position p ^ (c % 8). In the plain [column][row] layout every column is a
// multiple of 128 B away from the next, so the 8 lanes of an LDS.128 phase — rows (2g, 2g+1)
// for two g and four columns t — hit the same banks: 4-way conflicts, 16 wavefronts per
// instruction instead of 4 (ncu at config 2: 243 M shared wavefronts, 177 M of them conflicts;
// the smem pipe 83 % busy). With the swizzle and the k-step's four columns taken as
// {0, 2, 4, 6} / {1, 3, 5, 7} of each 8-column group (B's fragment order permuted to match,
// prep_dyn), a phase's eight pieces land on eight distinct positions.
template <int NT, int CW_ = 8, bool PIPE_ = false, int SB_ = 32768, bool SWZ_ = false, int RB_ = 512>
struct DmmaConsumer {
  // R = RB_ rows per row block: 512 (CW_ = 8 warps x 64 rows, or 16 x 32), or 1024 (16 warps x
  // 64 rows; TSM2X_RB=1024 experiment: 8 KB contiguous per column per stage)
  using Cfg = TmaCfg<double, NT, RB_ / (32 * CW_), CW_, SB_>;
  static constexpr bool kFragB = true;
  static constexpr bool kSwz = SWZ_;
  static_assert(!SWZ_ || Cfg::KC % 8 == 0, "swizzled layout: whole 8-column groups per stage");
  static constexpr bool kPipelined = PIPE_;  // k-step software pipeline (kernel loop below)
  static_assert(NT == 8 || NT == 16, "DMMA consumer needs NT in {8, 16}");
  static_assert(CW_ == 8 || CW_ == 16, "DMMA consumer: 8 or 16 consumer warps");
  static constexpr int NTI = NT / 8;       // N tiles
  static constexpr int RW = Cfg::R / CW_;  // rows per warp (64 or 32)
  static constexpr int Q = RW / 16;        // 16-row groups per warp
  double acc[Q][2][NTI][2];                // [row group][M tile (even/odd rows)][N tile][2 columns]
  int warp, lane;
  __device__ __forceinline__ void init(int consumer_thread) {
    warp = consumer_thread / 32;
    lane = consumer_thread % 32;
    zero();
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) acc[q][mt][nt][0] = acc[q][mt][nt][1] = 0.0;
  }
  // Per k-step of 4 columns: the B fragments (one LDS.64 per N tile), then per 16-row group one
  // LDS.128 (rows 2g, 2g+1 of column t) feeding the even- and odd-row M tiles. (A variant that
  // loaded a whole stage's fragments first — and a look-ahead loop loading stage s+1 before stage
  // s's DMMAs — spilled at n=16 and was slower under the power cap: profiles/envab_r01.json.)
  // One k-step's fragments (4 columns): the pipelined loop holds two of these, loading k-step j+1
  // while the DMMAs of k-step j issue, so the LDS latency hides behind the tensor pipe.
  static constexpr int KS = Cfg::KC / 4;
  struct Frag {
    double b[NTI];
    double2 av[Q];
  };
  KDIAG(int dg = 0;)  // diagnostic build: 16 = no fragment LDS (constants), 32 = no DMMA
  // A fragment pair (rows 2g, 2g+1 of 16-row group q, k-step column t) of k-step ks
  __device__ __forceinline__ const double2* a_ptr(const double* sA, int ks, int q) const {
    const int g = lane >> 2, t = lane & 3;
    if constexpr (SWZ_) {
      const int c = 8 * (ks >> 1) + 2 * t + (ks & 1);  // column within the stage
      const int ch = RW * warp / 16 + q;               // 16-row chunk within the row block
      return reinterpret_cast<const double2*>(sA + ch * (Cfg::KC * 16) + c * 16 + 2 * (g ^ (c & 7)));
    } else {
      const double* As = sA + (RW * warp / Cfg::BOX) * (Cfg::BOX * Cfg::KC) + (RW * warp % Cfg::BOX + 2 * g);
      return reinterpret_cast<const double2*>(As + (4 * ks + t) * Cfg::BOX + 16 * q);
    }
  }
  __device__ __forceinline__ void load_ks(const double* sA, const double* sB, int ks, Frag& f) const {
    KDIAG(if (dg & 16) {
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) f.b[nt] = 1.0 + ks;
#pragma unroll
      for (int q = 0; q < Q; ++q) f.av[q] = make_double2(lane + q, lane - q);
      return;
    })
#pragma unroll
    for (int nt = 0; nt < NTI; ++nt) f.b[nt] = sB[(ks * NTI + nt) * 32 + lane];
#pragma unroll
    for (int q = 0; q < Q; ++q) f.av[q] = *a_ptr(sA, ks, q);
  }
  __device__ __forceinline__ void mma_ks(const Frag& f) {
    KDIAG(if (dg & 32) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) acc[q][0][nt][0] += f.av[q].x + f.av[q].y + f.b[nt];
      return;
    })
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[q][0][nt][0]), "+d"(acc[q][0][nt][1]) : "d"(f.av[q].x), "d"(f.b[nt]));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[q][1][nt][0]), "+d"(acc[q][1][nt][1]) : "d"(f.av[q].y), "d"(f.b[nt]));
      }
  }
  __device__ __forceinline__ void stage(const double* sA, const double* sB) {
#pragma unroll
    for (int ks = 0; ks < Cfg::KC / 4; ++ks) {
      double b[NTI];
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) b[nt] = sB[(ks * NTI + nt) * 32 + lane];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double2 av = *a_ptr(sA, ks, q);
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[q][0][nt][0]), "+d"(acc[q][0][nt][1]) : "d"(av.x), "d"(b[nt]));
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[q][1][nt][0]), "+d"(acc[q][1][nt][1]) : "d"(av.y), "d"(b[nt]));
        }
      }
    }
  }
  // accumulator (q, mt, nt, e) holds row RW*w + 16q + 2g + mt, column 8nt + 2t + e
  __device__ __forceinline__ void finish(const DynArgs<double>& a, int64_t rb, int64_t item) const {
    const int g = lane >> 2, t = lane & 3;
    const int64_t base = rb * Cfg::R + RW * warp + 2 * g;
    const int64_t nch = a.it.nch();
    const int64_t c = nch == 1 ? 0 : a.it.chunk(item);
    const bool rmw = nch == 1 || a.ordered;
    if (!rmw) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int64_t row = base + 16 * q + mt;
          if (row >= a.m) continue;
#pragma unroll
          for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int j = 8 * nt + 2 * t + e;
              if (j < a.w) red_add(a.C + j * a.ldc + row, acc[q][mt][nt][e]);
            }
        }
      return;
    }
    const bool leader = warp == 0 && lane == 0;
    if (nch > 1) ticket_wait(a.tickets + rb, (unsigned)c, leader);
    const bool read_c = c > 0 || !a.c_is_zero;
    if (a.vec_c && rb * Cfg::R + Cfg::R <= a.m) {
      // whole row block, 16-B aligned C: the lane's two rows (2g, 2g+1) of a column are adjacent,
      // so each access is one 16-byte vector and a warp instruction covers four full 128-B lines
      // (8 row pairs x 4 columns) instead of eight half-filled sectors per column
      // one 16-row group at a time (its loads, then its stores): keeps the live registers to
      // one group's C values — the whole tile's would push the n=16 kernel into spills
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        double2 old[NTI][2];
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = 8 * nt + 2 * t + e;
            old[nt][e] = (read_c && j < a.w) ? __ldcg(reinterpret_cast<const double2*>(a.C + j * a.ldc + base + 16 * q))
                                              : make_double2(0.0, 0.0);
          }
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = 8 * nt + 2 * t + e;
            if (j >= a.w) continue;
            const double2 v = make_double2(old[nt][e].x + acc[q][0][nt][e], old[nt][e].y + acc[q][1][nt][e]);
            double2* dst = reinterpret_cast<double2*>(a.C + j * a.ldc + base + 16 * q);
            if (nch == 1)
              __stcs(dst, v);
            else
              __stcg(dst, v);
          }
      }
      if (nch > 1) ticket_pass(a.tickets + rb, c + 1 == nch ? 0u : (unsigned)(c + 1), leader);
      return;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {  // one 16-row group at a time (register pressure, see above)
      double old[2][NTI][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t row = base + 16 * q + mt;
            const int j = 8 * nt + 2 * t + e;
            old[mt][nt][e] = (read_c && row < a.m && j < a.w) ? __ldcg(a.C + j * a.ldc + row) : 0.0;
          }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int64_t row = base + 16 * q + mt;
        if (row >= a.m) continue;
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = 8 * nt + 2 * t + e;
            if (j < a.w) __stcg(a.C + j * a.ldc + row, old[mt][nt][e] + acc[q][mt][nt][e]);
          }
      }
    }
    if (nch > 1) ticket_pass(a.tickets + rb, c + 1 == nch ? 0u : (unsigned)(c + 1), leader);
  }
};

// Diagnostic only (TSM2X_CONSUMER=null): touches one element per stage and writes nothing —
// isolates the cost (time, power) of the TMA pipeline itself from the arithmetic. Results are
// garbage by design; never selected automatically.
template <typename T, int NT, int RPT_ = Vec<T>::N, int CW_ = 8, int SB_ = 32768>
struct NullConsumer {
  using Cfg = TmaCfg<T, NT, RPT_, CW_, SB_>;
  static constexpr bool kFragB = false;
  static constexpr bool kPipelined = false;
  T sink;
  int ct;
  __device__ __forceinline__ void init(int consumer_thread) {
    ct = consumer_thread;
    sink = T(0);
  }
  __device__ __forceinline__ void zero() {}
  __device__ __forceinline__ void stage(const T* sA, const T* sB) { sink += sA[ct] * sB[0]; }
  __device__ __forceinline__ void finish(const DynArgs<T>& a, int64_t rb, int64_t item) const {
    if (sink == T(12345.678)) a.C[0] = sink;
  }
};

template <typename T, int NT, typename Consumer>
__global__ void __launch_bounds__(Consumer::Cfg::THREADS, 1)
    tsm2r_stream_tma(const DynArgs<T> a, const __grid_constant__ CUtensorMap tmA) {
  using Cfg = typename Consumer::Cfg;  // row-block height / stage width of this consumer
  constexpr int R = Cfg::R, KC = Cfg::KC, STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* sA = reinterpret_cast<T*>(smem);
  T* sB = reinterpret_cast<T*>(smem + STAGES * Cfg::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (Cfg::A_BYTES + Cfg::B_BYTES_PAD));
  uint64_t* empty = full + STAGES;
  // per stage: (row block | stages in the item << 32, item id); id -1 = end
  longlong2* meta = reinterpret_cast<longlong2*>(empty + STAGES);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // diagnostic build: per-CTA timeline (globaltimer ns) at dbg[16 + 5*cta + {0 entry, 1 first TMA
  // issue, 2 first stage landed, 3 producer done, 4 consumers done}]
  KDIAG(unsigned long long* tl = a.dbg ? a.dbg + 16 + 5 * blockIdx.x : nullptr;
        if (tl && threadIdx.x == 0) tl[0] = gtimer();)
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], a.inline_b ? kInlineFullArrivals : 1);
      mbar_init(&empty[s], Cfg::CW * kArrivalsPerWarp);
    }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
  }
  __syncthreads();
  pdl_launch_dependents();  // only tsm2_finalize is launched as a programmatic dependent
  // Programmatic dependent launch: Bt and the zeroed accumulation target come from the prep
  // kernel, A does not. The producer fills the ring with A tiles first and waits for prep only
  // before the first Bt copy is due (the stage barriers expect both); the consumers wait at once
  // (they write C / the accumulator, which prep may have zeroed).

  if (warp == 0 && a.inline_b) {
    // ---------------- producer, inline B (one launch per call, no prep kernel).
    // The whole warp runs the loop. Lane 0 takes items and issues the A tensor loads exactly as
    // the prep-fed producer does; the 32 lanes gather each stage's KC rows of B (in the
    // consumer's Bt order, bt_elem) into registers and store them next to the A tile one
    // iteration later — after the NEXT stage's tensor load has been issued — so the gather's
    // L2 latency never sits between a free slot and its TMA issue. A stage's barrier expects the
    // TMA bytes (expect_tx, no arrival) before its loads are issued and completes on lane 0's
    // arrival after the B stores (__syncwarp orders the other lanes' stores before it).
    // Launched without programmatic serialization, so A and B are complete when the kernel starts.
    const uint64_t pol = policy_for(a.l2pol);
    constexpr int PER = (Cfg::B_ELEMS + 31) / 32;
    constexpr bool kFrag = FragOf<Consumer>::value;
    constexpr bool kSwzB = SwzOf<Consumer>::value;
    // stage cursor: current item range [item, last), the item's row block and column range
    int64_t item = 0, last = 0, rb = 0, col = 0, col1 = 0, nst = 0;
    int nbox = 0;
    auto open_item = [&]() {
      int64_t col0;
      a.it.decode(item, a.k, &rb, &col0, &col1);
      col = col0;
      nst = (col1 - col0 + KC - 1) / KC;
      nbox = (int)min64(Cfg::NBOX, (a.m - rb * R + Cfg::BOX - 1) / Cfg::BOX);
    };
    // the first grab of every CTA is static (item block blockIdx.x), later ones from the queue
    auto grab = [&](bool first_grab) -> bool {
      int64_t first;
      if (first_grab) {
        first = (int64_t)blockIdx.x * a.it.batch;
      } else {
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(a.queue, (unsigned long long)a.it.batch);
        q = __shfl_sync(0xffffffffu, q, 0);
        first = (int64_t)gridDim.x * a.it.batch + (int64_t)q;
      }
      if (first >= a.it.total) return false;
      item = first;
      last = min64(first + a.it.batch, a.it.total);
      open_item();
      return true;
    };
    bool have = grab(true);
    int it = 0;
    T v[PER];
    int prev_s = -1;  // slot whose B rows are in v, still to be stored and published
    while (have) {
      const int s = it % STAGES;
      const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
#ifdef TSM2X_RACECHECK
      mbar_wait(&empty[s], ph ^ 1u);  // racecheck build: every lane acquires the slot it writes
#endif
      if (lane == 0) {  // one lane polls (32 polling lanes would take smem cycles from the consumers)
        mbar_wait(&empty[s], ph ^ 1u);
        KDIAG(if (tl && it == 0) tl[1] = gtimer();)
        meta[s] = make_longlong2(rb | (nst << 32), item);
        mbar_expect_tx(&full[s], kSwzB ? (uint32_t)Cfg::A_BYTES : (uint32_t)(nbox * Cfg::BOX * KC * (int)sizeof(T)));
        if constexpr (kSwzB) {
          tma_load_3d(sA + (size_t)s * Cfg::A_ELEMS, &tmA, 0, (int)col, (int)(rb * R / 16), &full[s], pol);
        } else {
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(sA + (size_t)s * Cfg::A_ELEMS + b * (Cfg::BOX * KC), &tmA, (int)(rb * R + b * Cfg::BOX),
                        (int)col, &full[s], pol);
        }
      }
      if (prev_s >= 0) {  // the previous stage's B rows (gathered one iteration ago)
        T* dst = sB + (size_t)prev_s * (Cfg::B_BYTES_PAD / sizeof(T));
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int idx = lane + 32 * j;
          if (idx < Cfg::B_ELEMS) dst[bt_index<NT, kFrag>(idx % KC, idx / KC, kSwzB)] = v[j];
        }
        __syncwarp();
        inline_publish(&full[prev_s]);
      }
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int idx = lane + 32 * j;
        // source order (KC consecutive rows of one B column per group of KC lanes: whole 128-B
        // lines per warp load); the stores scatter into the consumer's Bt order (bt_index)
        const int r = idx % KC, c = idx / KC;
        v[j] = (idx < Cfg::B_ELEMS && col + r < a.k && c < a.w) ? __ldg(a.B + (col + r) + (int64_t)c * a.ldb) : T(0);
      }
      prev_s = s;
      ++it;
      // advance the cursor: next stage of this item, next item of the batch, or a new grab
      col += KC;
      if (col >= col1) {
        if (++item < last)
          open_item();
        else
          have = grab(false);
      }
    }
    if (prev_s >= 0) {
      T* dst = sB + (size_t)prev_s * (Cfg::B_BYTES_PAD / sizeof(T));
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int idx = lane + 32 * j;
        if (idx < Cfg::B_ELEMS) dst[bt_index<NT, kFrag>(idx % KC, idx / KC, kSwzB)] = v[j];
      }
    }
    __syncwarp();
    if (prev_s >= 0) inline_publish(&full[prev_s]);
    {  // end-of-work marker for the consumers
      const int s = it % STAGES;
      if (lane == 0) {
        KDIAG(if (tl) tl[3] = gtimer();)
        mbar_wait(&empty[s], ((uint32_t)(it / STAGES) & 1u) ^ 1u);
        meta[s] = make_longlong2(-1, -1);
      }
      __syncwarp();
      inline_publish(&full[s]);
    }
    if (lane == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(reinterpret_cast<unsigned*>(a.queue + 1), 1u);
      if (prev == gridDim.x - 1) {
        a.queue[0] = 0ull;
        a.queue[1] = 0ull;
        __threadfence();
      }
    }
    return;
  }
  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_for(a.l2pol);
      int it = 0;
      bool prep_done = false;
      int npend = 0;
      int pend_s[STAGES];
      int64_t pend_col[STAGES];
      auto flush_bt = [&]() {  // Bt copies of the stages issued before prep completed
        pdl_wait();
        KDIAG(if (tl) tl[3] = gtimer();)  // overwritten by "producer done" unless the diag asks for prep (bit 64)
        prep_done = true;
        for (int i = 0; i < npend; ++i)
          bulk_g2s(sB + (size_t)pend_s[i] * (Cfg::B_BYTES_PAD / sizeof(T)), a.Bt + pend_col[i] * NT, Cfg::B_BYTES,
                   &full[pend_s[i]]);
        npend = 0;
      };
      // the first grab of every CTA is static (item block blockIdx.x): no queue round trip before
      // the first TMA issue (~0.5 us of a small call); later grabs come from the queue, offset past
      // the gridDim.x static blocks
      bool first_grab = true;
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
          const int64_t row_base = rb * R;
          const int nbox = (int)min64(Cfg::NBOX, (a.m - row_base + Cfg::BOX - 1) / Cfg::BOX);
          // swizzled layout: one 3-D box per stage, always full (out-of-range chunks zero-filled)
          const uint32_t tx = SwzOf<Consumer>::value ? (uint32_t)(Cfg::A_BYTES + Cfg::B_BYTES)
                                                     : (uint32_t)(nbox * Cfg::BOX * KC * (int)sizeof(T) + Cfg::B_BYTES);
          const int64_t nst = (col1 - col0 + KC - 1) / KC;
          for (int64_t col = col0; col < col1; col += KC, ++it) {
            const int s = it % STAGES;
            const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
            mbar_wait(&empty[s], ph ^ 1u);
            KDIAG(if (tl && it == 0) tl[1] = gtimer();)
            meta[s] = make_longlong2(rb | (nst << 32), item);
            mbar_arrive_expect_tx(&full[s], tx);
            if constexpr (SwzOf<Consumer>::value) {
              tma_load_3d(sA + (size_t)s * Cfg::A_ELEMS, &tmA, 0, (int)col, (int)(row_base / 16), &full[s], pol);
            } else {
              for (int b = 0; b < nbox; ++b)
                tma_load_2d(sA + (size_t)s * Cfg::A_ELEMS + b * (Cfg::BOX * KC), &tmA, (int)(row_base + b * Cfg::BOX),
                            (int)col, &full[s], pol);
            }
            if (prep_done) {
              bulk_g2s(sB + (size_t)s * (Cfg::B_BYTES_PAD / sizeof(T)), a.Bt + col * NT, Cfg::B_BYTES, &full[s]);
            } else {
              pend_s[npend] = s;
              pend_col[npend] = col;
              if (++npend == STAGES) flush_bt();  // ring full: nothing more to issue before prep
            }
          }
        }
      }
      if (!prep_done) flush_bt();
      KDIAG(if (tl && !(a.diag & 64)) tl[3] = gtimer();)
      // end-of-work marker for the consumers
      const int s = it % STAGES;
      mbar_wait(&empty[s], ((uint32_t)(it / STAGES) & 1u) ^ 1u);
      meta[s] = make_longlong2(-1, -1);
      mbar_arrive(&full[s]);
      // the last producer out resets the queue for the next launch on this workspace
      __threadfence();
      const unsigned prev = atomicAdd(reinterpret_cast<unsigned*>(a.queue + 1), 1u);
      if (prev == gridDim.x - 1) {
        a.queue[0] = 0ull;
        a.queue[1] = 0ull;
        __threadfence();
      }
    }
    return;
  }

  // ---------------- consumers
  pdl_wait();
  Consumer cons;
  cons.init(threadIdx.x - 32);
  int64_t cur = -1, cur_rb = 0;
  if constexpr (Consumer::kPipelined) {
    // k-step software pipeline (KS = 2 k-steps of 4 columns per stage): while the DMMAs of one
    // k-step issue, the fragments of the next are already loaded; stage s is released as soon as
    // its last fragments are in registers, and the wait for stage s+1 happens with stage s's
    // first-half DMMAs already in the tensor pipe.
    constexpr int KS = Consumer::KS;
    static_assert(KS % 2 == 0, "pipelined loop alternates two fragment sets over an even k-step count");
    typename Consumer::Frag f0, f1;
    KDIAG(cons.dg = a.diag;)
    mbar_wait(&full[0], 0u);
    KDIAG(if (tl && threadIdx.x == 32) tl[2] = gtimer();)
    int left;
    {
      const longlong2 md = meta[0];
      if (md.y < 0) return;  // this CTA got no item
      cur = md.y;
      cur_rb = md.x & 0xffffffffll;
      left = (int)(md.x >> 32) - 1;
    }
    int s = 0;
    cons.load_ks(sA, sB, 0, f0);
    KDIAG(unsigned long long c_wait = 0, c_fin = 0, n_st = 0; const unsigned long long t_start = clock64();)
    for (int it = 1;; ++it) {
      const T* sa = sA + (size_t)s * Cfg::A_ELEMS;
      const T* sb = sB + (size_t)s * (Cfg::B_BYTES_PAD / sizeof(T));
      // k-steps 0 .. KS-2 of stage s: load the next k-step, issue this one; the stage is released
      // once its last k-step's fragments are loaded
#pragma unroll
      for (int ks = 0; ks < KS - 1; ++ks) {
        if (ks % 2 == 0) {
          cons.load_ks(sa, sb, ks + 1, f1);
          if (ks + 1 == KS - 1) {
            __syncwarp();
            warp_release(&empty[s]);
          }
          cons.mma_ks(f0);
        } else {
          cons.load_ks(sa, sb, ks + 1, f0);
          if (ks + 1 == KS - 1) {
            __syncwarp();
            warp_release(&empty[s]);
          }
          cons.mma_ks(f1);
        }
      }
      // last k-step (held in f1, KS even): fetch stage s+1's first k-step into f0 meanwhile
      const int s1 = it % STAGES;
      KDIAG(const unsigned long long tw0 = clock64();)
      mbar_wait(&full[s1], (uint32_t)(it / STAGES) & 1u);
      KDIAG(c_wait += clock64() - tw0; ++n_st;)
      bool end = false, sw = false;
      int64_t nxt = 0, nxt_rb = 0;
      if (left == 0) {
        const longlong2 md = meta[s1];
        end = md.y < 0;
        sw = !end;
        nxt = md.y;
        nxt_rb = md.x & 0xffffffffll;
        left = (int)(md.x >> 32);
      }
      if (!end) cons.load_ks(sA + (size_t)s1 * Cfg::A_ELEMS, sB + (size_t)s1 * (Cfg::B_BYTES_PAD / sizeof(T)), 0, f0);
      cons.mma_ks(f1);
      if (end) {
        cons.finish(a, cur_rb, cur);
        break;
      }
      if (sw) {
        KDIAG(const unsigned long long tf0 = clock64();)
        cons.finish(a, cur_rb, cur);
        cons.zero();
        cur = nxt;
        cur_rb = nxt_rb;
        KDIAG(c_fin += clock64() - tf0;)
      }
      --left;
      s = s1;
    }
    KDIAG(if (a.dbg && threadIdx.x == 32) {
      tl[4] = gtimer();
      atomicAdd(a.dbg + 0, c_wait);
      atomicAdd(a.dbg + 1, clock64() - t_start);  // "stage" = whole loop time
      atomicAdd(a.dbg + 2, c_fin);
      atomicAdd(a.dbg + 4, n_st);
    })
    return;
  }
  int left = 0;  // stages of the current item still to come: meta is read once per item (an LDS
                 // per stage queued behind the fragment loads of all warps cost ~15 % of issue)
  KDIAG(unsigned long long c_wait = 0, c_stage = 0, c_fin = 0, n_st = 0;)
  for (int it = 0;; ++it) {
    const int s = it % STAGES;
    const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
    KDIAG(const unsigned long long t0c = clock64();)
    mbar_wait(&full[s], ph);
    KDIAG(const unsigned long long t1c = clock64(); c_wait += t1c - t0c;
          if (tl && it == 0 && threadIdx.x == 32) tl[2] = gtimer();)
    if (left == 0) {
      const longlong2 md = meta[s];
      if (md.y < 0) {  // end marker (a CTA may get no item at all)
        if (cur >= 0) cons.finish(a, cur_rb, cur);
        break;
      }
      if (cur >= 0) {
        cons.finish(a, cur_rb, cur);
        cons.zero();
      }
      cur = md.y;
      cur_rb = md.x & 0xffffffffll;
      left = (int)(md.x >> 32);
    }
    --left;
    KDIAG(const unsigned long long t2c = clock64(); c_fin += t2c - t1c;)
    cons.stage(sA + (size_t)s * Cfg::A_ELEMS, sB + (size_t)s * (Cfg::B_BYTES_PAD / sizeof(T)));
    __syncwarp();
    warp_release(&empty[s]);
    KDIAG(c_stage += clock64() - t2c; ++n_st;)
  }
  KDIAG(if (a.dbg && threadIdx.x == 32) {
    tl[4] = gtimer();
    atomicAdd(a.dbg + 0, c_wait);
    atomicAdd(a.dbg + 1, c_stage);
    atomicAdd(a.dbg + 2, c_fin);
    atomicAdd(a.dbg + 4, n_st);
  })
}

// Bt in DMMA fragment order: for each group of 4 B rows (kg) and N tile (nt), the 32 values in
// lane order, lane (g = lane/4, t = lane%4) holding B[4kg + t][8nt + g]; zero padded like prep_bt.
template <int NT>
__global__ void prep_bfrag(const double* __restrict__ B, int64_t ldb, int64_t k, int64_t kpad, int w,
                           double* __restrict__ Bf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kpad * NT) return;
  const int lane = (int)(i % 32);
  const int64_t tile = i / 32;            // kg * (NT/8) + nt
  const int nt = (int)(tile % (NT / 8));
  const int64_t kg = tile / (NT / 8);
  const int64_t row = 4 * kg + (lane & 3);
  const int col = 8 * nt + (lane >> 2);
  Bf[i] = (row < k && col < w) ? B[row + col * ldb] : 0.0;
}

// Programmatic dependent launch: the prep kernel lets the stream kernel launch (and run its
// prologue: barrier init, tensor-map prefetch) while prep is still running; the stream kernel
// waits for prep's writes (Bt, zeroed accumulator) with griddepcontrol.wait before using them.

// One prep launch per pass of the dynamic kernel: Bt (row-major, or DMMA fragment order when
// FRAG) and, for split row blocks, the zeroed accumulation target (C itself for fp64 under the
// zero-C contract, or the fp64 accumulator for fp32) — zrows x zcols at zp with leading dim zld.
// swz: the swizzled DMMA layout's k-step order (k-step kg takes columns 8 (kg / 2) + 2t + kg % 2).
template <typename T, int NT, bool FRAG, typename Z>
__global__ void prep_dyn(const T* __restrict__ B, int64_t ldb, int64_t k, int64_t kpad, int w, T* __restrict__ Bt,
                         Z* __restrict__ zp, int64_t zld, int64_t zrows, int zcols, int swz = 0) {
  pdl_launch_dependents();
  const int64_t nb = kpad * NT, nz = zp ? zrows * zcols : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb + nz; i += stride) {
    if (i < nb) {
      Bt[i] = bt_elem<T, NT, FRAG>(B, ldb, k, w, swz != 0, i);
    } else {
      const int64_t z = i - nb, col = z / zrows, row = z - col * zrows;
      zp[row + col * zld] = Z(0);
    }
  }
}

// fp32 split row blocks: C = (float)((double)C + acc) (or (float)acc under the zero-C contract).
template <typename T>
__global__ void tsm2_finalize(const double* __restrict__ acc, int64_t ldacc, T* C, int64_t ldc, int64_t m, int w,
                              int c_is_zero) {
  pdl_wait();  // launched with programmatic dependent launch behind the stream kernel
  const int64_t tot = m * w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / m, r = i - j * m;
    const double v = acc[j * ldacc + r];
    T* c = C + j * ldc + r;
    *c = c_is_zero ? (T)v : (T)((double)*c + v);
  }
}

}  // namespace tsm2x
