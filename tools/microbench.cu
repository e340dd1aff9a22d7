// B200 micro-benchmarks that set the roofline denominators the driver does not measure:
// read-only HBM stream (LDG.128 and cp.async.bulk), DFMA / DMMA / FFMA / FFMA2 peaks,
// pinned H2D / D2H bandwidth. Build: make -C tools microbench ; run under gpurun.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <string>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

// ---------------------------------------------------------------- read stream (LDG.128)
template <int U>
__global__ void read_ldg(const double2* __restrict__ p, size_t n2, double* sink) {
  double acc = 0.0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                   : "=d"(v[u].x), "=d"(v[u].y) : "l"(p + i + u * stride));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) acc += p[i].x;
  if (acc == 12345.678) *sink = acc;
}

// ---------------------------------------------------------------- read stream (bulk copy)
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(b);
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
// one thread per CTA issues bulk copies into a STAGES-deep ring; all threads "consume" (sum) it.
template <int STAGES, int CHUNK>
__global__ void read_bulk(const char* __restrict__ p, size_t nchunks, double* sink) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], blockDim.x / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t first = blockIdx.x, step = gridDim.x;
  int niter = first < nchunks ? (int)((nchunks - first + step - 1) / step) : 0;
  if (threadIdx.x == 0) {
    for (int it = 0; it < min(niter, STAGES); ++it) {
      mbar_expect(&full[it], CHUNK);
      bulk_g2s(smem + it * CHUNK, p + (first + it * step) * CHUNK, CHUNK, &full[it]);
    }
  }
  double acc = 0;
  for (int it = 0; it < niter; ++it) {
    int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
    mbar_wait(&full[s], ph);
    const double2* t = reinterpret_cast<const double2*>(smem + s * CHUNK);
    for (int j = threadIdx.x; j < CHUNK / 16; j += blockDim.x) acc += t[j].x;
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&empty[s])) : "memory");
    if (threadIdx.x == 0 && it + STAGES < niter) {
      mbar_wait(&empty[s], ph);
      mbar_expect(&full[s], CHUNK);
      bulk_g2s(smem + s * CHUNK, p + (first + (it + STAGES) * step) * CHUNK, CHUNK, &full[s]);
    }
  }
  if (acc == 12345.678) *sink = acc;
}

// ---------------------------------------------------------------- FP peaks
__global__ void dfma_peak(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1.2345) *out = s;
}
__global__ void ffma_peak(float* out, int iters) {
  float a[16], b = 1.0000001f, c = 0.9999999f;
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], b, c);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += a[j];
  if (s == 1.2345f) *out = s;
}
__global__ void ffma2_peak(float* out, int iters) {
  unsigned long long a[8];
  float2 bb = make_float2(1.0000001f, 1.0000001f), cc = make_float2(0.9999999f, 0.9999999f);
  unsigned long long b = *reinterpret_cast<unsigned long long*>(&bb), c = *reinterpret_cast<unsigned long long*>(&cc);
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 t = make_float2(threadIdx.x + j, j); a[j] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(b), "l"(c));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 t = *reinterpret_cast<float2*>(&a[j]); s += t.x + t.y; }
  if (s == 1.2345f) *out = s;
}
__global__ void dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { d[j][0] = j; d[j][1] = -j; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  if (s == 1.2345) *out = s;
}

// half the warps DMMA, half DFMA: do the two share the FP64 datapath?
__global__ void mixed_fp64_peak(double* out, int iters) {
  const int w = threadIdx.x / 32;
  double s = 0;
  if (w & 1) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double d[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) { d[j][0] = j; d[j][1] = -j; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  } else {
    double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
    // DFMA warps do 8x the iterations' worth of lanes-FMAs to match DMMA work per warp: one DMMA
    // (256 FMA) == 8 warp-DFMAs (32 FMA each)
    for (int i = 0; i < iters * 8; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
  }
  if (s == 1.2345) *out = s;
}

static float time_kernel(void (*launch)(), int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  launch(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); launch(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
  }
  return best;
}

static double2* g_buf; static size_t g_n2; static double* g_sink; static int g_grid, g_block;
static void* g_fp;
static int g_iters;

int main(int argc, char** argv) {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  if (argc > 1 && std::string(argv[1]) == "--sustain") {
    size_t bytes = (size_t)8 << 30;
    CK(cudaMalloc(&g_buf, bytes)); CK(cudaMemset(g_buf, 0, bytes)); CK(cudaMalloc(&g_sink, 64));
    g_n2 = bytes / 16;
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    const bool bulk = argc > 2 && std::string(argv[2]) == "bulk";
    constexpr int ST = 4, CH = 16384;
    const size_t bsmem = ST * CH + 2 * ST * 8;
    CK(cudaFuncSetAttribute(read_bulk<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
    for (int i = 0; i < 1000; ++i) {
      if (i == 500) CK(cudaEventRecord(a));
      if (bulk)
        read_bulk<ST, CH><<<sms * 2, 256, bsmem>>>((const char*)g_buf, bytes / CH, g_sink);
      else
        read_ldg<8><<<sms * 2, 512>>>(g_buf, g_n2, g_sink);
    }
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    printf("{\"test\": \"read_%s_sustained_2nd_half\", \"GBps\": %.1f}\n", bulk ? "bulk" : "ldg", 500.0 * bytes / ms / 1e6);
    return 0;
  }
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu}\n", prop.name, sms, prop.l2CacheSize, prop.sharedMemPerBlockOptin);
  size_t bytes = (size_t)8 << 30;  // 8 GiB, far above L2
  CK(cudaMalloc(&g_buf, bytes)); CK(cudaMemset(g_buf, 0, bytes)); CK(cudaMalloc(&g_sink, 64));
  g_n2 = bytes / 16;
  // LDG stream sweep
  for (int block : {256, 512}) for (int occ : {1, 2, 4, 8}) {
    g_block = block; g_grid = sms * occ;
    if (block * occ > 2048) continue;
    float ms = time_kernel([] { read_ldg<8><<<g_grid, g_block>>>(g_buf, g_n2, g_sink); }, 5);
    printf("{\"test\": \"read_ldg_u8\", \"block\": %d, \"grid\": %d, \"GBps\": %.1f}\n", block, g_grid, bytes / ms / 1e6);
  }
  for (int occ : {2, 4}) {
    g_block = 256; g_grid = sms * occ;
    float ms = time_kernel([] { read_ldg<16><<<g_grid, g_block>>>(g_buf, g_n2, g_sink); }, 5);
    printf("{\"test\": \"read_ldg_u16\", \"block\": 256, \"grid\": %d, \"GBps\": %.1f}\n", g_grid, bytes / ms / 1e6);
  }
  // bulk-copy stream
  {
    constexpr int ST = 6, CH = 32768;
    size_t smem = ST * CH + 2 * ST * 8;
    CK(cudaFuncSetAttribute(read_bulk<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    g_grid = sms; g_block = 256;
    static size_t s_smem; s_smem = smem;
    float ms = time_kernel([] { read_bulk<6, 32768><<<g_grid, g_block, s_smem>>>((const char*)g_buf, (size_t(8) << 30) / 32768, g_sink); }, 5);
    printf("{\"test\": \"read_bulk_6x32K\", \"grid\": %d, \"GBps\": %.1f}\n", g_grid, bytes / ms / 1e6);
  }
  {
    constexpr int ST = 4, CH = 16384;
    size_t smem = ST * CH + 2 * ST * 8;
    CK(cudaFuncSetAttribute(read_bulk<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    g_grid = sms * 2; g_block = 256;
    static size_t s_smem; s_smem = smem;
    float ms = time_kernel([] { read_bulk<4, 16384><<<g_grid, g_block, s_smem>>>((const char*)g_buf, (size_t(8) << 30) / 16384, g_sink); }, 5);
    printf("{\"test\": \"read_bulk_4x16K_occ2\", \"grid\": %d, \"GBps\": %.1f}\n", g_grid, bytes / ms / 1e6);
  }
  // FP peaks: flops = grid*block*iters*chains*2 (*256/32 per lane for DMMA)
  CK(cudaMalloc(&g_fp, 64));
  g_grid = sms * 8; g_block = 256; g_iters = 4096;
  {
    float ms = time_kernel([] { dfma_peak<<<g_grid, g_block>>>((double*)g_fp, g_iters); }, 5);
    double fl = double(g_grid) * g_block * g_iters * 8 * 2;
    printf("{\"test\": \"dfma_peak\", \"TFLOPs\": %.2f}\n", fl / ms / 1e9);
  }
  {
    float ms = time_kernel([] { dmma_peak<<<g_grid, g_block>>>((double*)g_fp, g_iters); }, 5);
    double fl = double(g_grid) * (g_block / 32) * g_iters * 8 * 256 * 2;
    printf("{\"test\": \"dmma_m8n8k4_peak\", \"TFLOPs\": %.2f}\n", fl / ms / 1e9);
  }
  {
    float ms = time_kernel([] { mixed_fp64_peak<<<g_grid, g_block>>>((double*)g_fp, g_iters); }, 5);
    double fl = double(g_grid) * (g_block / 32) * g_iters * 8 * 256 * 2;  // both halves do the same FMAs
    printf("{\"test\": \"mixed_dmma_dfma_peak\", \"TFLOPs\": %.2f}\n", fl / ms / 1e9);
  }
  {
    float ms = time_kernel([] { ffma_peak<<<g_grid, g_block>>>((float*)g_fp, g_iters); }, 5);
    double fl = double(g_grid) * g_block * g_iters * 16 * 2;
    printf("{\"test\": \"ffma_peak\", \"TFLOPs\": %.2f}\n", fl / ms / 1e9);
  }
  {
    float ms = time_kernel([] { ffma2_peak<<<g_grid, g_block>>>((float*)g_fp, g_iters); }, 5);
    double fl = double(g_grid) * g_block * g_iters * 8 * 2 * 2;
    printf("{\"test\": \"ffma2_peak\", \"TFLOPs\": %.2f}\n", fl / ms / 1e9);
  }
  // pinned H2D / D2H
  {
    size_t hb = (size_t)1 << 30;
    void* h; CK(cudaMallocHost(&h, hb)); memset(h, 1, hb);
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    float best = 1e30f, bestd = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(a)); CK(cudaMemcpyAsync(g_buf, h, hb, cudaMemcpyHostToDevice)); CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
      CK(cudaEventRecord(a)); CK(cudaMemcpyAsync(h, g_buf, hb, cudaMemcpyDeviceToHost)); CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); bestd = std::min(bestd, ms);
    }
    printf("{\"test\": \"pinned_h2d\", \"GBps\": %.1f}\n{\"test\": \"pinned_d2h\", \"GBps\": %.1f}\n", hb / best / 1e6, hb / bestd / 1e6);
  }
  return 0;
}
