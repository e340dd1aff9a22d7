// tcgen05 kind::tf32 probe for the split-precision fp32 consumer: checks, on one CTA,
//  (1) the MN-major SWIZZLE_128B A operand (32-row chunks x 8-column atoms, as a 3-D TMA box
//      writes them) and MN-major SW128 / SW64 B operands,
//  (2) A from tensor memory (tcgen05.st of A_lo rows, K-major in TMEM),
//  (3) how the tensor core reduces fp32 inputs to tf32 (truncation or rounding), which decides how
//      A_lo = A - tf32(A) must be formed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe tools/tc_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)                       // D f32
         | (2u << 7) | (2u << 10)        // A, B tf32
         | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float tf32_trunc(float a) { return __uint_as_float(__float_as_uint(a) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_rna(float a) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(a));
  return __uint_as_float(r);
}

// mode 0: random; lo_mode 0 = a - trunc(a), 1 = a - rna(a); mode 1: rounding probe (no lo terms)
__global__ void probe(const float* A /*128x16 col-major*/, const float* B /*16x16, B[k*16+n]*/, float* out /*128x48*/,
                      int lo_mode) {
  __shared__ __align__(1024) unsigned char sA[128 * 16 * 4];   // 8 KB
  __shared__ __align__(1024) unsigned char sBc[16 * 32 * 4];   // 2 KB: [B_hi | B_lo] N-rows, K-major SW64
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // A: MN-major SWIZZLE_128B_BASE32B (TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 32-row chunk c at
  // c*2048 (LBO), 4-column group g at g*512 (SBO), column k%4 at 128 B, 32-B unit ((r%32)/8) ^ (k%4)
  for (int i = tid; i < 128 * 16; i += blockDim.x) {
    const int r = i % 128, k = i / 128;
    const uint32_t off = (r / 32) * 2048 + (k / 4) * 512 + (k % 4) * 128 + ((((r % 32) / 8) ^ (k % 4)) * 32) + (r % 8) * 4;
    *reinterpret_cast<float*>(sA + off) = A[r + 128 * k];
  }
  // B: K-major SWIZZLE_64B, 32 N-rows (0-15 B_hi = B, 16-31 B_lo) of 16 K values (64 B), 16-B unit
  // (k/4) ^ ((n/2)%4)
  for (int i = tid; i < 16 * 32; i += blockDim.x) {
    const int n = i % 32, k = i / 32;
    const float b = B[k * 16 + (n % 16)];
    const float v = n < 16 ? b : (lo_mode == 0 ? b - tf32_trunc(b) : b - tf32_rna(b));
    const uint32_t off = n * 64 + (((k / 4) ^ ((n >> 1) & 3)) * 16) + (k % 4) * 4;
    *reinterpret_cast<float*>(sBc + off) = v;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  // A_lo rows into TMEM columns 64..79 (lane = row)
  {
    const int r = tid;  // 128 threads
    uint32_t v[16];
    for (int k = 0; k < 16; ++k) {
      const float a = A[r + 128 * k];
      const float lo = lo_mode == 0 ? a - tf32_trunc(a) : a - tf32_rna(a);
      v[k] = __float_as_uint(lo);
    }
    const uint32_t addr = tb + ((uint32_t)(32 * warp) << 16) + 64;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (lo_mode == 2) {  // TMEM st -> ld round trip of the A_lo columns, no MMA
    uint32_t d[16];
    const uint32_t addr = tb + ((uint32_t)(32 * warp) << 16) + 64;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
          "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(d[j])::"memory");
    for (int j = 0; j < 16; ++j) out[tid * 48 + j] = __uint_as_float(d[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(128));
    return;
  }
  if (tid == 0) {
    const uint32_t id1 = idesc_tf32(128, 32, 1, 0), id2 = idesc_tf32(128, 16, 0, 0);
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t da = sdesc(sA + ks * 1024, 2048, 512, 1);
      const uint64_t db = sdesc(sBc + ks * 32, 0, 512, 4);
      const uint32_t en = ks > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tb + 0),
          "l"(da), "l"(db), "r"(id1), "r"(en));
      const uint64_t dbh = db;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tb + 32),
          "r"(tb + 64 + ks * 8), "l"(dbh), "r"(id2), "r"(en));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  // wait for MMA completion
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(smem_u32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t d[48];
    const uint32_t addr = tb + ((uint32_t)(32 * warp) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
        "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
          "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]),
          "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]),
          "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
        : "r"(addr));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[32]), "=r"(d[33]), "=r"(d[34]), "=r"(d[35]), "=r"(d[36]), "=r"(d[37]), "=r"(d[38]), "=r"(d[39]),
          "=r"(d[40]), "=r"(d[41]), "=r"(d[42]), "=r"(d[43]), "=r"(d[44]), "=r"(d[45]), "=r"(d[46]), "=r"(d[47])
        : "r"(addr + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    // tie the loaded registers to the wait so no use is scheduled above it
#pragma unroll
    for (int j = 0; j < 48; ++j) asm volatile("" : "+r"(d[j])::"memory");
    for (int j = 0; j < 48; ++j) out[tid * 48 + j] = __uint_as_float(d[j]);
    if (tid == 0) out[128 * 48] = (float)tb;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(128));
}

static float trunc_h(float a) {
  uint32_t u;
  memcpy(&u, &a, 4);
  u &= 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

int main() {
  float *dA, *dB, *dO;
  CK(cudaMalloc(&dA, 128 * 16 * 4));
  CK(cudaMalloc(&dB, 16 * 16 * 4));
  CK(cudaMalloc(&dO, 128 * 48 * 4 + 64));
  static float A[128 * 16], B[256], O[128 * 48 + 16];
  // ---- rounding probe: A = 1 + 3*2^-12 (0.75 tf32 ulp above 1), B = e_0 e_0^T
  for (int i = 0; i < 128 * 16; ++i) A[i] = 1.0f + 3.0f * ldexpf(1.0f, -12);
  for (int i = 0; i < 256; ++i) B[i] = 0.f;
  B[0] = 1.0f;
  CK(cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice));
  probe<<<1, 128>>>(dA, dB, dO, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(O, dO, sizeof O, cudaMemcpyDeviceToHost));
  printf("tmem base %g; row0:", (double)O[128 * 48]);
  for (int j = 0; j < 48; ++j) printf(" %g", (double)O[j]);
  printf("\n");
  printf("{\"probe\": \"tf32 reduction of A\", \"a\": %.10f, \"D1[0][0]\": %.10f, \"trunc\": %.10f, \"rna\": %.10f}\n",
         (double)A[0], (double)O[0], (double)trunc_h(A[0]), 1.0 + ldexp(1.0, -10));
  // ---- TMEM round trip (lo_mode 2): A_lo written by tcgen05.st, read back by tcgen05.ld
  {
    for (int i = 0; i < 128 * 16; ++i) A[i] = 1.0f + i * 1e-3f;
    CK(cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice));
    probe<<<1, 128>>>(dA, dB, dO, 2);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(O, dO, sizeof O, cudaMemcpyDeviceToHost));
    int ok = 0;
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 16; ++k) {
        const float a = A[r + 128 * k];
        const float lo = a - trunc_h(a);
        ok += O[r * 48 + k] == lo;
      }
    for (int w = 0; w < 4; ++w) {
      int okw = 0;
      for (int r = 32 * w; r < 32 * w + 32; ++r)
        for (int k = 0; k < 16; ++k) okw += O[r * 48 + k] == A[r + 128 * k] - trunc_h(A[r + 128 * k]);
      printf("warp %d: %d/512 match; row %d k0..3 got %g %g %g %g want %g %g %g %g\n", w, okw, 32 * w + 1,
             (double)O[(32 * w + 1) * 48 + 0], (double)O[(32 * w + 1) * 48 + 1], (double)O[(32 * w + 1) * 48 + 2],
             (double)O[(32 * w + 1) * 48 + 3], (double)(A[32 * w + 1] - trunc_h(A[32 * w + 1])),
             (double)(A[32 * w + 1 + 128] - trunc_h(A[32 * w + 1 + 128])),
             (double)(A[32 * w + 1 + 256] - trunc_h(A[32 * w + 1 + 256])),
             (double)(A[32 * w + 1 + 384] - trunc_h(A[32 * w + 1 + 384])));
    }
    printf("{\"probe\": \"tmem st/ld round trip\", \"matching\": %d, \"of\": %d, \"sample\": [%g, %g]}\n", ok, 128 * 16,
           (double)O[5 * 48 + 3], (double)(A[5 + 128 * 3] - trunc_h(A[5 + 128 * 3])));
  }
  // ---- random operands: check layouts and the split
  srand(7);
  for (int i = 0; i < 128 * 16; ++i) A[i] = (float)rand() / RAND_MAX;
  for (int i = 0; i < 256; ++i) B[i] = (float)rand() / RAND_MAX;
  CK(cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice));
  for (int lo_mode = 0; lo_mode < 2; ++lo_mode) {
    probe<<<1, 128>>>(dA, dB, dO, lo_mode);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(O, dO, sizeof O, cudaMemcpyDeviceToHost));
    double num = 0, den = 0, e_hi = 0, n_hi = 0, worst = 0;
    int bad_r = -1, bad_n = -1;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < 16; ++n) {
        double ex = 0, hi = 0;
        for (int k = 0; k < 16; ++k) {
          ex += (double)A[r + 128 * k] * (double)B[k * 16 + n];
          hi += (double)trunc_h(A[r + 128 * k]) * (double)trunc_h(B[k * 16 + n]);
        }
        const double got = (double)O[r * 48 + n] + (double)O[r * 48 + 16 + n] + (double)O[r * 48 + 32 + n];
        num += (got - ex) * (got - ex);
        den += ex * ex;
        e_hi += ((double)O[r * 48 + n] - hi) * ((double)O[r * 48 + n] - hi);
        n_hi += hi * hi;
        if (fabs(got - ex) > worst) {
          worst = fabs(got - ex);
          bad_r = r;
          bad_n = n;
        }
      }
    printf("{\"probe\": \"split product\", \"lo_mode\": \"%s\", \"rel_frob\": %.3e, \"hi_term_rel_frob_vs_trunc\": %.3e, "
           "\"worst_abs\": %.3e, \"at\": [%d, %d]}\n",
           lo_mode ? "rna" : "trunc", sqrt(num / den), sqrt(e_hi / n_hi), worst, bad_r, bad_n);
  }
  return 0;
}
