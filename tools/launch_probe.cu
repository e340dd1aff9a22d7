// Fixed cost of the launch pattern used by the dynamic kernel: a 148-CTA, 288-thread kernel with
// ~200 KB of dynamic shared memory, alone and behind a small prep kernel (with / without PDL, with
// / without the prep kernel asking for the max-shared carveout). Event-timed, back to back and
// isolated. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_big(int* p, int pdl) {
  extern __shared__ unsigned char sm[];
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    sm[0] = 1;
    p[blockIdx.x] = sm[0] + 1;
  }
}
__global__ void k_prep(int* p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  p[1024 + blockIdx.x * blockDim.x + threadIdx.x] = 1;
}

static float run(int mode, int reps, bool iso, int* d, size_t smem) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float tot = 0;
  int outer = iso ? reps : 1, inner = iso ? 1 : reps;
  for (int o = 0; o < outer; ++o) {
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < inner; ++i) {
      if (mode >= 1) k_prep<<<148, 256>>>(d);
      if (mode == 3) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(288);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_big, d, 1);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return -1.f; }
      } else {
        k_big<<<148, 288, smem>>>(d, 0);
      }
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    tot += ms;
  }
  return tot * 1000.f / reps;
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int* d;
  cudaMalloc(&d, 1 << 24);
  const size_t smem = (argc > 1 ? atoi(argv[1]) : 200) * 1024;  // dynamic smem of the big kernel, KB
  printf("big kernel: 148 CTAs x 288 threads, %zu KB dynamic shared memory\n", smem / 1024);
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[] = {"big alone", "prep + big", "prep(carveout 100) + big", "prep + big (PDL)",
                         "prep(carveout 100) + big (PDL)"};
  for (int pass = 0; pass < 2; ++pass) {
    for (int mode = 0; mode < 5; ++mode) {
      const bool c100 = mode == 2 || mode == 4;
      cudaFuncSetAttribute(k_prep, cudaFuncAttributePreferredSharedMemoryCarveout, c100 ? 100 : -1);
      const int m = mode == 4 ? 3 : mode == 2 ? 1 : mode;
      run(m, 50, false, d, smem);
      printf("%-32s back-to-back %6.2f us/iter   isolated %6.2f us/iter\n", names[mode], run(m, 1000, false, d, smem),
             run(m, 200, true, d, smem));
    }
    cudaFuncSetAttribute(k_prep, cudaFuncAttributePreferredSharedMemoryCarveout, -1);
    for (int mode = 0; mode < 2; ++mode) {
      printf("%-32s back-to-back %6.2f us/iter   isolated %6.2f us/iter  (no dyn smem)\n", names[mode],
             run(mode, 1000, false, d, 0), run(mode, 200, true, d, 0));
    }
    printf("--\n");
  }
  return 0;
}
