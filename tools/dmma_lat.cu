// DMMA (m8n8k4 fp64) throughput vs. warps per SM and independent accumulator chains per warp —
// how much parallelism the consumer warps of tsm2r_stream_tma need to keep the FP64 tensor path
// busy. One CTA per SM (148 CTAs) of W warps, each warp CH independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat tools/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_chains(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[CH][2];
#pragma unroll
  for (int j = 0; j < CH; ++j) { d[j][0] = j; d[j][1] = -j; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += d[j][0] + d[j][1];
  if (s == 1.2345) *out = s;
}

template <int CH>
void run(int sms, int warps, double* buf) {
  const int iters = 16384 / CH * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_chains<CH><<<sms, warps * 32>>>(buf, 16);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) dmma_chains<CH><<<sms, warps * 32>>>(buf, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = 5.0 * sms * warps * (double)iters * CH;
  const double fl = dmmas * 512.0;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("{\"warps_per_sm\": %d, \"chains\": %d, \"TFLOPs\": %.2f, \"sm_cycles_per_dmma_per_smsp\": %.2f}\n", warps, CH,
         fl / ms / 1e9, cyc / (dmmas / sms / 4));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  cudaMalloc(&buf, 64);
  for (int w : {4, 8, 16, 32}) {
    run<4>(sms, w, buf);
    run<8>(sms, w, buf);
    run<16>(sms, w, buf);
    run<32>(sms, w, buf);
  }
  return 0;
}
