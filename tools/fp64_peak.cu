// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64)
// vs SIMT DFMA issue throughput. Used once to fix the FP64 roofline
// denominator (MEASURED_PEAKS.json carries no FP64 figure).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 20000;
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int blocks_per_sm = 1; blocks_per_sm <= 2; ++blocks_per_sm) {
      int grid = sms * blocks_per_sm;
      dmma_loop<<<grid, warps * 32>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<<<grid, warps * 32>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * warps * grid;
      printf("DMMA warps/cta=%2d cta/sm=%d : %.2f TFLOP/s (%.3f ms)\n", warps, blocks_per_sm,
             flops / ms / 1e9, ms);
      dfma_loop<<<grid, warps * 32>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<<<grid, warps * 32>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * 32 * (double)iters * warps * grid;
      printf("DFMA warps/cta=%2d cta/sm=%d : %.2f TFLOP/s (%.3f ms)\n", warps, blocks_per_sm,
             flops / ms / 1e9, ms);
    }
  }
  printf("sms=%d clock_khz=%d err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
