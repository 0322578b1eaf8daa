// Dependent-chain latency of FP64 ops on sm_100a (cycles per op, one thread).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, int n) {
  double x = x0, y = x0 * 0.5;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = y + 1e-9;
  t1 = clock64(); cyc[1] = t1 - t0;
  // division chain
  double z = x0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = 1.0 / (z + 1.0);
  t1 = clock64(); cyc[2] = t1 - t0;
  // sqrt chain
  double w = x0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) w = sqrt(w + 1.0);
  t1 = clock64(); cyc[3] = t1 - t0;
  // rsqrt chain
  double r = x0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) r = rsqrt(r + 1.0);
  t1 = clock64(); cyc[4] = t1 - t0;
  // FFMA chain (fp32)
  float f = (float)x0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, 0.999999f, 1e-9f);
  t1 = clock64(); cyc[5] = t1 - t0;
  // shared-memory dependent chain
  __shared__ double sm[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = 0.0;
  __syncthreads();
  int idx = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = (int)sm[idx & 255] + (i & 1);
  t1 = clock64(); cyc[6] = t1 - t0;
  // __syncthreads cost
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); cyc[7] = t1 - t0;
  // DMMA m8n8k4 f64 dependent chain (same accumulator)
  double c0 = x0, c1 = x0;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(0.5), "d"(1e-9));
  t1 = clock64(); cyc[8] = t1 - t0;
  // double shuffle chain
  double sh = x0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) sh = __shfl_sync(0xffffffffu, sh, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64(); cyc[9] = t1 - t0;
  out[0] = x + y + z + w + r + f + idx + c0 + c1 + sh;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 10);
  const int n = 1000;
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(out, cyc, 0.5, n);
    lat<<<1, threads>>>(out, cyc, 0.5, n);
    cudaDeviceSynchronize();
    long long h[10];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[10] = {"DFMA", "DADD", "1/x (double div)", "sqrt(double)", "rsqrt(double)",
                             "FFMA", "LDS chain", "__syncthreads", "DMMA m8n8k4 chain",
                             "SHFL double + DADD"};
    printf("threads=%d\n", threads);
    for (int i = 0; i < 10; ++i) printf("  %-18s %7.1f cycles/op\n", names[i], (double)h[i] / n);
  }
  // empty kernel launch rate
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 1000; ++i) lat<<<1, 32>>>(out, cyc, 0.5, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("back-to-back 1-CTA launches: %.2f us each\n", ms);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
