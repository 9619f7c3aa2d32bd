// DMMA.8x8x4 issue rate of ONE warp per SM sub-partition (the sketch64 A-warp
// shape) against the number of independent accumulator chains, operands in
// registers (no shared-memory loads): does a single warp reach the pipe rate
// (1 DMMA / 16 clk / sub-partition at the 36.9 TF/s peak)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/dmma_warp_probe tools/dmma_warp_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_k(double* out, int n, long long* cyc) {
  double c[CH][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = 0.0;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
void run(int sms, int wps, double* d, long long* dc) {
  const int n = 4096;
  dmma_k<CH><<<sms, 32 * wps>>>(d, 64, dc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_k<CH><<<sms, 32 * wps>>>(d, n, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  const double flops = 512.0 * CH * n * (double)sms * wps;
  printf("warps/SM %2d chains %2d: %6.2f TF/s, %.1f clk per DMMA per warp\n", wps, CH, flops / ms / 1e9,
         (double)cyc / (n * CH));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  long long* dc;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&dc, 8);
  for (int wps : {4, 8}) {
    run<1>(sms, wps, d, dc);
    run<2>(sms, wps, d, dc);
    run<4>(sms, wps, d, dc);
    run<6>(sms, wps, d, dc);
    run<8>(sms, wps, d, dc);
    run<12>(sms, wps, d, dc);
  }
  return 0;
}
