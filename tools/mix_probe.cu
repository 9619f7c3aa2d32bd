// Does the FP64 tensor path (DMMA, tensor pipe) co-issue with DFMA (fp64
// pipe)?  Each warp runs CH DMMA chains and F DFMA chains (x4 per iteration);
// reports total fp64 TFLOP/s on all SMs, plus the dependent-DMMA latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mix_probe tools/mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, int F>
__global__ void mix(double* out, int n) {
  double c[CH > 0 ? CH : 1][2];
  double f[F > 0 ? F : 1];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int j = 0; j < (CH > 0 ? CH : 1); ++j) c[j][0] = c[j][1] = 0.0;
#pragma unroll
  for (int j = 0; j < (F > 0 ? F : 1); ++j) f[j] = j;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < F; ++j) f[j] = fma(f[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < (CH > 0 ? CH : 1); ++j) s += c[j][0] + c[j][1];
#pragma unroll
  for (int j = 0; j < (F > 0 ? F : 1); ++j) s += f[j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void lat(long long* out, int n) {
  double c0 = 0, c1 = 0, a = threadIdx.x, b = 1;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
  if (c0 == 1.2345) out[1] = (long long)c1;
}

template <int CH, int F>
void run(int sms, double* d, int wps) {
  const int n = 2048, blocks = sms * 2, threads = wps * 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mix<CH, F><<<blocks, threads>>>(d, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double fd = warps * n * 512.0 * CH, ff = warps * n * 32.0 * 2 * 4 * F;
  printf("{\"dmma_chains\": %d, \"dfma_chains_x4\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f, \"dmma_tf\": %.2f, "
         "\"dfma_tf\": %.2f}\n",
         CH, F, wps, (fd + ff) / best / 1e9, fd / best / 1e9, ff / best / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 1 << 20);
  long long* l;
  cudaMalloc(&l, 16);
  lat<<<1, 32>>>(l, 4096);
  long long h[2];
  cudaMemcpy(h, l, 16, cudaMemcpyDeviceToHost);
  printf("{\"dmma_dependent_latency_cycles\": %lld}\n", h[0]);
  for (int w : {4, 8}) {  // 1 / 2 warps per SM sub-partition: can one warp saturate the DMMA pipe?
    run<3, 0>(sms, d, w);
    run<6, 0>(sms, d, w);
    run<12, 0>(sms, d, w);
  }
  for (int w : {8, 16}) {
    run<8, 0>(sms, d, w);
    run<0, 8>(sms, d, w);
    run<8, 2>(sms, d, w);
    run<8, 4>(sms, d, w);
    run<8, 8>(sms, d, w);
    run<4, 8>(sms, d, w);
  }
  return 0;
}
