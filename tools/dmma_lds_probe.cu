// DMMA.8x8x4 rate when the operands come from shared memory, in the shapes of
// the sketch64 pass (csrc/dp2_sketch64.cu), without any barrier hand-offs:
//   A shape  per k-step: 1 LDS.64 (X fragment) + 3 LDS.64 (B image) + 3 DMMA, 6 chains
//   A128     per 2 k-steps: 1 LDS.128 + 3 LDS.128 + 6 DMMA (paired k-steps)
//   B shape  per k2: 3 LDS.64 (Y) + 4 LDS.64 (X^T) + 12 DMMA, 12 chains
//   B128     per 2 k2: 3 LDS.128 + 4 LDS.128 + 24 DMMA
//   mix      4 A warps + 16 B warps per SM (the pass's warp layout), equal DMMA
//            counts per sub-partition
// Answers: is the pass's 75% DMMA-pipe activity a property of LDS-fed DMMA
// streams (then wider loads may help) or of its hand-off structure?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/dmma_lds_probe tools/dmma_lds_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int XL = 516;  // padded row stride of the X stage (doubles)

// mode 0: A shape LDS.64, 1: A shape LDS.128, 2: B shape LDS.64, 3: B shape LDS.128,
// 4: mix (warps 0-3 A, 4-19 B), 5: mix with LDS.128, 6: registers only (A count)
template <int MODE>
__global__ void __launch_bounds__(704, 1) probe_k(double* out, int tiles) {
  extern __shared__ __align__(16) double sm[];
  double* xs = sm;                   // 8 x XL
  double* img = sm + 8 * XL;         // 32 k-steps x 3 x 32 per A warp x 4
  double* yf = img + 4 * 32 * 96;   // 2 x 3 x 32
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * XL + 4 * 32 * 96 + 192; i += blockDim.x) sm[i] = 1e-3 * (i & 7);
  __syncthreads();
  const bool is_a = MODE == 0 || MODE == 1 || MODE == 6 || ((MODE == 4 || MODE == 5) && warp < 4);
  const bool wide = MODE == 1 || MODE == 3 || MODE == 5;
  double acc = 0.0;
  if (is_a) {
    const int a = warp & 3, r = lane >> 2, q = lane & 3;
    const double* im = img + (size_t)a * 32 * 96 + lane;
    for (int t = 0; t < tiles; ++t) {
      asm volatile("" ::: "memory");  // the tile's operands are re-read, as in the pass
      double c[2][3][2] = {};
      if (MODE == 6) {
        double x = 1.0 + lane, o = 1.0 - lane;
#pragma unroll 4
        for (int k = 0; k < 32; k += 2)
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int j = 0; j < 3; ++j) dmma(c[u][j][0], c[u][j][1], x, o);
      } else if (!wide) {
        const double* xr = xs + (size_t)r * XL + a * 128 + q;
#pragma unroll 4
        for (int k = 0; k < 32; k += 2)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double x = xr[4 * (k + u)];
#pragma unroll
            for (int j = 0; j < 3; ++j) dmma(c[u][j][0], c[u][j][1], x, im[((k + u) * 3 + j) * 32]);
          }
      } else {
        // paired k-steps: lane (r, q) holds columns 8 m + 2 q, + 1; the image interleaves the pair
        const double2* xr = reinterpret_cast<const double2*>(xs + (size_t)r * XL + a * 128) + q;
        const double2* im2 = reinterpret_cast<const double2*>(img + (size_t)a * 32 * 96) + lane;
#pragma unroll 4
        for (int k = 0; k < 16; ++k) {
          const double2 x = xr[4 * k];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double2 o = im2[(k * 3 + j) * 32];
            dmma(c[0][j][0], c[0][j][1], x.x, o.x);
            dmma(c[1][j][0], c[1][j][1], x.y, o.y);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int j = 0; j < 3; ++j) acc += c[u][j][0] + c[u][j][1];
    }
  } else {
    const int bw = (MODE == 4 || MODE == 5) ? warp - 4 : warp % 16;
    double z[4][3][2] = {};
    for (int t = 0; t < tiles; ++t) {
      asm volatile("" ::: "memory");
      if (!wide) {
        const double* yv_ = yf + lane;
        const double* xb = xs + (size_t)(lane & 3) * XL + 32 * bw + (lane >> 2);
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) {
          double yv[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) yv[j] = yv_[(k2 * 3 + j) * 32];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double xv = xb[(size_t)4 * k2 * XL + 8 * i];
#pragma unroll
            for (int j = 0; j < 3; ++j) dmma(z[i][j][0], z[i][j][1], xv, yv[j]);
          }
        }
      } else {
        const double2* yv_ = reinterpret_cast<const double2*>(yf) + lane;
        const double2* xb = reinterpret_cast<const double2*>(xs + (size_t)(lane & 3) * XL + 32 * bw) + (lane >> 2);
        double2 yv[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) yv[j] = yv_[j * 32];
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const double2 xv = xb[(size_t)2 * k2 * XL + 8 * i];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              dmma(z[2 * i][j][0], z[2 * i][j][1], xv.x, k2 ? yv[j].y : yv[j].x);
              dmma(z[2 * i + 1][j][0], z[2 * i + 1][j][1], xv.y, k2 ? yv[j].y : yv[j].x);
            }
          }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) acc += z[i][j][0] + z[i][j][1];
  }
  if (acc == 12345.678) out[threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, int sms, int warps, double* d) {
  const int tiles = 2000;
  const size_t smem = (8 * XL + 4 * 32 * 96 + 192 + 64) * sizeof(double);
  cudaFuncSetAttribute(probe_k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_k<MODE><<<sms, 32 * warps, smem>>>(d, 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_k<MODE><<<sms, 32 * warps, smem>>>(d, tiles);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // DMMAs per tile: A warp 96 (32 k-steps x 3), B warp 24
  double dm;
  if (MODE == 0 || MODE == 1 || MODE == 6) dm = 96.0 * warps;
  else if (MODE == 2 || MODE == 3) dm = 24.0 * warps;
  else dm = 96.0 * 4 + 24.0 * (warps - 4);
  const double flops = 512.0 * dm * tiles * sms;
  printf("%-28s warps/SM %2d: %6.2f TF/s  (%s)\n", name, warps, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 1 << 20);
  for (int w : {4, 8}) run<6>("registers, 6 chains", sms, w, d);
  for (int w : {4, 8, 16}) run<0>("A shape LDS.64", sms, w, d);
  for (int w : {4, 8, 16}) run<1>("A shape LDS.128 (paired k)", sms, w, d);
  for (int w : {4, 16}) run<2>("B shape LDS.64", sms, w, d);
  for (int w : {4, 16}) run<3>("B shape LDS.128", sms, w, d);
  run<4>("mix 4 A + 16 B, LDS.64", sms, 20, d);
  run<5>("mix 4 A + 16 B, LDS.128", sms, 20, d);
  return 0;
}
