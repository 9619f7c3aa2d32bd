// Latency probe: one warp inverting a 10x10 SPD matrix (register Gauss-Jordan)
// and the building blocks (fp64 reciprocal, double shuffle chains), clock64.
#include <cstdio>
#include <cuda_runtime.h>
template <int RM>
__device__ bool gj(const double* A, int R, double* out) {
  const int lane = threadIdx.x & 31;
  double col[RM];
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    double v = 0.0;
    if (i < R) v = lane < R ? A[i * R + lane] : (lane < 2 * R && i == lane - R ? 1.0 : 0.0);
    col[i] = v;
  }
  bool okay = true;
#pragma unroll
  for (int k = 0; k < RM; ++k) {
    if (k < R) {
      const double piv = __shfl_sync(0xffffffffu, col[k], k);
      if (!(piv > 0.0)) okay = false;
      const double rk = col[k] * (1.0 / piv);
#pragma unroll
      for (int i = 0; i < RM; ++i)
        if (i < R) {
          const double f = __shfl_sync(0xffffffffu, col[i], k);
          col[i] = (i == k) ? rk : fma(-f, rk, col[i]);
        }
    }
  }
#pragma unroll
  for (int i = 0; i < RM; ++i)
    if (i < R && lane >= R && lane < 2 * R) out[i * R + lane - R] = col[i];
  return okay;
}
// compile-time R: no predicates
template <int R>
__device__ bool gjc(const double* A, double* out) {
  const int lane = threadIdx.x & 31;
  double col[R];
#pragma unroll
  for (int i = 0; i < R; ++i) col[i] = lane < R ? A[i * R + lane] : (lane < 2 * R && i == lane - R ? 1.0 : 0.0);
  bool okay = true;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double piv = __shfl_sync(0xffffffffu, col[k], k);
    okay &= piv > 0.0;
    const double rk = col[k] * (1.0 / piv);
    double f[R];
#pragma unroll
    for (int i = 0; i < R; ++i) f[i] = __shfl_sync(0xffffffffu, col[i], k);
#pragma unroll
    for (int i = 0; i < R; ++i) col[i] = (i == k) ? rk : fma(-f[i], rk, col[i]);
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (lane >= R && lane < 2 * R) out[i * R + lane - R] = col[i];
  return okay;
}
__global__ void probe(const double* Ag, double* out, long long* t, int R) {
  __shared__ double A[1024], O[1024];
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) A[i] = Ag[i];
  __syncthreads();
  long long t0 = clock64();
  bool ok = gj<16>(A, R, O);
  __syncwarp();
  long long t1 = clock64();
  bool ok2 = gjc<10>(A, O + 128);
  __syncwarp();
  long long t1b = clock64();
  // reciprocal chain
  double x = A[0] + 1.0;
  for (int i = 0; i < 10; ++i) x = 1.0 / (x + 1.0);
  long long t2 = clock64();
  // shuffle chain
  double y = A[1];
  for (int i = 0; i < 10; ++i) y = __shfl_sync(0xffffffffu, y, (threadIdx.x + 1) & 31) + 1.0;
  long long t3 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t1b - t1; t[2] = t3 - t2; out[0] = x + y + O[0] + ok + ok2 + O[128]; }
}
int main() {
  const int R = 10;
  double h[100];
  for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) h[i * R + j] = (i == j ? 20.0 : 1.0 / (1 + i + j));
  double *dA, *dO; long long* dt;
  cudaMalloc(&dA, 800); cudaMalloc(&dO, 800); cudaMalloc(&dt, 64);
  cudaMemcpy(dA, h, 800, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) probe<<<1, 32>>>(dA, dO, dt, R);
  cudaDeviceSynchronize();
  long long t[3]; cudaMemcpy(t, dt, 24, cudaMemcpyDeviceToHost);
  printf("gj<16> R=10 (runtime R): %lld cycles; gjc<10> (compile-time R): %lld; 10 dependent double shuffles: %lld\n", t[0], t[1], t[2]);
  return 0;
}
