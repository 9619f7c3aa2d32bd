// Latency probe for the ALS warp code on B200: dependent DFMA, double
// shuffles, fp64 rsqrt / sqrt / division, and one full register Jacobi
// sweep (dp2_als_persist.cuh jacobi_reg) per R x R slice, single warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -Ipaper_2203_12798_b200/csrc -Iinclude -o tools/bin/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include "dp2_als_persist.cuh"

using namespace dp2;

__global__ void lat(double* out, long long* cyc, double x0, int n) {
  const int lane = threadIdx.x;
  double x = x0 + lane * 1e-3, y = 1.0000001;
  long long t0, t1;
  // dependent DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  cyc[0] = (t1 - t0);
  // dependent double shuffle
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64();
  cyc[1] = (t1 - t0);
  // 10 independent double shuffles (throughput)
  double v[10];
  for (int i = 0; i < 10; ++i) v[i] = x + i;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 10; ++q) v[q] = __shfl_sync(0xffffffffu, v[q], (lane + 3) & 31);
  }
  t1 = clock64();
  cyc[2] = (t1 - t0);
  for (int i = 0; i < 10; ++i) x += v[i];
  // dependent rsqrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.5);
  t1 = clock64();
  cyc[3] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.5);
  t1 = clock64();
  cyc[4] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.5);
  t1 = clock64();
  cyc[5] = (t1 - t0);
  // dependent DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64();
  cyc[6] = (t1 - t0);
  // float MUFU rsqrt
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = rsqrtf(f + 1.5f);
  t1 = clock64();
  cyc[7] = (t1 - t0);
  out[lane] = x + f;
}

template <int R>
__global__ void jac(const double* A, int* sweeps, long long* cyc) {
  double a[R], v[R];
  const int lane = threadIdx.x;
  for (int i = 0; i < R; ++i) {
    a[i] = lane < R ? A[i * R + lane] : 0.0;
    v[i] = lane < R ? (i == lane ? 1.0 : 0.0) : 0.0;
  }
  __syncwarp();
  const long long t0 = clock64();
  const int sw = jacobi_reg<R>(a, v);
  const long long t1 = clock64();
  if (lane == 0) {
    sweeps[0] = sw;
    cyc[0] = t1 - t0;
  }
}


// bisection copy of jacobi_reg: NOV drops the v shuffles/updates, FIXROT uses a
// fixed small rotation (no angle math), ROUNDS rounds of one sweep only
template <int R, bool NOV, bool FIXROT>
__global__ void jac_var(const double* A, long long* cyc, double* out) {
  constexpr int N = R + (R & 1);
  double a[R], v[R];
  const int lane = threadIdx.x;
  for (int i = 0; i < R; ++i) {
    a[i] = lane < R ? A[i * R + lane] : 0.0;
    v[i] = lane < R ? (i == lane ? 1.0 : 0.0) : 0.0;
  }
  __syncwarp();
  const long long t0 = clock64();
  for (int sw = 0; sw < 6; ++sw) {
#pragma unroll 1
    for (int r = 0; r < N - 1; ++r) {
      int pj = (2 * r - lane + 2 * (N - 1)) % (N - 1);
      pj = (lane == r) ? N - 1 : pj;
      pj = (lane == N - 1) ? r : pj;
      const int p = lane < N ? pj : lane;
      double pa[R], pv[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        pa[i] = __shfl_sync(0xffffffffu, a[i], p);
        if (!NOV) pv[i] = __shfl_sync(0xffffffffu, v[i], p);
      }
      double al0 = 0.0, be0 = 0.0, ga0 = 0.0, al1 = 0.0, be1 = 0.0, ga1 = 0.0;
#pragma unroll
      for (int i = 0; i < R; i += 2) {
        al0 = fma(a[i], a[i], al0);
        be0 = fma(pa[i], pa[i], be0);
        ga0 = fma(a[i], pa[i], ga0);
        if (i + 1 < R) {
          al1 = fma(a[i + 1], a[i + 1], al1);
          be1 = fma(pa[i + 1], pa[i + 1], be1);
          ga1 = fma(a[i + 1], pa[i + 1], ga1);
        }
      }
      const double al = al0 + al1, be = be0 + be1, ga = ga0 + ga1;
      const bool lower = lane < p;
      const double alpha = lower ? al : be, beta = lower ? be : al;
      double c = 1.0, s = 0.0;
      if (FIXROT) {
        c = 0.9999999 + 1e-30 * (alpha + beta + ga);
        s = 1e-4;
      } else if (p != lane && ga * ga > 1e-28 * (alpha * beta)) {
        const double d = beta - alpha, g2 = 2.0 * ga;
        const int hi = __double2hiint(alpha + beta);
        const int ex = min(max(((hi >> 20) & 0x7ff) - 1023, -1000), 1000);
        const double sc = __hiloint2double((1023 - ex) << 20, 0);
        const float df = (float)(d * sc), gf = (float)(g2 * sc);
        const float tf = (df >= 0.f ? gf : -gf) * rcp_approx(fabsf(df) + sqrt_approx(fmaf(df, df, gf * gf)));
        const double t = (double)tf;
        const double x = fma(t, t, 1.0);
        double y = (double)rsqrt_approx((float)x);
        y = y * fma(-0.5 * x, y * y, 1.5);
        y = y * fma(-0.5 * x, y * y, 1.5);
        c = y;
        s = c * t;
      }
      const double so = lower ? -s : s;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        a[i] = fma(c, a[i], so * pa[i]);
        if (!NOV) v[i] = fma(c, v[i], so * pv[i]);
      }
    }
  }
  const long long t1 = clock64();
  double acc = 0.0;
  for (int i = 0; i < R; ++i) acc += a[i] + v[i];
  out[lane] = acc;
  if (lane == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  int* sw;
  cudaMalloc(&out, 1024);
  cudaMallocManaged(&cyc, 64);
  cudaMallocManaged(&sw, 16);
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(out, cyc, 0.5, n);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA dep", "SHFL.f64 dep", "10x SHFL.f64 indep (per iter)", "rsqrt(f64) dep",
                         "sqrt(f64) dep", "1/x (f64) dep", "DADD dep", "rsqrtf dep"};
  for (int i = 0; i < 8; ++i) printf("%-32s %.1f cyc\n", names[i], (double)cyc[i] / n);
  constexpr int R = 10;
  double h[R * R];
  srand(1);
  for (int i = 0; i < R * R; ++i) h[i] = (double)rand() / RAND_MAX - 0.5;
  double* dA;
  cudaMalloc(&dA, sizeof(h));
  cudaMemcpy(dA, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) jac<R><<<1, 32>>>(dA, sw, cyc);
  cudaDeviceSynchronize();
  printf("jacobi R=%d cold: %d sweeps, %lld cyc, %.0f cyc/round (%s)\n", R, sw[0], cyc[0],
         (double)cyc[0] / (sw[0] * (R - 1)), cudaGetErrorString(cudaGetLastError()));
  const char* vn[] = {"full", "no v", "fixed rot", "no v + fixed rot"};
  for (int vi = 0; vi < 4; ++vi) {
    for (int rep = 0; rep < 2; ++rep) {
      if (vi == 0) jac_var<R, false, false><<<1, 32>>>(dA, cyc, out);
      if (vi == 1) jac_var<R, true, false><<<1, 32>>>(dA, cyc, out);
      if (vi == 2) jac_var<R, false, true><<<1, 32>>>(dA, cyc, out);
      if (vi == 3) jac_var<R, true, true><<<1, 32>>>(dA, cyc, out);
    }
    cudaDeviceSynchronize();
    printf("variant %-18s %.0f cyc/round\n", vn[vi], (double)cyc[0] / (6 * (R - 1)));
  }
  return 0;
}
