// Shared device helpers for the DPar2 B200 kernels (sm_100a).
//
// Everything numeric that is not a streaming pass lives here: warp/block
// reductions, the fp64 m8n8k4 tensor-core MMA wrapper, a block-cooperative
// cyclic Jacobi eigensolver for small symmetric matrices (the reference uses
// LAPACK gesdd on the same tiny matrices: P/linalg.py:87,143) and a warp
// one-sided Jacobi polar factor (P/solver.py:59 only ever consumes Z_k P_k^T).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/dpar2_b200.h"

#define DP2_DEV __device__ __forceinline__

namespace dp2 {

constexpr double kEps = 1.1102230246251565e-16;  // 2^-53

// ---------------------------------------------------------------- status
// Device-side status block (int64 x 8), read by the host after a sync.
//   [0] lowest slice index holding a non-finite value (INT64_MAX = none)
//   [1] reserved (fatal non-convergence)
//   [2] lowest slice index whose sketch had numerical rank < R
//   [3] lowest slice index with a failed polar factor
//   [4] count of Jacobi solves that hit the sweep cap (informational: the
//       result is still at the rounding floor)
enum { ST_NONFINITE = 0, ST_NOCONV = 1, ST_RANKDEF = 2, ST_POLAR = 3, ST_SWEEPCAP = 4 };

DP2_DEV void status_min(int64_t* st, int slot, int64_t v) {
  atomicMin(reinterpret_cast<unsigned long long*>(st + slot), (unsigned long long)v);
}

// ---------------------------------------------------------------- reductions
DP2_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum: warp tree, then warp 0 sums the warp results in
// warp order.  ``red`` must hold >= 32 doubles.  All threads get the result.
DP2_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- fp64 MMA
// D(8x8) += A(8x4, row) * B(4x8, col); one double of A and B per lane,
// two of C/D.  Fragment layout (PTX ISA, mma.m8n8k4.f64):
//   a0 = A[lane>>2][lane&3]   b0 = B[lane&3][lane>>2]
//   c0,c1 = C[lane>>2][2*(lane&3) + {0,1}]
DP2_DEV void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- cp.async
DP2_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
DP2_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
DP2_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------- pairing
// Round-robin ("chess tournament") ordering for parallel Jacobi: in round r
// of n_even-1 rounds, pair i couples positions i and n_even-1-i; position 0
// is fixed, the others rotate.  Index n (odd n padding) is a dummy.
DP2_DEV void rr_pair(int n_even, int r, int i, int& p, int& q) {
  auto at = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + r) % (n_even - 1)); };
  p = at(i);
  q = at(n_even - 1 - i);
  if (p > q) { int t = p; p = q; q = t; }
}

// ---------------------------------------------------------------- rotations
// Jacobi rotation (c, s) annihilating g for the 2x2 symmetric problem with
// diagonal difference d (= b - a): t = sgn(d) 2g / (|d| + sqrt(d^2 + 4g^2)).
// The angle is estimated in fp32 on the scaled pair (any angle that shrinks g
// keeps the sweep converging); (c, s) are then made orthonormal to fp64
// precision: c = (1 + t^2)^(-1/2) by two Newton steps, s = c t.  This keeps the
// accumulated rotations exactly orthogonal while avoiding the fp64 div/sqrt
// sequences on the latency-critical path.
DP2_DEV void rot_params(double d, double g, double& c, double& s) {
  const float df = (float)d, gf = (float)(2.0 * g);
  const float m = fmaxf(fabsf(df), fabsf(gf));
  double t;
  if (m > 1e-30f && m < 1e30f) {
    const float inv = __frcp_rn(m);
    const float dn = df * inv, gn = gf * inv;
    const float tf = (dn >= 0.0f ? gn : -gn) * __frcp_rn(fabsf(dn) + sqrtf(fmaf(dn, dn, gn * gn)));
    t = (double)tf;
  } else {  // out of fp32 range: exact fp64 formula
    const double ze = d / (2.0 * g);
    t = (ze >= 0.0 ? 1.0 : -1.0) / (fabs(ze) + sqrt(ze * ze + 1.0));
  }
  const double x = fma(t, t, 1.0);
  double r = (double)rsqrtf((float)x);
  r = r * fma(-0.5 * x, r * r, 1.5);
  r = r * fma(-0.5 * x, r * r, 1.5);
  c = r;
  s = r * t;
}

// ---------------------------------------------------------------- Jacobi eig
// Block-cooperative cyclic Jacobi for a symmetric n x n matrix A (row-major,
// leading dim lda, shared memory).  On return diag(A) holds the eigenvalues and
// V (n x n, ldv) the eigenvectors as columns.  ``cs`` needs 3*(n/2+1) doubles
// and ``flag`` one int of shared scratch.  Rotations are skipped when
// |a_pq| <= n eps sqrt(|a_pp a_qq|) (relative criterion: PSD inputs keep
// high relative accuracy in their small eigenvalues; n eps is the rounding
// floor).  Returns sweeps used (max_sweeps+1 when the cap was hit).
DP2_DEV int jacobi_eig_block(double* A, int lda, double* V, int ldv, int n, double* cs, int* flag,
                             int max_sweeps = 40, bool init_v = true) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (init_v)  // else V holds a starting basis (the rotations accumulate onto it)
    for (int i = tid; i < n * n; i += nt) V[(i / n) * ldv + (i % n)] = (i / n == i % n) ? 1.0 : 0.0;
  if (n < 2) { __syncthreads(); return 0; }
  const int ne = n + (n & 1), np = ne / 2;
  const double tol = n * kEps;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < ne - 1; ++r) {
      for (int i = tid; i < np; i += nt) {
        int p, q;
        rr_pair(ne, r, i, p, q);
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = A[p * lda + q], app = A[p * lda + p], aqq = A[q * lda + q];
          if (apq != 0.0 && apq * apq > (tol * tol) * fabs(app * aqq)) {
            rot_params(aqq - app, apq, c, s);
            *flag = 1;
          }
        }
        cs[3 * i] = c;
        cs[3 * i + 1] = s;
        cs[3 * i + 2] = (double)(p * 1024 + q);
      }
      __syncthreads();
      // columns: A <- A J, V <- V J (a pair per warp, lanes over the rows)
      const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
      for (int pr = warp; pr < np; pr += nw) {
        const double s = cs[3 * pr + 1];
        if (s == 0.0) continue;
        const double c = cs[3 * pr];
        const int pq = (int)cs[3 * pr + 2], p = pq >> 10, q = pq & 1023;
        for (int i = lane; i < n; i += 32) {
          double a = A[i * lda + p], b = A[i * lda + q];
          A[i * lda + p] = c * a - s * b;
          A[i * lda + q] = s * a + c * b;
          a = V[i * ldv + p];
          b = V[i * ldv + q];
          V[i * ldv + p] = c * a - s * b;
          V[i * ldv + q] = s * a + c * b;
        }
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int pr = warp; pr < np; pr += nw) {
        const double s = cs[3 * pr + 1];
        if (s == 0.0) continue;
        const double c = cs[3 * pr];
        const int pq = (int)cs[3 * pr + 2], p = pq >> 10, q = pq & 1023;
        for (int j = lane; j < n; j += 32) {
          const double a = A[p * lda + j], b = A[q * lda + j];
          A[p * lda + j] = c * a - s * b;
          A[q * lda + j] = s * a + c * b;
        }
      }
      __syncthreads();
    }
    const int any = *flag;
    __syncthreads();
    if (!any) break;
  }
  return sweep + 1;
}

// Single-warp version of jacobi_eig_block (same ordering, rotations and
// thresholds; __syncwarp instead of __syncthreads).  For the R x R pinvs and
// other n <= 64 problems where a whole block would mostly idle.
DP2_DEV int jacobi_eig_warp(double* A, int lda, double* V, int ldv, int n, double* cs, int max_sweeps = 40,
                            bool init_v = true) {
  const int lane = threadIdx.x & 31;
  if (init_v)
    for (int i = lane; i < n * n; i += 32) V[(i / n) * ldv + (i % n)] = (i / n == i % n) ? 1.0 : 0.0;
  __syncwarp();
  if (n < 2) return 0;
  const int ne = n + (n & 1), np = ne / 2;
  const double tol = n * kEps;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < ne - 1; ++r) {
      for (int i = lane; i < np; i += 32) {
        int p, q;
        rr_pair(ne, r, i, p, q);
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = A[p * lda + q], app = A[p * lda + p], aqq = A[q * lda + q];
          if (apq != 0.0 && apq * apq > (tol * tol) * fabs(app * aqq)) {
            rot_params(aqq - app, apq, c, s);
            rotated = 1;
          }
        }
        cs[3 * i] = c;
        cs[3 * i + 1] = s;
        cs[3 * i + 2] = (double)(p * 1024 + q);
      }
      __syncwarp();
      for (int it = lane; it < n * np; it += 32) {
        const int i = it / np, pr = it % np;
        const double s = cs[3 * pr + 1];
        if (s == 0.0) continue;
        const double c = cs[3 * pr];
        const int pq = (int)cs[3 * pr + 2], p = pq >> 10, q = pq & 1023;
        double a = A[i * lda + p], b = A[i * lda + q];
        A[i * lda + p] = c * a - s * b;
        A[i * lda + q] = s * a + c * b;
        a = V[i * ldv + p];
        b = V[i * ldv + q];
        V[i * ldv + p] = c * a - s * b;
        V[i * ldv + q] = s * a + c * b;
      }
      __syncwarp();
      for (int it = lane; it < n * np; it += 32) {
        const int pr = it / n, j = it % n;
        const double s = cs[3 * pr + 1];
        if (s == 0.0) continue;
        const double c = cs[3 * pr];
        const int pq = (int)cs[3 * pr + 2], p = pq >> 10, q = pq & 1023;
        const double a = A[p * lda + j], b = A[q * lda + j];
        A[p * lda + j] = c * a - s * b;
        A[q * lda + j] = s * a + c * b;
      }
      __syncwarp();
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
  return sweep + 1;
}

// Sort eigenpairs by descending eigenvalue (stable on index): writes the
// permutation into ``perm`` (n ints, shared).  Single-threaded; n is tiny.
DP2_DEV void sort_desc_perm(const double* A, int lda, int n, int* perm) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = 1; i < n; ++i) {
      int v = perm[i];
      double key = A[v * lda + v];
      int j = i - 1;
      while (j >= 0 && A[perm[j] * lda + perm[j]] < key) { perm[j + 1] = perm[j]; --j; }
      perm[j + 1] = v;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- polar
// Warp one-sided (Hestenes) Jacobi on the columns of T (n x n, column-major,
// leading dim ldt, shared).  On return T's columns are mutually orthogonal
// (T_final = T0 Vr) and Vr (column-major, ldv) holds the accumulated right
// rotations, so T0 = Z Sigma Vr^T with Z = normalised columns of T_final.
// ``Vr`` may be pre-loaded with a warm-start orthogonal matrix when T0 was
// already multiplied by it.  Lane i owns pair i (n <= 64).
DP2_DEV int jacobi_onesided_warp(double* T, int ldt, double* Vr, int ldv, int n, int max_sweeps = 60) {
  const int lane = threadIdx.x & 31;
  if (n < 2) return 0;
  const int ne = n + (n & 1), np = ne / 2;
  const double tol = n * kEps;  // rounding floor of the length-n dot products
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < ne - 1; ++r) {
      for (int i = lane; i < np; i += 32) {
        int p, q;
        rr_pair(ne, r, i, p, q);
        if (q >= n) continue;
        double* tp = T + p * ldt;
        double* tq = T + q * ldt;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int k = 0; k < n; ++k) {
          const double x = tp[k], y = tq[k];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        if (ga != 0.0 && ga * ga > (tol * tol) * (al * be)) {
          double c, s;
          rot_params(be - al, ga, c, s);
          for (int k = 0; k < n; ++k) {
            const double x = tp[k], y = tq[k];
            tp[k] = c * x - s * y;
            tq[k] = s * x + c * y;
          }
          double* vp = Vr + p * ldv;
          double* vq = Vr + q * ldv;
          for (int k = 0; k < n; ++k) {
            const double x = vp[k], y = vq[k];
            vp[k] = c * x - s * y;
            vq[k] = s * x + c * y;
          }
          rotated = 1;
        }
      }
      __syncwarp();
    }
    rotated = __any_sync(0xffffffffu, rotated);
    if (!rotated) break;
  }
  return sweep + 1;
}

// ---------------------------------------------------------------- register Jacobi
DP2_DEV float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
DP2_DEV float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
DP2_DEV float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One-sided Jacobi (Hestenes) on an R x R matrix held column-wise in
// registers: lane j < R holds column j (a) and, with WITHV, column j of the
// accumulated right rotations V (v); a zero column pads odd R.  For a
// symmetric PSD input the converged columns are lambda_j u_j (eigenpairs) and
// V is not needed.  Round-robin pairing, N - 1 rounds per
// sweep.  Both lanes of a pair compute bitwise-identical (alpha, beta, gamma)
// -- fma(x, y, z) is symmetric in x, y -- hence the same rotation.  The
// rotation angle only has to be accurate enough to converge: t comes from
// fp32 arithmetic on the power-of-two-scaled (beta - alpha, 2 gamma), while
// c = (1 + t^2)^-1/2 and s = c t are fp64, so every applied rotation is
// orthogonal to fp64 rounding.  Stops after a sweep whose largest relative
// off-diagonal |gamma| / sqrt(alpha beta) was below 1e-6 (quadratic
// convergence leaves ~1e-12 after it).  Returns the sweeps used (cap + 1
// when not converged).  Measured on B200 (tools/fp64_probe.cu): ~630 cycles
// per round at R = 10, about half of it the angle's dependent chain.
// ``n`` (<= R): the live columns -- the tournament pairs only those (a
// padded register width R with zero columns n.. needs no rotations).
template <int R, bool WITHV, bool LOOSE = false>
DP2_DEV int jacobi_cols(double (&a)[R], double (&v)[R], int n = R) {
  // stop threshold on the largest relative off-diagonal seen in a sweep
  // (squared): 1e-6 -> ~1e-12 left after it; LOOSE: 1e-4 -> ~1e-8
  constexpr float STOP2 = LOOSE ? 1e-8f : 1e-12f;
  constexpr int CAP = 40;
  const int N = n + (n & 1);
  constexpr double TOL = 4.0 * R * 2.220446049250313e-16, TOL2 = TOL * TOL;
  const int lane = threadIdx.x & 31;
  // round-robin partner (2 r - lane) mod (N - 1), advanced by 2 per round
  const int base0 = N > 1 ? (2 * (N - 1) - lane % (N - 1)) % (N - 1) : 0;
  for (int sw = 0; sw < CAP; ++sw) {
    bool big = false;
    int pr = base0;
#pragma unroll 1
    for (int r = 0; r < N - 1; ++r, pr = (pr + 2 >= N - 1) ? pr + 2 - (N - 1) : pr + 2) {
      int pj = pr;
      pj = (lane == r) ? N - 1 : pj;
      pj = (lane == N - 1) ? r : pj;
      const int p = lane < N ? pj : lane;
      double pa[R], pv[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        pa[i] = __shfl_sync(0xffffffffu, a[i], p);
        if (WITHV) pv[i] = __shfl_sync(0xffffffffu, v[i], p);
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
      const double g2ab = ga * ga, ab = alpha * beta;
      double c = 1.0, s = 0.0;
      if (p != lane && g2ab > TOL2 * ab) {
        const double d = beta - alpha, g2 = 2.0 * ga;
        const int hi = max(__double2hiint(alpha), __double2hiint(beta));  // both > 0
        const int ex = min(max(((hi >> 20) & 0x7ff) - 1023, -1000), 1000);
        const double sc = __hiloint2double((1023 - ex) << 20, 0);  // 2^-ex: max(alpha, beta) sc in [1, 2)
        const float df = (float)(d * sc), gf = (float)(g2 * sc);
        const float af = (float)(alpha * sc), bf = (float)(beta * sc);
        big |= 0.25f * gf * gf > STOP2 * (af * bf);  // relative off-diagonal above the stop threshold
        float tf = (df >= 0.f ? gf : -gf) * rcp_approx(fabsf(df) + sqrt_approx(fmaf(df, df, gf * gf)));
        double t = (double)tf;
        if (fabsf(tf) <= 1e-30f) t = g2 / (2.0 * d);  // |zeta| beyond fp32 range: t ~ 1 / (2 zeta)
        // c = (1 + t^2)^-1/2 to fp64 accuracy: fp32 estimate + two Newton steps
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
        if (WITHV) v[i] = fma(c, v[i], so * pv[i]);
      }
    }
    if (!__any_sync(0xffffffffu, big)) return sw + 1;
  }
  return CAP + 1;
}

// fp32 one-sided Jacobi (same pairing as jacobi_cols): the cheap first phase
// of a mixed-precision SVD -- rounds are shorter (half the shuffles, fp32
// latencies); it stops as below or after ``cap`` sweeps.  The caller
// re-orthonormalises V in fp64 and finishes with jacobi_cols.
template <int R>
DP2_DEV int jacobi_cols_f32(float (&a)[R], float (&v)[R], int cap, int n = R) {
  const int N = n + (n & 1);
  constexpr float TOL2 = 1e-11f, STOP2 = 1e-6f;  // rotate above fp32 noise; stop after a sweep with max ratio < 1e-3
  const int lane = threadIdx.x & 31;
  const int base0 = N > 1 ? (2 * (N - 1) - lane % (N - 1)) % (N - 1) : 0;
  for (int sw = 0; sw < cap; ++sw) {
    bool big = false;
    int pr = base0;
#pragma unroll 1
    for (int r = 0; r < N - 1; ++r, pr = (pr + 2 >= N - 1) ? pr + 2 - (N - 1) : pr + 2) {
      int pj = pr;
      pj = (lane == r) ? N - 1 : pj;
      pj = (lane == N - 1) ? r : pj;
      const int p = lane < N ? pj : lane;
      float pa[R], pv[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        pa[i] = __shfl_sync(0xffffffffu, a[i], p);
        pv[i] = __shfl_sync(0xffffffffu, v[i], p);
      }
      float al = 0.f, be = 0.f, ga = 0.f;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        al = fmaf(a[i], a[i], al);
        be = fmaf(pa[i], pa[i], be);
        ga = fmaf(a[i], pa[i], ga);
      }
      const bool lower = lane < p;
      const float alpha = lower ? al : be, beta = lower ? be : al;
      float c = 1.f, s = 0.f;
      if (p != lane && ga * ga > TOL2 * (alpha * beta)) {
        big |= ga * ga > STOP2 * (alpha * beta);
        const float d = beta - alpha, g2 = 2.f * ga;
        const float t = (d >= 0.f ? g2 : -g2) * rcp_approx(fabsf(d) + sqrt_approx(fmaf(d, d, g2 * g2)));
        c = rsqrt_approx(fmaf(t, t, 1.f));
        s = c * t;
      }
      const float so = lower ? -s : s;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        a[i] = fmaf(c, a[i], so * pa[i]);
        v[i] = fmaf(c, v[i], so * pv[i]);
      }
    }
    if (!__any_sync(0xffffffffu, big)) return sw + 1;
  }
  return cap;
}

DP2_DEV int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

}  // namespace dp2
