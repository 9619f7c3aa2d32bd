// Device helpers shared by the ALS translation units (dp2_als.cu and the
// persistent-loop instances dp2_als_ps*.cu): workspace buffer set, polar
// factor with orthonormal completion, warp R x R products and the R x R
// pseudo-inverse of the solves (P/linalg.py:135-151).
#pragma once
#include "dp2_common.cuh"

namespace dp2 {

struct AlsBufs {
  double *theta, *pprev, *cc, *nh, *HtH, *VtV, *pinv3, *G1, *WtW, *summed, *WtW2, *L;
  double *t3, *zz, *gp;  // R > 16 GEMM form of modes 2/3: R^3 stack product, R^3 operand, split-K partials
  double* pwarm;  // 3 x (R x R + 8): warm eigen bases of the solve_h / solve_v pinvs (block_pinv_sym)
  double *s_g1, *s_wtw, *s_m2, *s_wtw2, *s_e, *G2, *g3;
  double *GD, *ps_slots, *ps_e, *ps_C;  // persistent loop: D^T D, per-CTA partial slots, V = D C
  int64_t* ps_stamps;                  // persistent loop: optional phase stamps (64 iterations x 16)
  double* ps_gslots;                   // persistent loop: per-group partial slots
  unsigned* ps_gcnt;                   // persistent loop: per-group arrival counters
  int32_t* ctl;  // [0] stop flag, [1] warm-start valid, [8] persistent-loop grid barrier counter
  int nwt;       // total warps in the per-slice kernels
  int wpb;       // warps per block
  int nb;        // blocks == partial slots
  int nbm;       // metric kernel blocks (slots)
  int nbr, wpbr; // rotate kernel blocks (slots of s_g1 / s_wtw) and warps per block
};

__host__ __device__ inline int wpb_for(int R) { return R <= 16 ? 8 : (R <= 32 ? 4 : 1); }
__host__ __device__ inline int ldt_for(int R) { return R | 1; }
// per-warp smem: Ts, Vr (R x ldt), Fs, Th, Pi (R x R), two partial accumulators (R x R), tmp (4R)
__host__ __device__ inline size_t warp_smem_doubles(int R) {
  const int ldt = ldt_for(R);
  return (size_t)2 * R * ldt + 5 * (size_t)R * R + 4 * R;
}
__host__ __device__ inline size_t cta_shared_doubles(int R) { return 3 * (size_t)R * R + 2 * R; }

DP2_DEV uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct CtaShared {
  double *cc, *H, *E, *aux, *vec;
};
DP2_DEV CtaShared carve_cta(double* base, int R) {
  CtaShared s;
  s.cc = base;
  s.H = s.cc + R * R;
  s.E = s.H + R * R;
  s.aux = s.E + R;
  s.vec = s.aux + R * R;
  return s;
}

// ------------------------------------------------------------ polar factor
// Pi = Z P^T of T (column-major in Ts, already multiplied by the warm start
// Vr = P_prev) via one-sided Jacobi; exact-zero singular directions are
// completed to an orthonormal set (LAPACK likewise returns some completion).
DP2_DEV void warp_polar(double* Ts, double* Vr, int ldt, int R, double* pi, double* nrm, int64_t* status,
                        int64_t k) {
  const int lane = threadIdx.x & 31;
  const int sw = jacobi_onesided_warp(Ts, ldt, Vr, ldt, R);
  if (sw > 60 && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
  for (int i = lane; i < R; i += 32) {
    double s = 0.0;
    for (int a = 0; a < R; ++a) s = fma(Ts[i * ldt + a], Ts[i * ldt + a], s);
    nrm[i] = sqrt(s);
  }
  __syncwarp();
  for (int e = lane; e < R * R; e += 32) {
    const int i = e / R, a = e % R;
    const double n = nrm[i];
    Ts[i * ldt + a] = n > 1e-300 ? Ts[i * ldt + a] / n : 0.0;
  }
  __syncwarp();
  if (lane == 0) {
    bool def = false;
    for (int i = 0; i < R; ++i) def |= !(nrm[i] > 1e-300);
    if (def) {
      for (int i = 0; i < R; ++i) {
        if (nrm[i] > 1e-300) continue;
        for (int t = 0; t < R; ++t) {
          double* z = Ts + i * ldt;
          for (int a = 0; a < R; ++a) z[a] = (a == t) ? 1.0 : 0.0;
          for (int pass = 0; pass < 2; ++pass)
            for (int c = 0; c < R; ++c) {
              if (c == i || !(nrm[c] > 1e-300)) continue;
              double d = 0.0;
              for (int a = 0; a < R; ++a) d = fma(Ts[c * ldt + a], z[a], d);
              for (int a = 0; a < R; ++a) z[a] = fma(-d, Ts[c * ldt + a], z[a]);
            }
          double n2 = 0.0;
          for (int a = 0; a < R; ++a) n2 = fma(z[a], z[a], n2);
          if (n2 > 0.25) {
            const double inv = 1.0 / sqrt(n2);
            for (int a = 0; a < R; ++a) z[a] *= inv;
            nrm[i] = 1.0;
            break;
          }
        }
        if (!(nrm[i] > 1e-300)) status_min(status, ST_POLAR, k);
      }
    }
  }
  __syncwarp();
  for (int e = lane; e < R * R; e += 32) {  // Pi[a][d] = sum_i Z[a][i] P[d][i]
    const int a = e / R, d = e % R;
    double s = 0.0;
    for (int i = 0; i < R; ++i) s = fma(Ts[i * ldt + a], Vr[i * ldt + d], s);
    pi[e] = s;
  }
  __syncwarp();
}

// C = op(A) op(B) for R x R row-major smem matrices; lanes over outputs
template <int R, bool TA, bool TB>
DP2_DEV void wmm(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int it = 0; it < (R * R + 31) / 32; ++it) {
    const int e = lane + 32 * it;
    if (e < R * R) {
      const int i = e / R, j = e % R;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) s = fma(TA ? A[q * R + i] : A[i * R + q], TB ? B[j * R + q] : B[q * R + j], s);
      C[e] = s;
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------ solves (1 CTA)
// pinv of the symmetric PSD R x R Hadamard-of-Grams matrix (P/linalg.py:135-151).
// Fast path (warp 0): Cholesky A = L L^T and the explicit inverse; it is
// accepted when every pivot is positive and the Frobenius condition estimate
// ||A||_F ||A^-1||_F < 1e10, i.e. far from the reference's drop threshold
// (sigma <= R sigma_max 1e-12), where pinv(A) == inv(A) up to rounding.
// Otherwise: Jacobi eigen-decomposition with the reference's threshold.
DP2_DEV bool warp_chol_inverse(const double* A, int R, double* Lw, double* out, double* dinv) {
  const int lane = threadIdx.x & 31;
  // factor: column k pivot by lane 0, then lanes fill column k below the diagonal
  bool okay = true;
  for (int k = 0; k < R; ++k) {
    double d = 0.0;
    if (lane == 0) {
      double t = A[k * R + k];
      for (int m = 0; m < k; ++m) t = fma(-Lw[k * R + m], Lw[k * R + m], t);
      d = t;
    }
    d = __shfl_sync(0xffffffffu, d, 0);
    if (!(d > 0.0)) { okay = false; break; }
    const double l = sqrt(d);
    for (int i = k + 1 + lane; i < R; i += 32) {
      double t = A[i * R + k];
      for (int m = 0; m < k; ++m) t = fma(-Lw[i * R + m], Lw[k * R + m], t);
      Lw[i * R + k] = t / l;
    }
    if (lane == 0) Lw[k * R + k] = l;
    __syncwarp();
  }
  if (!okay) return false;
  // inverse: lane j solves L y = e_j then L^T x = y (column j of A^-1), in
  // place in ``out`` (shared) with reciprocal pivots -- no local arrays
  for (int i = lane; i < R; i += 32) dinv[i] = 1.0 / Lw[i * R + i];
  __syncwarp();
  double an = 0.0, in = 0.0;
  for (int j = lane; j < R; j += 32) {
    for (int i = 0; i < R; ++i) {
      double t = (i == j) ? 1.0 : 0.0;
      for (int m = j; m < i; ++m) t = fma(-Lw[i * R + m], out[m * R + j], t);
      out[i * R + j] = i < j ? 0.0 : t * dinv[i];
    }
    for (int i = R - 1; i >= 0; --i) {
      double t = out[i * R + j];
      for (int m = i + 1; m < R; ++m) t = fma(-Lw[m * R + i], out[m * R + j], t);
      out[i * R + j] = t * dinv[i];
    }
    for (int i = 0; i < R; ++i) {
      an = fma(A[i * R + j], A[i * R + j], an);
      in = fma(out[i * R + j], out[i * R + j], in);
    }
  }
  an = warp_sum(an);
  in = warp_sum(in);
  __syncwarp();
  return sqrt(an) * sqrt(in) < 1e10;
}

// Register Gauss-Jordan inverse, R known at compile time: lane c < 2R owns
// column c of [A | I] in registers; per pivot k the row factors come from
// lane k by shuffle, so a step is one reciprocal and R independent
// shuffle+FMA pairs (a runtime R would predicate every shuffle; measured 3.75x
// slower -- tools/inv_probe.cu).  No pivoting: only the SPD fast path, accepted
// under the Cholesky path's tests (positive pivots, ||A||_F ||A^-1||_F < 1e10).
template <int R>
DP2_DEV bool warp_gj_inverse(const double* A, double* out) {
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
  double an = 0.0, in = 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (lane < R) an = fma(A[i * R + lane], A[i * R + lane], an);
    if (lane >= R && lane < 2 * R) {
      out[i * R + (lane - R)] = col[i];
      in = fma(col[i], col[i], in);
    }
  }
  an = warp_sum(an);
  in = warp_sum(in);
  __syncwarp();
  return okay && sqrt(an) * sqrt(in) < 1e10;
}

DP2_DEV bool warp_fast_inverse(const double* A, int R, double* Lw, double* out, double* dinv) {
  switch (R) {
#define DP2_GJ(n) \
  case n:         \
    return warp_gj_inverse<n>(A, out);
    DP2_GJ(2) DP2_GJ(3) DP2_GJ(4) DP2_GJ(5) DP2_GJ(6) DP2_GJ(7) DP2_GJ(8) DP2_GJ(9) DP2_GJ(10) DP2_GJ(11) DP2_GJ(12)
    DP2_GJ(13) DP2_GJ(14) DP2_GJ(15) DP2_GJ(16)
#undef DP2_GJ
    default:
      return warp_chol_inverse(A, R, Lw, out, dinv);
  }
}

// RC > 0: R == RC known at compile time (no dispatch over the register inverses)
// ``warm`` (optional, global R x R + 1): the eigenvector basis of the previous
// call at this site and, in warm[R * R], 1.0 once it is valid.  The Jacobi
// fallback then diagonalises W^T A W starting from V = W (the ALS Gram
// products change little between iterations: a few sweeps instead of ~15
// from the identity) and leaves its basis there for the next call.
template <int RC = 0>
DP2_DEV void block_pinv_sym(double* A, double* U, double* out, int R, double* cs, int64_t* status,
                            double* warm = nullptr) {
  __shared__ double lmax;
  __shared__ int fast;
  if (threadIdx.x < 32) {
    bool okay;
    if constexpr (RC >= 2 && RC <= 16) okay = warp_gj_inverse<RC>(A, out);
    else okay = warp_fast_inverse(A, R, U, out, cs);
    if (threadIdx.x == 0) fast = okay ? 1 : 0;
  }
  __syncthreads();
  if (fast) return;
  const bool wv = warm != nullptr && warm[R * R] == 1.0;
  if (wv) {  // A <- W^T A W (symmetrised), U = W
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int i = e / R, c = e % R;
      double acc = 0.0;
      for (int q = 0; q < R; ++q) acc = fma(A[i * R + q], warm[q * R + c], acc);
      out[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int i = e / R, c = e % R;
      double acc = 0.0;
      for (int q = 0; q < R; ++q) acc = fma(warm[q * R + i], out[q * R + c], acc);
      U[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int i = e / R, c = e % R;
      A[e] = 0.5 * (U[i * R + c] + U[c * R + i]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) U[e] = warm[e];
    __syncthreads();
  }
  if (RC == 0 && R > 32) {  // large R: the whole block on the Jacobi rounds
    __shared__ int jflag;
    const int sw = jacobi_eig_block(A, R, U, R, R, cs, &jflag, 40, !wv);
    if (sw > 40 && threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int i = 0; i < R; ++i) m = fmax(m, fabs(A[i * R + i]));
      lmax = m;
    }
  } else if (threadIdx.x < 32) {
    const int sw = jacobi_eig_warp(A, R, U, R, R, cs, 40, !wv);
    if (sw > 40 && threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int i = 0; i < R; ++i) m = fmax(m, fabs(A[i * R + i]));
      lmax = m;
    }
  }
  __syncthreads();
  if (warm) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) warm[e] = U[e];
    if (threadIdx.x == 0) warm[R * R] = 1.0;
  }
  const double tolr = R * lmax * 1e-12;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e % R;
    double s = 0.0;
    if (lmax > 0.0)
      for (int q = 0; q < R; ++q) {
        const double l = A[q * R + q];
        if (fabs(l) > tolr) s += U[i * R + q] * (1.0 / l) * U[j * R + q];
      }
    out[e] = s;
  }
  __syncthreads();
}

}  // namespace dp2
