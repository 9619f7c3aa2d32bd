// Small dense linear algebra shared by the stage-1 and stage-2 kernels
// (device code only): DMMA Gram tiles, register Cholesky, register Jacobi
// eigensolver, CGS2 with re-randomisation.
#pragma once
#include "dp2_common.cuh"

namespace dp2 {

// CGS2 with re-randomisation of (numerically) dependent columns on the
// columns c < s of the J x ld shared-memory block qs (whole CTA).
DP2_DEV void cgs2_smem(double* qs, int J, int ld, int s, double* h, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int c = 0; c < s; ++c) {
    for (int attempt = 0;; ++attempt) {
      if (attempt > 0) {
        const int e = (c + attempt - 1) % J;
        for (int i = tid; i < J; i += nt) qs[i * ld + c] = (i == e) ? 1.0 : 0.0;
        __syncthreads();
      }
      for (int pass = 0; pass < 2; ++pass) {
        for (int i = warp; i < c; i += nw) {
          double acc = 0.0;
          for (int r = lane; r < J; r += 32) acc = fma(qs[r * ld + i], qs[r * ld + c], acc);
          acc = warp_sum(acc);
          if (lane == 0) h[i] = acc;
        }
        __syncthreads();
        for (int r = tid; r < J; r += nt) {
          double acc = qs[r * ld + c];
          for (int i = 0; i < c; ++i) acc = fma(-h[i], qs[r * ld + i], acc);
          qs[r * ld + c] = acc;
        }
        __syncthreads();
      }
      double part2 = 0.0;
      for (int r = tid; r < J; r += nt) part2 = fma(qs[r * ld + c], qs[r * ld + c], part2);
      const double nrm2 = block_sum(part2, red);
      const bool ok = attempt == 0 ? (nrm2 > 1e-300) : (nrm2 > 0.25);
      if (ok || attempt > J + 1) {
        const double inv = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
        for (int r = tid; r < J; r += nt) qs[r * ld + c] *= inv;
        __syncthreads();
        break;
      }
    }
  }
}

// ------------------------------------------------------------ DMMA Gram tiles
// Upper-triangular 8x8 blocks (bi <= bj) of T^T T for a 32-row tile T held in
// warp-private shared memory (row stride LD): 8 k-steps of m8n8k4 per block.
template <int SP>
struct GramBlocks {
  static constexpr int NB = SP / 8, NBLK = NB * (NB + 1) / 2;
};

template <int SP, typename T, int LD>
DP2_DEV void gram_tile_dmma(const T* tile, double (&acc)[GramBlocks<SP>::NBLK][2]) {
  constexpr int NB = SP / 8;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const T* tr = tile + (4 * kk + (lane & 3)) * LD + (lane >> 2);
    double f[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) f[b] = (double)tr[8 * b];
    int blk = 0;
#pragma unroll
    for (int bi = 0; bi < NB; ++bi)
#pragma unroll
      for (int bj = bi; bj < NB; ++bj, ++blk) dmma_8x8x4(acc[blk][0], acc[blk][1], f[bi], f[bj]);
  }
}

// Block partials of every warp -> full symmetric SP x SP matrix (warp order)
template <int SP>
DP2_DEV void gram_store(double (&acc)[GramBlocks<SP>::NBLK][2], double* wpart, double* out) {
  constexpr int NB = SP / 8, NBLK = GramBlocks<SP>::NBLK;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int blk = 0; blk < NBLK; ++blk) {
    wpart[(warp * NBLK + blk) * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = acc[blk][0];
    wpart[(warp * NBLK + blk) * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc[blk][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < SP * SP; e += blockDim.x) {
    int a = e / SP, b = e - a * SP;
    if (a / 8 > b / 8) { const int t = a; a = b; b = t; }
    const int bi = a / 8, bj = b / 8;
    const int blk = bi * NB - bi * (bi - 1) / 2 + (bj - bi);
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += wpart[(w * NBLK + blk) * 64 + (a % 8) * 8 + (b % 8)];
    out[e] = v;
  }
}

// Cholesky of the s x s Gram G (shared, row stride ldg) by one warp into L
// (lower, row-major, stride SP) and 1/diag; false when a pivot falls to
// rel_floor * max diag(G) (the caller then falls back to CGS2).
DP2_DEV bool chol_warp_smem(const double* G, int ldg, double* L, int ldl, double* dinv, int s, double rel_floor) {
  const int lane = threadIdx.x & 31;
  double gmax = 0.0;
  for (int i = 0; i < s; ++i) gmax = fmax(gmax, G[i * ldg + i]);
  if (!(gmax > 0.0)) return false;
  for (int c = 0; c < s; ++c) {
    double d = 0.0;
    if (lane == 0) {
      d = G[c * ldg + c];
      for (int m = 0; m < c; ++m) d = fma(-L[c * ldl + m], L[c * ldl + m], d);
    }
    d = __shfl_sync(0xffffffffu, d, 0);
    if (!(d > rel_floor * gmax)) return false;
    const double l = sqrt(d), il = 1.0 / l;
    for (int i = c + 1 + lane; i < s; i += 32) {
      double t = G[i * ldg + c];
      for (int m = 0; m < c; ++m) t = fma(-L[i * ldl + m], L[c * ldl + m], t);
      L[i * ldl + c] = t * il;
    }
    if (lane == 0) {
      L[c * ldl + c] = l;
      dinv[c] = il;
    }
    __syncwarp();
  }
  return true;
}

// Register Cholesky of the s x s SPD matrix G (s <= SP <= 32), one warp:
// lane j holds column j; step k broadcasts the scaled pivot column by
// shuffles (entries below the diagonal only) and every lane updates its own
// column.  Writes L (lower, row-major) and 1/diag; false when a pivot falls to
// rel_floor * max diag(G).
template <int SP>
DP2_DEV bool chol_reg(const double* G, int ldg, double* L, int ldl, double* dinv, int s, double rel_floor) {
  const int lane = threadIdx.x & 31;
  double g[SP];
#pragma unroll
  for (int i = 0; i < SP; ++i) g[i] = (lane < s && i < s) ? G[i * ldg + lane] : 0.0;
  double dg = 0.0;
#pragma unroll
  for (int i = 0; i < SP; ++i) dg = (i == lane) ? g[i] : dg;
  double gmax = dg;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
  if (!(gmax > 0.0)) return false;
#pragma unroll
  for (int k = 0; k < SP; ++k) {
    if (k >= s) break;
    const double d = __shfl_sync(0xffffffffu, g[k], k);
    if (!(d > rel_floor * gmax)) return false;
    const double l = sqrt(d), il = 1.0 / l;
    double lk[SP];
#pragma unroll
    for (int i = k + 1; i < SP; ++i) lk[i] = __shfl_sync(0xffffffffu, g[i], k) * il;
    double ljk = 0.0;
#pragma unroll
    for (int i = k + 1; i < SP; ++i) ljk = (i == lane) ? lk[i] : ljk;
    if (lane > k && lane < s) {
#pragma unroll
      for (int i = k + 1; i < SP; ++i) g[i] = fma(-lk[i], ljk, g[i]);
    }
    if (lane == k) {
      L[k * ldl + k] = l;
      dinv[k] = il;
#pragma unroll
      for (int i = k + 1; i < SP; ++i)
        if (i < s) L[i * ldl + k] = lk[i];
    }
  }
  __syncwarp();
  return true;
}

// Symmetric PSD eigenproblem (n <= SP) by register one-sided Jacobi: lane j
// holds column j; converged columns are lambda_j u_j, so the eigenvalues are
// the column norms (written to A's diagonal) and the eigenvectors the
// normalised columns (into U's columns).  Returns false (caller falls back to
// the shared-memory two-sided Jacobi) on an exactly zero or non-finite column
// norm or no convergence.
template <int SP>
DP2_DEV bool eig_sym_reg(double* A, int lda, double* U, int ldu, int n) {
  const int lane = threadIdx.x & 31;
  double a[SP], dummy[SP];
  // (fp64 throughout: these are Gram-type matrices whose condition number is
  // squared -- fp32 sweeps cannot resolve the small eigenvalues, measured
  // slower than fp64 alone)
#pragma unroll
  for (int i = 0; i < SP; ++i) a[i] = (lane < n && i < n) ? A[i * lda + lane] : 0.0;
  const int sw = jacobi_cols<SP, false>(a, dummy, n);
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < SP; ++i) s2 = fma(a[i], a[i], s2);
  const double lam = sqrt(s2);
  const bool bad = lane < n && !(lam > 0.0 && lam < 1e300);
  __syncwarp();
  if (__any_sync(0xffffffffu, bad) || sw > 40) return false;
  if (lane < n) {
    const double inv = 1.0 / lam;
#pragma unroll
    for (int i = 0; i < SP; ++i)
      if (i < n) U[i * ldu + lane] = a[i] * inv;
  }
  __syncwarp();
  if (lane < n) A[lane * lda + lane] = lam;
  __syncwarp();
  return true;
}

}  // namespace dp2
