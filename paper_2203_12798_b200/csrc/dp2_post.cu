// Tensor checks, final Q assembly and fitness.
//   slice_stats : isfinite + squared norms per slice (P/tensor.py:61,79-80)
//   assemble_q  : Q_k = A_k (Z_k P_k^T)                (P/solver.py:186-189)
//   fitness     : sum ||X_k||^2, sum ||X_k - Q_k (H*w_k) V^T||^2 in one pass
//                 over X (P/analysis.py:23-45)
#include "dp2_common.cuh"
#include "dp2_internal.h"

namespace dp2 {

// per (slice, row-chunk) CTA: flat sum over the chunk's rows (cols < J); the
// chunk partials are summed per slice in chunk order (deterministic)
template <typename T>
__global__ void __launch_bounds__(256) slice_stats_kernel(const T* X, int64_t ldx, int64_t J,
                                                          const int64_t* row_off, int64_t K, int chunk_rows,
                                                          const int64_t* chunk_begin, double* part,
                                                          int64_t* status) {
  __shared__ double red[32];
  const int64_t c = blockIdx.x;
  // find the slice of chunk c (chunk_begin[k] = first chunk of slice k)
  int64_t lo = 0, hi = K;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (chunk_begin[mid] <= c) lo = mid; else hi = mid;
  }
  const int64_t k = lo;
  const int64_t r0 = row_off[k] + (c - chunk_begin[k]) * chunk_rows;
  const int64_t r1 = imin64(row_off[k + 1], r0 + chunk_rows);
  double s = 0.0;
  int bad = 0;
  for (int64_t r = r0; r < r1; ++r) {
    const T* row = X + r * ldx;
    for (int64_t j = threadIdx.x; j < J; j += blockDim.x) {
      const double v = (double)row[j];
      s = fma(v, v, s);
      bad |= !isfinite(v);
    }
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[c] = s;
  if (__syncthreads_or(bad) && threadIdx.x == 0) status_min(status, ST_NONFINITE, k);
}

__global__ void slice_stats_reduce(const int64_t* chunk_begin, int64_t K, const double* part, double* sqnorm) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  double s = 0.0;
  for (int64_t c = chunk_begin[k]; c < chunk_begin[k + 1]; ++c) s += part[c];
  sqnorm[k] = s;
}

__global__ void chunk_begin_kernel(const int64_t* row_off, int64_t K, int chunk_rows, int64_t* chunk_begin) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t c = 0;
  for (int64_t k = 0; k < K; ++k) {
    chunk_begin[k] = c;
    c += (row_off[k + 1] - row_off[k] + chunk_rows - 1) / chunk_rows;
  }
  chunk_begin[K] = c;
}

__global__ void __launch_bounds__(256) assemble_q_kernel(const double* A, const int32_t* piece_slice,
                                                          const int64_t* piece_row0, const int32_t* piece_rows,
                                                          int R, const double* polar, const double* sgn,
                                                          double* Q) {
  extern __shared__ double pis[];
  const int p = blockIdx.x;
  const int64_t k = piece_slice[p];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x)
    pis[e] = sgn ? sgn[k * R + e / R] * polar[k * R * R + e] : polar[k * R * R + e];
  __syncthreads();
  const int64_t r0 = piece_row0[p], nr = piece_rows[p];
  for (int64_t e = threadIdx.x; e < nr * R; e += blockDim.x) {
    const int64_t i = r0 + e / R;
    const int c = (int)(e % R);
    double acc = 0.0;
    for (int d = 0; d < R; ++d) acc = fma(A[i * R + d], pis[d * R + c], acc);
    Q[i * R + c] = acc;
  }
}

// Q rows = A rows Pi_k for R known at compile time: one thread per row, the
// row of A in registers, Pi_k in shared memory (broadcast reads), the same
// fma order as assemble_q_kernel (so results are bit-identical to it).
template <int R>
__global__ void __launch_bounds__(256) assemble_q_rows_kernel(const double* A, const int32_t* piece_slice,
                                                              const int64_t* piece_row0, const int32_t* piece_rows,
                                                              const double* polar, const double* sgn, double* Q) {
  __shared__ __align__(16) double pis[R * R];
  const int p = blockIdx.x;
  const int64_t k = piece_slice[p];
  // with sgn (the deferred column signs of A, dp2_stage1_signs): row d of
  // Pi_k times sign d, so unsigned A rows give the signed A's Q exactly
  for (int e = threadIdx.x; e < R * R; e += blockDim.x)
    pis[e] = sgn ? sgn[k * R + e / R] * polar[k * R * R + e] : polar[k * R * R + e];
  __syncthreads();
  const int64_t r0 = piece_row0[p];
  const int nr = piece_rows[p];
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    const double* a = A + (r0 + i) * R;
    double x[R], y[R];
    if constexpr (R % 2 == 0) {  // rows are 16-byte aligned: paired loads / stores
#pragma unroll
      for (int d = 0; d < R / 2; ++d) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(a) + d);
        x[2 * d] = v.x;
        x[2 * d + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int d = 0; d < R; ++d) x[d] = __ldg(a + d);
    }
    // y[c] = sum_d x[d] Pi[d][c], accumulated over d in order for every c
    // (the same fma chain per c as assemble_q_kernel); Pi's row d is read as
    // 16-byte pairs (half the shared-memory reads of a column-wise loop)
#pragma unroll
    for (int c = 0; c < R; ++c) y[c] = 0.0;
#pragma unroll
    for (int d = 0; d < R; ++d) {
      if constexpr (R % 2 == 0) {
#pragma unroll
        for (int c = 0; c < R / 2; ++c) {
          const double2 pp = reinterpret_cast<const double2*>(pis + d * R)[c];
          y[2 * c] = fma(x[d], pp.x, y[2 * c]);
          y[2 * c + 1] = fma(x[d], pp.y, y[2 * c + 1]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < R; ++c) y[c] = fma(x[d], pis[d * R + c], y[c]);
      }
    }
    double* q = Q + (r0 + i) * R;
    if constexpr (R % 2 == 0) {
#pragma unroll
      for (int c = 0; c < R / 2; ++c) reinterpret_cast<double2*>(q)[c] = make_double2(y[2 * c], y[2 * c + 1]);
    } else {
#pragma unroll
      for (int c = 0; c < R; ++c) q[c] = y[c];
    }
  }
}

// one warp per row: u = q H * w_k (R), recon_j = sum_a u_a V[j][a]
template <typename T>
__global__ void __launch_bounds__(256) fitness_kernel(const T* X, int64_t ldx, int64_t J,
                                                      const int32_t* piece_slice, const int64_t* piece_row0,
                                                      const int32_t* piece_rows, const double* Q, int R,
                                                      const double* H, const double* V, const double* W,
                                                      int v_in_smem, double* part) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  double* Hs = sm;                 // R x R
  double* us = Hs + R * R;         // 8 warps x R
  double* Vs = us + 8 * R;         // J x R (optional)
  const int p = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t k = piece_slice[p];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Hs[e] = H[e] * W[k * R + e % R];
  if (v_in_smem)
    for (int64_t e = threadIdx.x; e < J * R; e += blockDim.x) Vs[e] = V[e];
  __syncthreads();
  const double* Vp = v_in_smem ? Vs : V;
  const int64_t r0 = piece_row0[p], nr = piece_rows[p];
  double tot = 0.0, res = 0.0;
  double* u = us + warp * R;
  for (int64_t i = r0 + warp; i < r0 + nr; i += 8) {
    for (int c = lane; c < R; c += 32) {
      double acc = 0.0;
      for (int d = 0; d < R; ++d) acc = fma(Q[i * R + d], Hs[d * R + c], acc);
      u[c] = acc;
    }
    __syncwarp();
    for (int64_t j = lane; j < J; j += 32) {
      double rec = 0.0;
      for (int a = 0; a < R; ++a) rec = fma(u[a], Vp[j * R + a], rec);
      const double x = (double)X[i * ldx + j];
      const double d = x - rec;
      tot = fma(x, x, tot);
      res = fma(d, d, res);
    }
    __syncwarp();
  }
  tot = block_sum(tot, red);
  res = block_sum(res, red);
  if (threadIdx.x == 0) {
    part[2 * (size_t)p] = tot;
    part[2 * (size_t)p + 1] = res;
  }
}

__global__ void fitness_reduce_kernel(const double* part, int64_t np, double* out2) {
  if (threadIdx.x == 0) {
    double t = 0.0, r = 0.0;
    for (int64_t p = 0; p < np; ++p) {
      t += part[2 * p];
      r += part[2 * p + 1];
    }
    out2[0] = t;
    out2[1] = r;
  }
}

cudaError_t run_slice_stats(const dp2_store* st, double* sqnorm, int64_t* status, cudaStream_t stream) {
  // chunks of >= 64 rows; total chunks <= total_rows / 64 + K
  const int chunk_rows = 64;
  const int64_t K = st->K;
  const int64_t maxc = st->total_rows / chunk_rows + K + 1;
  int64_t* chunk_begin = nullptr;
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&chunk_begin, (K + 1) * sizeof(int64_t), stream);
  if (e == cudaSuccess) e = cudaMallocAsync(&part, maxc * sizeof(double), stream);
  if (e != cudaSuccess) return e;
  chunk_begin_kernel<<<1, 1, 0, stream>>>(st->row_off, K, chunk_rows, chunk_begin);
  int64_t nchunks = 0;
  e = cudaMemcpyAsync(&nchunks, chunk_begin + K, sizeof(int64_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  if (st->dtype == DP2_F64)
    slice_stats_kernel<double><<<(unsigned)nchunks, 256, 0, stream>>>(
        static_cast<const double*>(st->X), st->ldx, st->J, st->row_off, K, chunk_rows, chunk_begin, part, status);
  else
    slice_stats_kernel<float><<<(unsigned)nchunks, 256, 0, stream>>>(
        static_cast<const float*>(st->X), st->ldx, st->J, st->row_off, K, chunk_rows, chunk_begin, part, status);
  slice_stats_reduce<<<(unsigned)((K + 255) / 256), 256, 0, stream>>>(chunk_begin, K, part, sqnorm);
  cudaFreeAsync(part, stream);
  cudaFreeAsync(chunk_begin, stream);
  return cudaGetLastError();
}

cudaError_t run_assemble_q(const dp2_store* st, const double* A, int R, const double* polar, double* Q,
                           cudaStream_t stream, const double* sgn) {
  const unsigned P = (unsigned)st->npieces;
  switch (R) {
#define DP2_AQ(N)                                                                                             \
  case N:                                                                                                     \
    assemble_q_rows_kernel<N><<<P, 256, 0, stream>>>(A, st->piece_slice, st->piece_row0, st->piece_rows, polar, sgn, Q); \
    return cudaGetLastError();
    DP2_AQ(1) DP2_AQ(2) DP2_AQ(3) DP2_AQ(4) DP2_AQ(5) DP2_AQ(6) DP2_AQ(7) DP2_AQ(8) DP2_AQ(9) DP2_AQ(10)
    DP2_AQ(11) DP2_AQ(12) DP2_AQ(13) DP2_AQ(14) DP2_AQ(15) DP2_AQ(16)
#undef DP2_AQ
    default: break;
  }
  assemble_q_kernel<<<(unsigned)st->npieces, 256, (size_t)R * R * 8, stream>>>(
      A, st->piece_slice, st->piece_row0, st->piece_rows, R, polar, sgn, Q);
  return cudaGetLastError();
}

size_t fitness_bytes(const dp2_store* st) { return (size_t)st->npieces * 2 * 8 + 256; }

cudaError_t run_fitness(const dp2_store* st, const double* Q, int R, const double* H, const double* V,
                        const double* W, double* out2, char* ws, cudaStream_t stream) {
  double* part = reinterpret_cast<double*>(ws);
  const size_t vbytes = (size_t)st->J * R * 8;
  const int vin = vbytes <= 160 * 1024;
  const size_t smem = ((size_t)R * R + 8 * R) * 8 + (vin ? vbytes : 0);
  cudaError_t e;
  if (st->dtype == DP2_F64) {
    e = cudaFuncSetAttribute(fitness_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fitness_kernel<double><<<(unsigned)st->npieces, 256, smem, stream>>>(
        static_cast<const double*>(st->X), st->ldx, st->J, st->piece_slice, st->piece_row0, st->piece_rows, Q,
        R, H, V, W, vin, part);
  } else {
    e = cudaFuncSetAttribute(fitness_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fitness_kernel<float><<<(unsigned)st->npieces, 256, smem, stream>>>(
        static_cast<const float*>(st->X), st->ldx, st->J, st->piece_slice, st->piece_row0, st->piece_rows, Q,
        R, H, V, W, vin, part);
  }
  fitness_reduce_kernel<<<1, 32, 0, stream>>>(part, st->npieces, out2);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- zero-pass fitness
// for factors fresh from fit_dpar2 on an fp64 tensor,
//   ||X_k - Q_k G_k V^T||^2 = ||X_k||^2 - 2 tr(Pi_k G_k B_k) + ||G_k V^T||^2,
// G_k = H diag(w_k), B_k = V^T M_k (M_k the slice's block of the stage-1 M,
// MtV = M^T V holds B_k^T), Pi_k the polar factor (Q_k^T X_k = Pi_k^T M_k^T).
// One warp per slice; terms[k] = sq_k - 2 cross_k + norm_k.
__global__ void zero_pass_terms_kernel(const double* MtV, const double* H, const double* W, const double* polar,
                                       const double* VV, const double* sq, int64_t K, int R, double* terms) {
  const int lane = threadIdx.x & 31;
  const int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= K) return;
  const double* w = W + k * R;
  const double* Bt = MtV + k * R * R;  // Bt[c][b] = B_k[b][c]
  const double* P = polar + k * R * R;
  double cross = 0.0, norm = 0.0;
  for (int e = lane; e < R * R; e += 32) {
    const int j = e / R, i = e % R;
    // (G_k B_k)[j][i] = sum_b H[j][b] w[b] B_k[b][i]
    double gb = 0.0;
    for (int b = 0; b < R; ++b) gb = fma(H[j * R + b] * w[b], Bt[i * R + b], gb);
    cross = fma(P[i * R + j], gb, cross);
    // (G_k VV)[j][i] G_k[j][i]
    double gv = 0.0;
    for (int b = 0; b < R; ++b) gv = fma(H[j * R + b] * w[b], VV[b * R + i], gv);
    norm = fma(gv, H[j * R + i] * w[i], norm);
  }
  cross = warp_sum(cross);
  norm = warp_sum(norm);
  if (lane == 0) terms[k] = sq[k] - 2.0 * cross + norm;
}

// out2 = [sum_k sq_k, sum_k terms_k] in slice order (one thread: deterministic)
__global__ void zero_pass_reduce_kernel(const double* sq, const double* terms, int64_t K, double* out2) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    a += sq[k];
    b += terms[k];
  }
  out2[0] = a;
  out2[1] = b;
}

// VV = V^T V (R x R), one block, fixed-order sums over J
__global__ void gram_v_kernel(const double* V, int64_t J, int R, double* VV) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int a = e / R, b = e % R;
    double acc = 0.0;
    for (int64_t j = 0; j < J; ++j) acc = fma(V[j * R + a], V[j * R + b], acc);
    VV[e] = acc;
  }
}

size_t zero_pass_bytes(int64_t K, int R) { return ((size_t)K + (size_t)R * R) * 8 + 512; }

cudaError_t run_zero_pass_fitness(const double* MtV, int64_t K, int64_t J, int R, const double* H, const double* V,
                                  const double* W, const double* polar, const double* sq, double* out2, char* ws,
                                  cudaStream_t st) {
  double* terms = reinterpret_cast<double*>(ws);
  double* VV = terms + ((K + 31) & ~(int64_t)31);
  gram_v_kernel<<<1, 256, 0, st>>>(V, J, R, VV);
  zero_pass_terms_kernel<<<(unsigned)((K + 7) / 8), 256, 0, st>>>(MtV, H, W, polar, VV, sq, K, R, terms);
  zero_pass_reduce_kernel<<<1, 32, 0, st>>>(sq, terms, K, out2);
  return cudaGetLastError();
}

}  // namespace dp2
