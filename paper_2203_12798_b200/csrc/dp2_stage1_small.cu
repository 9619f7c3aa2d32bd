// Stage-1 per-slice factorizations for sketch widths s <= 32 (every config
// except the rank sweep's large R): the small-matrix steps between and after
// the two streaming passes, restructured for parallelism (see dp2_stage1.cu
// for the math; references P/linalg.py:124-131, P/compress.py:108).
//
//   orth_smem     Q_Z = CGS2(sum of pass-1 partials), slice matrix in smem
//   gram_y_piece  (tensor-core pass) per piece G partial = Y_p^T Y_p, DMMA
//   gather_dmma   C = sum of pass-2 partials; CC = C^T C (DMMA); G = sum of
//                 the per-piece Y^T Y partials
//   factor_warp   one warp per slice: G = L L^T (Cholesky; Jacobi-eig fallback
//                 for rank deficiency), B B^T = L^-1 CC L^-T, register Jacobi
//                 eig -> P = L^-T U_R, S = sqrt(mu_R)
//   argmax_cand   per piece: per-column max |A| (first index on ties)
//                 candidates of A = Y P, A not stored
//   signs_m       per slice: sign rule (P/linalg.py:62-70), P *= sign,
//                 M block = C^T P (= V S of the reference, P/compress.py:108)
//   write_a       A = Y P (signed P), one pass
#include "dp2_common.cuh"
#include "dp2_internal.h"
#include "dp2_small_linalg.cuh"

#include <algorithm>
#include <cstdlib>
#include <utility>

namespace dp2 {

// ------------------------------------------------------------ orth (smem CGS2)
__global__ void __launch_bounds__(256) orth_smem_kernel(const double* part, const int32_t* slice_piece,
                                                         const int32_t* s_k, int J, int sp, double* Q) {
  extern __shared__ __align__(16) double qs[];  // J x ld, ld = sp + 1 (odd: conflict-free column walks)
  __shared__ double h[32];
  __shared__ double red[32];
  const int k = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int p0 = slice_piece[k], p1 = slice_piece[k + 1];
  const int s = s_k[k], ld = sp + 1;
  const int n = J * sp;
  for (int i = tid; i < n; i += nt) {
    double acc = 0.0;
    for (int p = p0; p < p1; ++p) acc += part[(size_t)p * n + i];
    qs[(i / sp) * ld + i % sp] = acc;
  }
  __syncthreads();
  cgs2_smem(qs, J, ld, s, h, red);
  double* Qk = Q + (size_t)k * n;
  for (int i = tid; i < n; i += nt) Qk[i] = qs[(i / sp) * ld + i % sp];
}

// G partial of one piece from its pass-2 Y rows (tensor-core pass: Y fp32):
// each warp streams 32-row tiles through its own shared-memory slab (16 B
// loads) and accumulates the Gram blocks on fp64 DMMA.
template <typename Y, int SP>
__global__ void __launch_bounds__(256) gram_y_piece_kernel(const Y* y2, const int64_t* piece_row0,
                                                           const int32_t* piece_rows, double* gpart) {
  constexpr int EPC = 16 / (int)sizeof(Y), LD = SP + EPC, NBLK = GramBlocks<SP>::NBLK;
  extern __shared__ __align__(16) double sm[];
  const int p = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Y* tile = reinterpret_cast<Y*>(sm) + warp * 32 * LD;
  double* wpart = sm + (8 * 32 * LD * sizeof(Y)) / 8;
  const int64_t r0 = piece_row0[p];
  const int nr = piece_rows[p];
  double acc[NBLK][2];
#pragma unroll
  for (int b = 0; b < NBLK; ++b) acc[b][0] = acc[b][1] = 0.0;
  for (int t = warp * 32; t < nr; t += 256) {
    const int rows = min(32, nr - t);
    constexpr int NQ = SP / EPC;  // 16 B chunks per row; lane q-th chunk of the tile: all loads first
    float4 v[NQ];
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int q = lane + 32 * u, r = q / NQ, c = q - r * NQ;
      v[u] = r < rows ? __ldg(reinterpret_cast<const float4*>(y2 + (r0 + t + r) * SP + EPC * c))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int q = lane + 32 * u, r = q / NQ, c = q - r * NQ;
      *reinterpret_cast<float4*>(tile + r * LD + EPC * c) = v[u];
    }
    __syncwarp();
    gram_tile_dmma<SP, Y, LD>(tile, acc);
    __syncwarp();
  }
  gram_store<SP>(acc, wpart, gpart + (size_t)p * SP * SP);
}

// G partials of the fp32 Y rows (the tensor-core pass) on the FMA pipes.
// Per piece (one block of 4 warps): 128-row tiles of Y are double-buffered
// into shared memory with cp.async (row stride SP + 4 floats: conflict-free
// 16 B reads); warp h owns a quarter of the upper-triangle (a <= b) pairs and
// runs over all rows of a tile, 4 per lane (lane = row, the row in
// registers), accumulating in fp32 (Y carries the tf32-product error ~1e-4
// already; the <= nr / 32 term fp32 sums add ~1e-6).  The lanes are summed
// in fp64 in a fixed order -> gpart[p] (full symmetric SP x SP).  Replaces
// the DMMA Gram (the fp64 tensor pipe does 4x fewer FMAs per cycle).
template <int SP>
struct GramFfma {
  static constexpr int NP = SP * (SP + 1) / 2;
  static constexpr int NH = 4;                      // warps = pair groups
  static constexpr int NPH = (NP + NH - 1) / NH;
  static constexpr int TR = 128, LD = SP + 4;        // tile rows, row stride (floats)
  static constexpr size_t RING = (size_t)2 * TR * LD * 4;
  static constexpr size_t STAGE = (size_t)NH * NPH * 33 * 4;
  static constexpr size_t SMEM = RING > STAGE ? RING : STAGE;
};

// upper-triangle pair j -> (a, b), row-major over a (b >= a)
template <int SP>
DP2_DEV constexpr int pair_a(int j) {
  int a = 0;
  while (j >= SP - a) {
    j -= SP - a;
    ++a;
  }
  return a;
}
template <int SP>
DP2_DEV constexpr int pair_b(int j) {
  int a = 0;
  while (j >= SP - a) {
    j -= SP - a;
    ++a;
  }
  return a + j;
}
template <int SP, int PJ>
DP2_DEV void pair_fma(const float (&v)[SP], float& acc) {
  if constexpr (PJ < GramFfma<SP>::NP) {
    constexpr int a = pair_a<SP>(PJ), b = pair_b<SP>(PJ);
    acc = fmaf(v[a], v[b], acc);
  }
}
template <int SP, int H, int... J>
DP2_DEV void pairs_fma(const float (&v)[SP], float (&acc)[GramFfma<SP>::NPH], std::integer_sequence<int, J...>) {
  (pair_fma<SP, H * GramFfma<SP>::NPH + J>(v, acc[J]), ...);
}

template <int SP>
DP2_DEV void gram_tile_load(const float* y, int64_t r0, int nr, int t0, float* buf) {
  constexpr int Q = SP / 4, TR = GramFfma<SP>::TR, LD = GramFfma<SP>::LD;
  for (int e = threadIdx.x; e < TR * Q; e += blockDim.x) {
    const int r = e / Q, q = e - r * Q;
    const bool in = t0 + r < nr;
    cp_async16(buf + r * LD + 4 * q, y + (r0 + (in ? t0 + r : 0)) * SP + 4 * q, in ? 16 : 0);
  }
}

template <int SP, int H>
DP2_DEV void gram_ffma_piece(const float* y, int64_t r0, int nr, int lane, float* sm, double* red) {
  using GF = GramFfma<SP>;
  constexpr int NPH = GF::NPH, TR = GF::TR, LD = GF::LD;
  float acc[NPH];
#pragma unroll
  for (int j = 0; j < NPH; ++j) acc[j] = 0.f;
  const int ntile = (nr + TR - 1) / TR;
  gram_tile_load<SP>(y, r0, nr, 0, sm);
  cp_async_commit();
  for (int it = 0; it < ntile; ++it) {
    float* cur = sm + (it & 1) * TR * LD;
    if (it + 1 < ntile) gram_tile_load<SP>(y, r0, nr, (it + 1) * TR, sm + ((it + 1) & 1) * TR * LD);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
#pragma unroll 1
    for (int u = 0; u < TR / 32; ++u) {  // rows past the piece end are zero-filled
      const float4* row = reinterpret_cast<const float4*>(cur + (lane + 32 * u) * LD);
      float v[SP];
#pragma unroll
      for (int q = 0; q < SP / 4; ++q) {
        const float4 f = row[q];
        v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
      }
      pairs_fma<SP, H>(v, acc, std::make_integer_sequence<int, NPH>{});
    }
    __syncthreads();
  }
  // lane sums in fp64 through a (pair x lane) staging tile (row stride 33),
  // aliasing the (drained) tile ring
  float* stage = sm + H * NPH * 33;
#pragma unroll
  for (int j = 0; j < NPH; ++j) stage[j * 33 + lane] = acc[j];
  __syncwarp();
  for (int j = lane; j < NPH; j += 32) {
    double d = 0.0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) d += (double)stage[j * 33 + l];
    if (H * NPH + j < GF::NP) red[H * NPH + j] = d;
  }
}

template <int SP>
__global__ void __launch_bounds__(128) gram_y_ffma_kernel(const float* y2, const int64_t* piece_row0,
                                                          const int32_t* piece_rows, double* gpart) {
  using GF = GramFfma<SP>;
  __shared__ double red[GF::NH * GF::NPH];
  extern __shared__ __align__(16) float gsm[];
  const int p = blockIdx.x, lane = threadIdx.x & 31, h = threadIdx.x >> 5;
  const int64_t r0 = piece_row0[p];
  const int nr = piece_rows[p];
  switch (h) {
    case 0: gram_ffma_piece<SP, 0>(y2, r0, nr, lane, gsm, red); break;
    case 1: gram_ffma_piece<SP, 1>(y2, r0, nr, lane, gsm, red); break;
    case 2: gram_ffma_piece<SP, 2>(y2, r0, nr, lane, gsm, red); break;
    default: gram_ffma_piece<SP, 3>(y2, r0, nr, lane, gsm, red); break;
  }
  __syncthreads();
  double* out = gpart + (size_t)p * SP * SP;
  for (int e = threadIdx.x; e < SP * SP; e += blockDim.x) {
    int a = e / SP, b = e - a * SP;
    if (a > b) { const int t = a; a = b; b = t; }
    out[e] = red[a * SP - a * (a - 1) / 2 + (b - a)];  // upper-triangle pair index
  }
}

// Per slice: C = sum of the pass-2 partials (J x SP, written out), CC = C^T C
// on DMMA over warp tiles (lane = row, rows r, r + 256 of the slice: 16-byte
// loads of each piece's row), G = sum of the per-piece Y^T Y partials.
template <int SP, int RPT>
__global__ void __launch_bounds__(256) gather_dmma_kernel(const double* part, const double* gpart,
                                                          const int32_t* slice_piece, int J, double* Ct,
                                                          double* CCg, double* Gg) {
  constexpr int LD = SP + 1, NBLK = GramBlocks<SP>::NBLK;
  extern __shared__ __align__(16) double sm[];
  const int k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* tile = sm + warp * 32 * LD;
  double* wpart = sm + 8 * 32 * LD;
  const int p0 = slice_piece[k], p1 = slice_piece[k + 1];
  const size_t n = (size_t)J * SP;
  for (int e = tid; e < SP * SP; e += 256) {
    double acc = 0.0;
    for (int p = p0; p < p1; ++p) acc += gpart[(size_t)p * SP * SP + e];
    Gg[(size_t)k * SP * SP + e] = acc;
  }
  double acc[NBLK][2];
#pragma unroll
  for (int b = 0; b < NBLK; ++b) acc[b][0] = acc[b][1] = 0.0;
  double* C = Ct + (size_t)k * n;
#pragma unroll 1
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + 256 * u;
    double z[SP];
#pragma unroll
    for (int c = 0; c < SP; ++c) z[c] = 0.0;
    if (r < J) {
      for (int p = p0; p < p1; ++p) {
        const double2* src = reinterpret_cast<const double2*>(part + (size_t)p * n + (size_t)r * SP);
#pragma unroll
        for (int c = 0; c < SP / 2; ++c) {
          const double2 v = __ldg(src + c);
          z[2 * c] += v.x;
          z[2 * c + 1] += v.y;
        }
      }
      double2* dst = reinterpret_cast<double2*>(C + (size_t)r * SP);
#pragma unroll
      for (int c = 0; c < SP / 2; ++c) dst[c] = make_double2(z[2 * c], z[2 * c + 1]);
    }
#pragma unroll
    for (int c = 0; c < SP; ++c) tile[lane * LD + c] = z[c];
    __syncwarp();
    gram_tile_dmma<SP, double, LD>(tile, acc);
    __syncwarp();
  }
  gram_store<SP>(acc, wpart, CCg + (size_t)k * SP * SP);
}

// ------------------------------------------------------------ orth (CholQR2)
// Q_Z = orth(Z), Z = sum of the slice's pass-1 partials (P/linalg.py:124-126):
// CholQR -- G = Z^T Z on DMMA, G = L L^T, Z <- Z L^-T (row-wise substitution
// in registers); in exact arithmetic the Gram-Schmidt / positive-diagonal-QR
// Q.  One pass suffices here: Q_Z only seeds the second streaming pass, and
// everything downstream depends on span(Q_Z) alone, which a nonsingular right
// factor preserves up to the product's rounding; with the pivot guard below,
// kappa(Q_Z) <= 1 + ~1e-4.  A pivot below 1e-12 of the largest (kappa(Z)
// beyond ~1e6, or a dependent column) flags the slice for CGS2 with
// re-randomisation (orth_fallback_kernel).  Each lane keeps its rows of Z in
// registers (rows r, r + 256, ... of the slice); warp-private 32-row tiles in
// shared memory feed the DMMA Gram only, so two CTAs fit per SM.
// Three kernels so that no SM idles behind a serial Cholesky: the Gram of
// each slice (DMMA over warp tiles of Z rows), one warp per slice for the
// Cholesky (all slices at once), then the row-parallel substitution.  G and
// L are staged in the slice's own output slot (Q_k, J x SP), which the last
// kernel reads into shared memory before writing Q rows over it.
template <int SP, int RPT>  // RPT: rows per thread (J <= 256 RPT)
__global__ void __launch_bounds__(256) orth_gram_kernel(const double* part, const int32_t* slice_piece, int J,
                                                        double* Q) {
  constexpr int LD = SP + 1, NBLK = GramBlocks<SP>::NBLK;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* tile = sm + warp * 32 * LD;
  double* wpart = sm + 8 * 32 * LD;
  const int k = blockIdx.x;
  const int p0 = slice_piece[k], p1 = slice_piece[k + 1];
  const size_t n = (size_t)J * SP;
  double acc[NBLK][2];
#pragma unroll
  for (int b = 0; b < NBLK; ++b) acc[b][0] = acc[b][1] = 0.0;
#pragma unroll 1
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + 256 * u;
    double z[SP];
#pragma unroll
    for (int c = 0; c < SP; ++c) z[c] = 0.0;
    if (r < J)
      for (int p = p0; p < p1; ++p) {
        const double2* src = reinterpret_cast<const double2*>(part + (size_t)p * n + (size_t)r * SP);
#pragma unroll
        for (int c = 0; c < SP / 2; ++c) {
          const double2 v = __ldg(src + c);
          z[2 * c] += v.x;
          z[2 * c + 1] += v.y;
        }
      }
#pragma unroll
    for (int c = 0; c < SP; ++c) tile[lane * LD + c] = z[c];
    __syncwarp();
    gram_tile_dmma<SP, double, LD>(tile, acc);
    __syncwarp();
  }
  gram_store<SP>(acc, wpart, Q + (size_t)k * n);  // G into Q_k[0 : SP*SP]
}

template <int SP>
__global__ void __launch_bounds__(128) orth_chol_kernel(const int32_t* s_k, int K, int J, double* Q, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (k >= K) return;
  double* slot = Q + (size_t)k * J * SP;
  // G at slot[0 : SP^2], L to slot[SP^2 : 2 SP^2], 1/diag to slot[2 SP^2 : + SP]
  const bool ok = chol_reg<SP>(slot, SP, slot + SP * SP, SP, slot + 2 * SP * SP, s_k[k], 1e-12);
  if (lane == 0) flag[k] = ok ? 0 : 1;
}

template <int SP, int RPT>
__global__ void __launch_bounds__(256) orth_apply_kernel(const double* part, const int32_t* slice_piece,
                                                         const int32_t* s_k, int J, double* Q, const int32_t* flag) {
  __shared__ double L[SP * SP];
  __shared__ double dinv[SP];
  const int k = blockIdx.x, tid = threadIdx.x;
  if (flag[k]) return;  // orth_fallback_kernel
  const int p0 = slice_piece[k], p1 = slice_piece[k + 1];
  const int s = s_k[k];
  const size_t n = (size_t)J * SP;
  double* Qk = Q + (size_t)k * n;
  for (int e = tid; e < SP * SP; e += 256) L[e] = Qk[SP * SP + e];
  if (tid < SP) dinv[tid] = Qk[2 * SP * SP + tid];
  __syncthreads();
#pragma unroll 1
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + 256 * u;
    if (r >= J) break;
    double q[SP];
#pragma unroll
    for (int c = 0; c < SP; ++c) q[c] = 0.0;
    for (int p = p0; p < p1; ++p) {
      const double2* src = reinterpret_cast<const double2*>(part + (size_t)p * n + (size_t)r * SP);
#pragma unroll
      for (int c = 0; c < SP / 2; ++c) {
        const double2 v = __ldg(src + c);
        q[2 * c] += v.x;
        q[2 * c + 1] += v.y;
      }
    }
#pragma unroll
    for (int i = 0; i < SP; ++i) {
      if (i < s) {
        double t = q[i];
#pragma unroll
        for (int m = 0; m < i; ++m) t = fma(-L[i * SP + m], q[m], t);
        q[i] = t * dinv[i];
      }
    }
    double2* dst = reinterpret_cast<double2*>(Qk + (size_t)r * SP);
#pragma unroll
    for (int c = 0; c < SP / 2; ++c) dst[c] = make_double2(q[2 * c], q[2 * c + 1]);
  }
}

// the slices orth_cholqr flagged: CGS2 with re-randomisation on the shared-memory slab
__global__ void __launch_bounds__(256) orth_fallback_kernel(const double* part, const int32_t* slice_piece,
                                                            const int32_t* s_k, int J, int sp, double* Q,
                                                            const int32_t* flag) {
  extern __shared__ __align__(16) double qs[];
  __shared__ double h[32];
  __shared__ double red[32];
  const int k = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  if (!flag[k]) return;
  const int p0 = slice_piece[k], p1 = slice_piece[k + 1];
  const int s = s_k[k], ld = sp + 1;
  const int n = J * sp;
  for (int i = tid; i < n; i += nt) {
    double acc = 0.0;
    for (int p = p0; p < p1; ++p) acc += part[(size_t)p * n + i];
    qs[(i / sp) * ld + i % sp] = acc;
  }
  __syncthreads();
  cgs2_smem(qs, J, ld, s, h, red);
  double* Qk = Q + (size_t)k * n;
  for (int i = tid; i < n; i += nt) Qk[i] = qs[(i / sp) * ld + i % sp];
}

template <int SP, int RPT>
cudaError_t orth_rt(const dp2_store* st, const int32_t* s_dev, const double* part1, double* qz, int32_t* flag,
                    cudaStream_t stream) {
  constexpr int NBLK = GramBlocks<SP>::NBLK;
  const int K = (int)st->K, J = (int)st->J;
  if ((size_t)J * SP < (size_t)2 * SP * SP + SP) return cudaErrorInvalidValue;  // staging needs the slot
  const size_t bytes = ((size_t)8 * 32 * (SP + 1) + 8 * NBLK * 64) * 8;
  cudaError_t e = cudaFuncSetAttribute(orth_gram_kernel<SP, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes);
  if (e != cudaSuccess) return e;
  orth_gram_kernel<SP, RPT><<<K, 256, bytes, stream>>>(part1, st->slice_piece, J, qz);
  orth_chol_kernel<SP><<<(K + 3) / 4, 128, 0, stream>>>(s_dev, K, J, qz, flag);
  orth_apply_kernel<SP, RPT><<<K, 256, 0, stream>>>(part1, st->slice_piece, s_dev, J, qz, flag);
  const size_t qb = (size_t)J * (SP + 1) * 8;
  e = cudaFuncSetAttribute(orth_fallback_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qb);
  if (e != cudaSuccess) return e;
  orth_fallback_kernel<<<K, 256, qb, stream>>>(part1, st->slice_piece, s_dev, J, SP, qz, flag);
  return cudaGetLastError();
}

template <int SP>
cudaError_t orth_t(const dp2_store* st, const int32_t* s_dev, const double* part1, double* qz, int32_t* flag,
                   cudaStream_t stream) {
  const int J = (int)st->J;
  if ((size_t)J * (SP + 1) * 8 > 200 * 1024) return cudaErrorInvalidValue;  // no fallback slab
  if (J <= 256) return orth_rt<SP, 1>(st, s_dev, part1, qz, flag, stream);
  if (J <= 512) return orth_rt<SP, 2>(st, s_dev, part1, qz, flag, stream);
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------ factor (warp / slice)
template <int SP>
__global__ void __launch_bounds__(128) factor_warp_kernel(const double* Gg, const double* CCg, const int32_t* s_k,
                                                           int K, int sp, int R, double* Pm, double* Sv,
                                                           int32_t* rank_out, int64_t* status) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int k = blockIdx.x * (blockDim.x >> 5) + wib;
  const int ld = sp + 1;
  const size_t per = 4 * (size_t)sp * ld + 4 * (size_t)sp;
  double* G = sm + wib * per;   // L or T
  double* CC = G + sp * ld;     // X / Bg
  double* W = CC + sp * ld;
  double* U = W + sp * ld;
  double* lam = U + sp * ld;    // sp
  double* cs = lam + sp;        // 3 * (sp/2 + 1) <= 3 sp
  __shared__ int perm_s[4][64];
  int* perm = perm_s[wib];
  if (k >= K) return;
  const int s = s_k[k];
  for (int e = lane; e < s * s; e += 32) {
    const int a = e / s, b = e % s;
    G[a * ld + b] = Gg[(size_t)k * sp * sp + a * sp + b];
    CC[a * ld + b] = CCg[(size_t)k * sp * sp + a * sp + b];
  }
  __syncwarp();
  // ---- Cholesky of G with a relative pivot floor (registers; L overwrites G's
  // lower triangle, the upper triangle is not read afterwards)
  const bool chol = chol_reg<SP>(G, ld, G, ld, lam, s, 1e-13);
  int rp = s;
  if (chol) {
    // X = L^-1 CC (lanes own columns), then Bg = X L^-T: Bg[r][:] = (L^-1 X[r][:]^T)^T
    for (int c = lane; c < s; c += 32)
      for (int i = 0; i < s; ++i) {
        double t = CC[i * ld + c];
        for (int m = 0; m < i; ++m) t = fma(-G[i * ld + m], CC[m * ld + c], t);
        CC[i * ld + c] = t / G[i * ld + i];
      }
    __syncwarp();
    for (int r = lane; r < s; r += 32)
      for (int i = 0; i < s; ++i) {
        double t = CC[r * ld + i];
        for (int m = 0; m < i; ++m) t = fma(-G[i * ld + m], W[r * ld + m], t);
        W[r * ld + i] = t / G[i * ld + i];
      }
    __syncwarp();
    for (int e = lane; e < s * s; e += 32) {  // symmetrise into CC
      const int a = e / s, b = e % s;
      CC[a * ld + b] = 0.5 * (W[a * ld + b] + W[b * ld + a]);
    }
    __syncwarp();
  } else {
    // rank-deficient sketch: eigen basis of G, drop lambda <= 1e-13 lambda_max
    for (int e = lane; e < s * s; e += 32) {
      const int a = e / s, b = e % s;
      G[a * ld + b] = Gg[(size_t)k * sp * sp + a * sp + b];
    }
    __syncwarp();
    const int sw = jacobi_eig_warp(G, ld, W, ld, s, cs);
    if (sw > 40 && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
    if (lane == 0) {
      for (int i = 0; i < s; ++i) perm[i] = i;
      for (int i = 1; i < s; ++i) {
        const int v = perm[i];
        const double key = G[v * ld + v];
        int j = i - 1;
        while (j >= 0 && G[perm[j] * ld + perm[j]] < key) { perm[j + 1] = perm[j]; --j; }
        perm[j + 1] = v;
      }
    }
    __syncwarp();
    for (int i = lane; i < s; i += 32) lam[i] = G[perm[i] * ld + perm[i]];
    __syncwarp();
    const double lmax = lam[0] > 0.0 ? lam[0] : 0.0;
    rp = 0;
    for (int i = 0; i < s; ++i) rp += (lam[i] > 1e-13 * lmax && lam[i] > 0.0) ? 1 : 0;
    for (int e = lane; e < s * s; e += 32) {  // T = W[:, perm] / sqrt(lam) -> G
      const int a = e / s, c = e % s;
      G[a * ld + c] = c < rp ? W[a * ld + perm[c]] / sqrt(lam[c]) : 0.0;
    }
    __syncwarp();
    for (int e = lane; e < s * rp; e += 32) {  // tmp = CC T -> W
      const int a = e / rp, c = e % rp;
      double acc = 0.0;
      for (int b = 0; b < s; ++b) acc = fma(CC[a * ld + b], G[b * ld + c], acc);
      W[a * ld + c] = acc;
    }
    __syncwarp();
    for (int e = lane; e < rp * rp; e += 32) {  // Bg = T^T tmp -> U (then CC)
      const int a = e / rp, c = e % rp;
      double acc = 0.0;
      for (int b = 0; b < s; ++b) acc = fma(G[b * ld + a], W[b * ld + c], acc);
      U[a * ld + c] = acc;
    }
    __syncwarp();
    for (int e = lane; e < rp * rp; e += 32) {
      const int a = e / rp, c = e % rp;
      CC[a * ld + c] = 0.5 * (U[a * ld + c] + U[c * ld + a]);
    }
    __syncwarp();
  }
  // ---- eig(Bg) -> U, descending
  if (!eig_sym_reg<SP>(CC, ld, U, ld, rp)) {
    const int sw = jacobi_eig_warp(CC, ld, U, ld, rp, cs);
    if (sw > 40 && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
  }
  if (lane == 0) {
    for (int i = 0; i < rp; ++i) perm[i] = i;
    for (int i = 1; i < rp; ++i) {
      const int v = perm[i];
      const double key = CC[v * ld + v];
      int j = i - 1;
      while (j >= 0 && CC[perm[j] * ld + perm[j]] < key) { perm[j + 1] = perm[j]; --j; }
      perm[j + 1] = v;
    }
  }
  __syncwarp();
  double* Pk = Pm + (size_t)k * sp * R;
  double* Sk = Sv + (size_t)k * R;
  // P[:, r] = T U[:, perm[r]]:  Cholesky path solves L^T p = u (lanes over r)
  for (int r = lane; r < R; r += 32) {
    const double mu = r < rp ? CC[perm[r] * ld + perm[r]] : 0.0;
    Sk[r] = mu > 0.0 ? sqrt(mu) : 0.0;
    if (r >= rp) {
      for (int a = 0; a < sp; ++a) Pk[a * R + r] = 0.0;
      continue;
    }
    const int col = perm[r];
    if (chol) {
      for (int i = s - 1; i >= 0; --i) {
        double t = U[i * ld + col];
        for (int m = i + 1; m < s; ++m) t = fma(-G[m * ld + i], Pk[m * R + r], t);
        Pk[i * R + r] = t / G[i * ld + i];
      }
    } else {
      for (int a = 0; a < s; ++a) {
        double acc = 0.0;
        for (int b = 0; b < rp; ++b) acc = fma(G[a * ld + b], U[b * ld + col], acc);
        Pk[a * R + r] = acc;
      }
    }
    for (int a = s; a < sp; ++a) Pk[a * R + r] = 0.0;
  }
  __syncwarp();
  if (lane == 0) {
    int rk = 0;
    for (int r = 0; r < R; ++r) rk += Sk[r] > 0.0 ? 1 : 0;
    rank_out[k] = rk;
    if (rk < R) status_min(status, ST_RANKDEF, k);
  }
}

// One row of Y (SP entries, fp32 or fp64 storage) into fp64 registers, entries
// >= s zeroed (16 B loads).
// One row of Y (SP entries) into registers in its storage type (fp32 rows
// stay fp32: half the registers; the products convert exactly), entries >= s
// zeroed (16 B loads).
template <typename Y, int SP>
DP2_DEV void load_y_row(const Y* yr, int s, Y (&y)[SP]) {
  if constexpr (sizeof(Y) == 4) {
#pragma unroll
    for (int q = 0; q < SP / 4; ++q) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(yr) + q);
      y[4 * q] = f.x; y[4 * q + 1] = f.y; y[4 * q + 2] = f.z; y[4 * q + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < SP / 2; ++q) {
      const double2 f = __ldg(reinterpret_cast<const double2*>(yr) + q);
      y[2 * q] = f.x; y[2 * q + 1] = f.y;
    }
  }
#pragma unroll
  for (int a = 0; a < SP; ++a) y[a] = a < s ? y[a] : (Y)0;
}

// (y0 P[:, c], y1 P[:, c]) in fp64 with P stored transposed in shared memory
// (Pt = R x SP, rows >= s of P zero): fma over a = 0..SP-1 in order, so padded
// entries add exact zeros.
template <int SP, typename Y>
DP2_DEV void dot_pcol(const Y (&y0)[SP], const Y (&y1)[SP], const double* Pt, int c, double& a0, double& a1) {
  const double2* pc = reinterpret_cast<const double2*>(Pt + c * SP);
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int q = 0; q < SP / 2; ++q) {
    const double2 pp = pc[q];
    s0 = fma((double)y0[2 * q], pp.x, s0);
    s1 = fma((double)y1[2 * q], pp.x, s1);
    s0 = fma((double)y0[2 * q + 1], pp.y, s0);
    s1 = fma((double)y1[2 * q + 1], pp.y, s1);
  }
  a0 = s0;
  a1 = s1;
}

// (y0 P[:, c], y1 P[:, c]) in the rows' own type T (fp32 rows: fp32 products
// -- Y carries tf32-product error ~1e-4, the 1e-7 of an fp32 dot is below
// it; fp64 rows: fp64), P transposed in shared memory as T (rows >= s zero),
// fma over a = 0..SP-1 in order.
template <int SP, typename T>
DP2_DEV void dot_pcol_t(const T (&y0)[SP], const T (&y1)[SP], const T* Pt, int c, T& a0, T& a1) {
  T s0 = 0, s1 = 0;
  if constexpr (sizeof(T) == 4) {
    const float4* pc = reinterpret_cast<const float4*>(Pt + c * SP);
#pragma unroll
    for (int q = 0; q < SP / 4; ++q) {
      const float4 pp = pc[q];
      s0 = fmaf(y0[4 * q], pp.x, s0);
      s1 = fmaf(y1[4 * q], pp.x, s1);
      s0 = fmaf(y0[4 * q + 1], pp.y, s0);
      s1 = fmaf(y1[4 * q + 1], pp.y, s1);
      s0 = fmaf(y0[4 * q + 2], pp.z, s0);
      s1 = fmaf(y1[4 * q + 2], pp.z, s1);
      s0 = fmaf(y0[4 * q + 3], pp.w, s0);
      s1 = fmaf(y1[4 * q + 3], pp.w, s1);
    }
  } else {
    const double2* pc = reinterpret_cast<const double2*>(Pt + c * SP);
#pragma unroll
    for (int q = 0; q < SP / 2; ++q) {
      const double2 pp = pc[q];
      s0 = fma(y0[2 * q], pp.x, s0);
      s1 = fma(y1[2 * q], pp.x, s1);
      s0 = fma(y0[2 * q + 1], pp.y, s0);
      s1 = fma(y1[2 * q + 1], pp.y, s1);
    }
  }
  a0 = s0;
  a1 = s1;
}

// ------------------------------------------------------------ A = Y P and its argmax candidates
// Per piece: A = Y P for its rows, written UNSIGNED (the column signs are
// applied afterwards by apply_signs_kernel, or deferred to the caller), and
// the column-wise max |A| entry (first row on ties) as the piece's candidate
// for the sign rule.  One thread per row pair (rows i, i + 256 of a 512-row
// tile): the rows of Y in registers (16 B loads), R dot products against P in
// shared memory (broadcast), each A value both staged for a coalesced store
// and compared with the thread's running best (shared memory, per column);
// a thread's rows increase, so strict '>' keeps the first index, and the
// block merge orders ties by row.  The values written and the values
// compared are the same doubles, so the sign chosen from a candidate is the
// sign of the stored entry.
template <typename Y, int SP>
__global__ void __launch_bounds__(256) a_cand_kernel(const Y* y2, const int64_t* row_off,
                                                     const int32_t* piece_slice, const int64_t* piece_row0,
                                                     const int32_t* piece_rows, const int32_t* s_k,
                                                     const double* Pm, int R, double* A, double* cand_abs,
                                                     int64_t* cand_row, int32_t* cand_neg) {
  extern __shared__ __align__(16) double sm[];
  double* at = sm;                                   // 512 x R output tile
  double* bval = at + 512 * R;                       // R x 256 signed best values
  int* brow = reinterpret_cast<int*>(bval + R * 256);  // R x 256 row within the piece
  Y* Pt = reinterpret_cast<Y*>(brow + R * 256);      // R x SP (P transposed, as Y), entries a >= s zero
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = piece_slice[p], s = s_k[k];
  const int64_t base = row_off[k], r0 = piece_row0[p];
  const int nr = piece_rows[p];
  for (int i = tid; i < SP * R; i += 256) {
    const int c = i / SP, a = i - c * SP;
    Pt[i] = a < s ? (Y)Pm[(size_t)k * SP * R + a * R + c] : (Y)0;
  }
  for (int c = 0; c < R; ++c) brow[c * 256 + tid] = -1;  // own slots
  __syncthreads();
  for (int t0 = 0; t0 < nr; t0 += 512) {
    const int i = t0 + tid;
    if (i < nr) {
      const bool two = i + 256 < nr;
      Y y0[SP], y1[SP];
      load_y_row<Y, SP>(y2 + (r0 + i) * SP, s, y0);
      if (two) load_y_row<Y, SP>(y2 + (r0 + i + 256) * SP, s, y1);
      else {
#pragma unroll
        for (int a = 0; a < SP; ++a) y1[a] = (Y)0;
      }
#pragma unroll 1
      for (int c = 0; c < R; ++c) {
        Y a0y, a1y;
        dot_pcol_t<SP, Y>(y0, y1, Pt, c, a0y, a1y);
        const double a0 = (double)a0y, a1 = (double)a1y;  // exact widening: stored = compared
        at[tid * R + c] = a0;
        at[(tid + 256) * R + c] = a1;
        double bv = bval[c * 256 + tid];
        int rw = brow[c * 256 + tid];
        if (rw < 0 || fabs(a0) > fabs(bv)) { bv = a0; rw = i; }
        if (two && fabs(a1) > fabs(bv)) { bv = a1; rw = i + 256; }
        bval[c * 256 + tid] = bv;
        brow[c * 256 + tid] = rw;
      }
    }
    __syncthreads();
    const int rows = min(512, nr - t0);
    double* dst = A + (r0 + t0) * R;
    if ((R & 1) == 0) {  // the tile's rows are one contiguous, 16-byte aligned run
      const int n2 = rows * R / 2;
      for (int e = tid; e < n2; e += 256)
        reinterpret_cast<double2*>(dst)[e] = reinterpret_cast<const double2*>(at)[e];
    } else {
      for (int e = tid; e < rows * R; e += 256) dst[e] = at[e];
    }
    __syncthreads();
  }
  for (int c = warp; c < R; c += 8) {
    double ba = -1.0, bv = 0.0;
    int br = INT32_MAX;
    for (int t = lane; t < 256; t += 32) {
      const int rw = brow[c * 256 + t];
      if (rw < 0) continue;
      const double v = bval[c * 256 + t], a = fabs(v);
      if (a > ba || (a == ba && rw < br)) { ba = a; br = rw; bv = v; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oa = __shfl_xor_sync(0xffffffffu, ba, o);
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int orw = __shfl_xor_sync(0xffffffffu, br, o);
      if (oa > ba || (oa == ba && orw < br)) { ba = oa; br = orw; bv = ov; }
    }
    if (lane == 0) {
      cand_abs[(size_t)p * R + c] = ba;
      cand_row[(size_t)p * R + c] = br == INT32_MAX ? INT64_MAX : r0 + br - base;
      cand_neg[(size_t)p * R + c] = bv < 0.0;
    }
  }
}

// A rows of a piece *= the slice's column signs (in place, 16 B when R is even).
__global__ void __launch_bounds__(256) apply_signs_kernel(const int32_t* piece_slice, const int64_t* piece_row0,
                                                          const int32_t* piece_rows, const double* sgn, int R,
                                                          double* A) {
  __shared__ double sg[64];
  const int p = blockIdx.x, tid = threadIdx.x;
  const int k = piece_slice[p];
  if (tid < R) sg[tid] = sgn[(size_t)k * R + tid];
  __syncthreads();
  double* a = A + piece_row0[p] * R;
  const int64_t n = (int64_t)piece_rows[p] * R;
  if ((R & 1) == 0) {
    double2* a2 = reinterpret_cast<double2*>(a);
    for (int64_t e = tid; e < n / 2; e += 256) {
      const int c = (int)((2 * e) % R);
      double2 v = a2[e];
      v.x *= sg[c];
      v.y *= sg[c + 1];
      a2[e] = v;
    }
  } else {
    for (int64_t e = tid; e < n; e += 256) a[e] *= sg[e % R];
  }
}

// ------------------------------------------------------------ signs + M
template <int SP>
// sgn_out[k][r]: the sign A's column r takes (the candidate's sign for r below
// the slice's numerical rank, +1 for the columns complete_kernel replaces);
// P and M take the candidate's sign for every column.
// grid (K, row blocks): every block of slice k derives the slice's signs from
// the candidates (a few reads), the first one records them; each block forms
// M's rows for its share of j with P signed in shared memory (P itself is not
// needed signed afterwards).
__global__ void __launch_bounds__(128) signs_m_kernel(const int32_t* slice_piece, const double* cand_abs,
                                                       const int64_t* cand_row, const int32_t* cand_neg,
                                                       const double* Pm, const double* Ct, int K, int J, int sp,
                                                       int R, const int32_t* rank_found, double* sgn_out,
                                                       double* M) {
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;  // sp x R (signed)
  __shared__ double sgn[64];
  const int k = blockIdx.x, tid = threadIdx.x;
  const int p0 = slice_piece[k], p1 = slice_piece[k + 1];
  for (int r = tid; r < R; r += blockDim.x) {
    double ba = -1.0;
    int64_t br = INT64_MAX;
    int bn = 0;
    for (int p = p0; p < p1; ++p) {
      const double va = cand_abs[(size_t)p * R + r];
      const int64_t ra = cand_row[(size_t)p * R + r];
      if (va > ba || (va == ba && ra < br)) { ba = va; br = ra; bn = cand_neg[(size_t)p * R + r]; }
    }
    sgn[r] = bn ? -1.0 : 1.0;
    if (blockIdx.y == 0) sgn_out[(size_t)k * R + r] = r < rank_found[k] ? sgn[r] : 1.0;
  }
  __syncthreads();
  const double* Pk = Pm + (size_t)k * sp * R;
  for (int i = tid; i < sp * R; i += blockDim.x) Ps[i] = Pk[i] * sgn[i % R];
  __syncthreads();
  const double* C = Ct + (size_t)k * J * sp;
  const int64_t KR = (int64_t)K * R;
  // thread = row j of C (16 B loads), the slice's R outputs of M's row j
  for (int j = blockIdx.y * blockDim.x + tid; j < J; j += gridDim.y * blockDim.x) {
    double cr[SP];
    const double2* src = reinterpret_cast<const double2*>(C + (size_t)j * SP);
#pragma unroll
    for (int q = 0; q < SP / 2; ++q) {
      const double2 v = __ldg(src + q);
      cr[2 * q] = v.x;
      cr[2 * q + 1] = v.y;
    }
    double* mrow = M + j * KR + (int64_t)k * R;
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < SP; ++a) acc = fma(cr[a], Ps[a * R + r], acc);
      mrow[r] = acc;
    }
  }
}

// ------------------------------------------------------------ host
size_t small_factor_smem(int sp) { return (4 * (size_t)sp * (sp + 1) + 4 * (size_t)sp) * 8; }

// factor -> argmax candidates -> signs + M -> signed A, for padded width SP
template <int SP>
cudaError_t post_t(const dp2_store* st, const int32_t* s_dev, int R, const double* part2, const double* gpart,
                   double* gscratch, double* Gg, double* CCg, double* Ct, const double* y2, bool y32, double* Pm,
                   double* Sv, double* sgn, double* cand_abs, int64_t* cand_row, int32_t* cand_neg, double* A,
                   double* M, int32_t* rank_out, int64_t* status, cudaStream_t stream, double* a_signs) {
  const int K = (int)st->K, J = (int)st->J, P = (int)st->npieces;
  cudaError_t e = cudaSuccess;
  if (!gpart && !y32) {  // DMMA pass in column groups (J > 512): G partials per piece from its fp64 Y rows
    const size_t gs = (size_t)8 * 32 * (SP + 2) * 8 + (size_t)8 * GramBlocks<SP>::NBLK * 64 * 8;
    e = cudaFuncSetAttribute(gram_y_piece_kernel<double, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gs);
    if (e != cudaSuccess) return e;
    gram_y_piece_kernel<double, SP><<<P, 256, gs, stream>>>(y2, st->piece_row0, st->piece_rows, gscratch);
    gpart = gscratch;
  }
  if (!gpart) {  // tensor-core pass: G partials per piece from its fp32 Y rows
    static const bool dmma = getenv("DP2_GRAM_DMMA") && atoi(getenv("DP2_GRAM_DMMA")) != 0;
    if (dmma) {
      const size_t gs = (size_t)8 * 32 * (SP + 4) * 4 + (size_t)8 * GramBlocks<SP>::NBLK * 64 * 8;
      e = cudaFuncSetAttribute(gram_y_piece_kernel<float, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gs);
      if (e != cudaSuccess) return e;
      gram_y_piece_kernel<float, SP><<<P, 256, gs, stream>>>(reinterpret_cast<const float*>(y2), st->piece_row0,
                                                             st->piece_rows, gscratch);
    } else {
      const size_t fs = GramFfma<SP>::SMEM;
      e = cudaFuncSetAttribute(gram_y_ffma_kernel<SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs);
      if (e != cudaSuccess) return e;
      gram_y_ffma_kernel<SP><<<P, 128, fs, stream>>>(reinterpret_cast<const float*>(y2), st->piece_row0,
                                                     st->piece_rows, gscratch);
    }
    gpart = gscratch;
  }
  const size_t gb = ((size_t)8 * 32 * (SP + 1) + (size_t)8 * GramBlocks<SP>::NBLK * 64) * 8;
  if (J <= 256) {
    e = cudaFuncSetAttribute(gather_dmma_kernel<SP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb);
    if (e != cudaSuccess) return e;
    gather_dmma_kernel<SP, 1><<<K, 256, gb, stream>>>(part2, gpart, st->slice_piece, J, Ct, CCg, Gg);
  } else if (J <= 512) {
    e = cudaFuncSetAttribute(gather_dmma_kernel<SP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb);
    if (e != cudaSuccess) return e;
    gather_dmma_kernel<SP, 2><<<K, 256, gb, stream>>>(part2, gpart, st->slice_piece, J, Ct, CCg, Gg);
  } else {
    e = cudaFuncSetAttribute(gather_dmma_kernel<SP, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb);
    if (e != cudaSuccess) return e;
    gather_dmma_kernel<SP, 8><<<K, 256, gb, stream>>>(part2, gpart, st->slice_piece, J, Ct, CCg, Gg);
  }
  const int wpb = SP <= 24 ? 4 : 2;
  const size_t fs = wpb * small_factor_smem(SP);
  e = cudaFuncSetAttribute(factor_warp_kernel<SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs);
  if (e != cudaSuccess) return e;
  factor_warp_kernel<SP><<<(K + wpb - 1) / wpb, 32 * wpb, fs, stream>>>(Gg, CCg, s_dev, K, SP, R, Pm, Sv, rank_out,
                                                                          status);
  // A unsigned + candidates -> signs (and signed P, M) -> A signs applied,
  // unless the caller takes them (a_signs: A stays unsigned)
  const size_t as = (512 * (size_t)R + (size_t)R * 256) * 8 + (size_t)R * 256 * 4 + (size_t)SP * R * (y32 ? 4 : 8);
  double* sA = a_signs ? a_signs : sgn;
  if (y32) {
    e = cudaFuncSetAttribute(a_cand_kernel<float, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)as);
    if (e != cudaSuccess) return e;
    a_cand_kernel<float, SP><<<P, 256, as, stream>>>(reinterpret_cast<const float*>(y2), st->row_off,
                                                     st->piece_slice, st->piece_row0, st->piece_rows, s_dev, Pm, R,
                                                     A, cand_abs, cand_row, cand_neg);
  } else {
    e = cudaFuncSetAttribute(a_cand_kernel<double, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)as);
    if (e != cudaSuccess) return e;
    a_cand_kernel<double, SP><<<P, 256, as, stream>>>(y2, st->row_off, st->piece_slice, st->piece_row0,
                                                      st->piece_rows, s_dev, Pm, R, A, cand_abs, cand_row, cand_neg);
  }
  signs_m_kernel<SP><<<dim3(K, std::min(16, (J + 127) / 128)), 128, (size_t)SP * R * 8, stream>>>(
      st->slice_piece, cand_abs, cand_row, cand_neg, Pm, Ct, K, J, SP, R, rank_out, sA, M);
  if (!a_signs)
    apply_signs_kernel<<<P, 256, 0, stream>>>(st->piece_slice, st->piece_row0, st->piece_rows, sA, R, A);
  return cudaGetLastError();
}

cudaError_t run_stage1_small(const dp2_store* st, const int32_t* s_dev, int sp, int R, const double* part1,
                             const double* part2, const double* gpart, double* qz, double* Ct, double* CCg,
                             double* Gg, const double* y2, double* Pm, double* Sv, double* sgn, double* cand_abs,
                             int64_t* cand_row, int32_t* cand_neg, double* A, double* M, int32_t* rank_out,
                             int64_t* status, int phase, cudaStream_t stream, bool y32, double* gscratch,
                             double* a_signs) {
  const int K = (int)st->K, J = (int)st->J;
  cudaError_t e = cudaSuccess;
  if (phase == 0) {  // between the passes
    cudaError_t eo = cudaErrorInvalidValue;
    int32_t* flag = reinterpret_cast<int32_t*>(gscratch);  // free until pass 2's Gram partials
    switch (sp) {
      case 8: eo = orth_t<8>(st, s_dev, part1, qz, flag, stream); break;
      case 16: eo = orth_t<16>(st, s_dev, part1, qz, flag, stream); break;
      case 24: eo = orth_t<24>(st, s_dev, part1, qz, flag, stream); break;
      case 32: eo = orth_t<32>(st, s_dev, part1, qz, flag, stream); break;
      default: break;
    }
    if (eo == cudaSuccess) return eo;
    (void)cudaGetLastError();  // slab does not fit: shared-memory CGS2
    const size_t qb = (size_t)J * (sp + 1) * 8;
    e = cudaFuncSetAttribute(orth_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qb);
    if (e != cudaSuccess) return e;
    orth_smem_kernel<<<K, 256, qb, stream>>>(part1, st->slice_piece, s_dev, J, sp, qz);
    return cudaGetLastError();
  }
  switch (sp) {
    case 8: return post_t<8>(st, s_dev, R, part2, gpart, gscratch, Gg, CCg, Ct, y2, y32, Pm, Sv, sgn, cand_abs, cand_row, cand_neg, A, M, rank_out, status, stream, a_signs);
    case 16: return post_t<16>(st, s_dev, R, part2, gpart, gscratch, Gg, CCg, Ct, y2, y32, Pm, Sv, sgn, cand_abs, cand_row, cand_neg, A, M, rank_out, status, stream, a_signs);
    case 24: return post_t<24>(st, s_dev, R, part2, gpart, gscratch, Gg, CCg, Ct, y2, y32, Pm, Sv, sgn, cand_abs, cand_row, cand_neg, A, M, rank_out, status, stream, a_signs);
    case 32: return post_t<32>(st, s_dev, R, part2, gpart, gscratch, Gg, CCg, Ct, y2, y32, Pm, Sv, sgn, cand_abs, cand_row, cand_neg, A, M, rank_out, status, stream, a_signs);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dp2
