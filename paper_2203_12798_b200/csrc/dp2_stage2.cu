// Stage 2: randomized SVD of the concatenated right parts
// M = [V_1 S_1 | ... | V_K S_K] (J x KR, P/compress.py:108-111), fp64.
//
//   Y  = M Omega2           (J x s2)     DMMA split-K partials + ordered reduce
//   Z  = M^T Y              (KR x s2)    DMMA
//   Y2 = M Z                (J x s2)     = the reference's M (M^T M Omega2)
//   Q2 = orth(Y2)                        CholQR2 in one CTA (CGS2 fallback; the reference's np.linalg.qr)
//   C  = M^T Q2             (KR x s2)    B2 = Q2^T M = C^T
//   B2 B2^T = C^T C = U mu U^T           register Jacobi (block Jacobi fallback); E = sqrt(mu_R)
//   D = Q2 U_R (sign rule, P/linalg.py:62-70), F = C U_R / E (same flips)
#include "dp2_common.cuh"
#include "dp2_internal.h"
#include "dp2_small_linalg.cuh"

#include <algorithm>

namespace dp2 {

// ---------------------------------------------------------------- skinny fp64 GEMMs (DMMA)
// The four products with M (J x KR) and the Gram C^T C are tall-skinny fp64
// GEMMs: every output is s2 (<= ~100) columns wide, so they stream M (or C)
// once with m8n8k4 DMMA fragments read straight from global memory (M is
// L2-resident between the passes: 41 MB at c2) and write per-split partials
// that a fixed-order reduction sums (deterministic, like the reference's
// ascending reductions).

// part[ks] (m x n) = A[:, ks-th K range] B[ks-th K range, :], A row-major (m x K),
// B row-major (K x n).  Block: 8 warps; warp w -> output rows 64 bx + 8 w,
// columns 24 bz .. +24 (3 DMMA n-blocks).
__global__ void __launch_bounds__(256) nn_dmma_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                       int64_t K, const double* __restrict__ B, int ldb, int n,
                                                       int64_t kc, double* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 64 + warp * 8 + (lane >> 2);
  const int ks = blockIdx.y, c0 = blockIdx.z * 24;
  const int64_t k0 = (int64_t)ks * kc, k1 = imin64(K, k0 + kc);
  const bool rok = row < m;
  const double* a = A + (rok ? row : 0) * lda + (lane & 3);
  const int bcol = c0 + (lane >> 2);
  double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
  for (int64_t k = k0; k < k1; k += 4) {
    const int64_t kk = k + (lane & 3);
    const bool kok = kk < k1;
    const double av = (rok && kok) ? __ldg(a + k) : 0.0;
    const double* b = B + (kok ? kk : 0) * ldb;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = bcol + 8 * j;
      const double bv = (kok && c < n) ? __ldg(b + c) : 0.0;
      dmma_8x8x4(acc[j][0], acc[j][1], av, bv);
    }
  }
  // C fragment: row (lane >> 2) of the warp's block, columns 8 j + 2 (lane & 3), +1
  const int64_t orow = (int64_t)blockIdx.x * 64 + warp * 8 + (lane >> 2);
  if (orow < m) {
    double* o = part + ((size_t)ks * m + orow) * n;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = c0 + 8 * j + 2 * (lane & 3);
      if (c < n) o[c] = acc[j][0];
      if (c + 1 < n) o[c + 1] = acc[j][1];
    }
  }
}

// part[ms] (K x n) = A[ms-th m range, :]^T B[ms-th m range, :], A row-major (m x K),
// B row-major (m x n).  Warp w -> output rows (columns of A) 64 bx + 8 w, +8.
__global__ void __launch_bounds__(256) tn_dmma_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                       int64_t K, const double* __restrict__ B, int ldb, int n,
                                                       int64_t mc, double* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t acol = (int64_t)blockIdx.x * 64 + warp * 8 + (lane >> 2);  // A-fragment row = column of A
  const int c0 = blockIdx.z * 24, ms = blockIdx.y;
  const int64_t m0 = (int64_t)ms * mc, m1 = imin64(m, m0 + mc);
  const bool cok = acol < K;
  const int bcol = c0 + (lane >> 2);
  double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
  for (int64_t i = m0; i < m1; i += 4) {
    const int64_t ii = i + (lane & 3);
    const bool iok = ii < m1;
    const double av = (cok && iok) ? __ldg(A + ii * lda + acol) : 0.0;
    const double* b = B + (iok ? ii : 0) * ldb;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = bcol + 8 * j;
      const double bv = (iok && c < n) ? __ldg(b + c) : 0.0;
      dmma_8x8x4(acc[j][0], acc[j][1], av, bv);
    }
  }
  const int64_t orow = (int64_t)blockIdx.x * 64 + warp * 8 + (lane >> 2);
  if (orow < K) {
    double* o = part + ((size_t)ms * K + orow) * n;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = c0 + 8 * j + 2 * (lane & 3);
      if (c < n) o[c] = acc[j][0];
      if (c + 1 < n) o[c + 1] = acc[j][1];
    }
  }
}

__global__ void reduce_parts_kernel(const double* part, int nparts, int64_t size, double* out) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < size;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < nparts; ++c) acc += part[(size_t)c * size + idx];
    out[idx] = acc;
  }
}

// Q2 = orth(Y2) (J x s, row-major, in place), one CTA: the J x SP slab in
// shared memory, shifted CholeskyQR3 (G = Y^T Y on DMMA, register Cholesky,
// row substitution): a shifted pass, a plain pass, then a plain pass whose
// pivots must stay above 1e-3 of the largest -- i.e. the columns entering it
// are orthonormal to ~1e-3 -- else CGS2 with re-randomisation (cgs2_smem).
// The middle pass has no pivot floor: its job is to finish what the shifted
// pass started, and a (numerically) rank-deficient Y2 -- noiseless rank-R
// data with s2 > R -- is caught by the last pass's floor or leaves
// orthonormal columns either way (tests/test_gpu_stage2.py).
template <int SP>
__global__ void __launch_bounds__(256) orth2_cholqr_kernel(double* Y2, int J, int s) {
  constexpr int LD = SP + 1, NBLK = GramBlocks<SP>::NBLK;
  extern __shared__ __align__(16) double sm[];
  __shared__ double h[32];
  __shared__ double red[32];
  __shared__ int ok_s;
  const int JP = (J + 31) & ~31;
  double* Z = sm;
  double* wpart = Z + (size_t)JP * LD;
  double* G = wpart + 8 * NBLK * 64;
  double* L = G + SP * SP;
  double* dinv = L + SP * SP;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < JP * SP; i += 256) {
    const int r = i / SP, c = i - r * SP;
    Z[r * LD + c] = (r < J && c < s) ? Y2[(size_t)r * s + c] : 0.0;
  }
  __syncthreads();
  // Shifted CholeskyQR3: the power iteration makes Y2 = M M^T M Omega
  // ill-conditioned (plain CholQR fails its pivot floor on such inputs), so
  // the first pass factors G + 11 (J s + s (s + 1)) u ||Y||_F^2 I -- always
  // positive definite, leaving kappa ~ u^-1/2 -- and two plain passes then
  // orthonormalise to rounding.  A failure past that takes CGS2.  (Q2 enters
  // stage 2 only through its range.)
  // mode: 1 shifted, 2 plain, 3 last plain (pivot floor 1e-3), 4 done
  bool chol = true;
  int mode = 1;
  while (mode < 4) {
    double acc[NBLK][2];
#pragma unroll
    for (int b = 0; b < NBLK; ++b) acc[b][0] = acc[b][1] = 0.0;
    for (int t = warp * 32; t < JP; t += 256) gram_tile_dmma<SP, double, LD>(Z + t * LD, acc);
    gram_store<SP>(acc, wpart, G);
    __syncthreads();
    if (warp == 0) {
      if (mode == 1) {
        double tr = (tid < s) ? G[tid * SP + tid] : 0.0;
        for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
        const double shift = 11.0 * ((double)J * s + (double)s * (s + 1)) * 1.1102230246251565e-16 * tr;
        if (tid < s) G[tid * SP + tid] += shift;
        __syncwarp();
      }
      const double floor_rel = mode == 3 ? 1e-3 : 0.0;
      const bool okk = chol_reg<SP>(G, SP, L, SP, dinv, s, floor_rel);
      if (tid == 0) ok_s = okk;
    }
    __syncthreads();
    if (!ok_s) {
      chol = false;
      break;
    }
    for (int r = tid; r < J; r += 256) {
      double q[SP];
#pragma unroll
      for (int i = 0; i < SP; ++i) {
        if (i < s) {
          double t = Z[r * LD + i];
#pragma unroll
          for (int m = 0; m < i; ++m) t = fma(-L[i * SP + m], q[m], t);
          q[i] = t * dinv[i];
        }
      }
#pragma unroll
      for (int i = 0; i < SP; ++i)
        if (i < s) Z[r * LD + i] = q[i];
    }
    __syncthreads();
    ++mode;
  }
  if (!chol) {
    for (int i = tid; i < J * SP; i += 256) {
      const int r = i / SP, c = i - r * SP;
      Z[r * LD + c] = c < s ? Y2[(size_t)r * s + c] : 0.0;
    }
    __syncthreads();
    cgs2_smem(Z, J, LD, s, h, red);
  }
  for (int i = tid; i < J * s; i += 256) Y2[i] = Z[(i / s) * LD + i % s];
}

template <int SP>
bool orth2_t(double* Y2, int64_t J, int s, cudaStream_t st) {
  constexpr int NBLK = GramBlocks<SP>::NBLK;
  const int JP = (int)((J + 31) & ~31);
  const size_t bytes = ((size_t)JP * (SP + 1) + 8 * NBLK * 64 + 2 * SP * SP + SP) * 8;
  if (bytes > 200 * 1024) return false;
  if (cudaFuncSetAttribute(orth2_cholqr_kernel<SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  orth2_cholqr_kernel<SP><<<1, 256, bytes, st>>>(Y2, (int)J, s);
  return true;
}

bool run_orth2(double* Y2, int64_t J, int s, cudaStream_t st) {
  if (s <= 8) return orth2_t<8>(Y2, J, s, st);
  if (s <= 16) return orth2_t<16>(Y2, J, s, st);
  if (s <= 24) return orth2_t<24>(Y2, J, s, st);
  if (s <= 32) return orth2_t<32>(Y2, J, s, st);
  return false;
}

// eig of the s x s Gram BB by warp 0 in registers (s <= 32); the block
// Jacobi below only when it declines (a zero eigenvalue / no convergence)
DP2_DEV bool eig_reg_any(double* A, int s, double* U) {
  if (s <= 8) return eig_sym_reg<8>(A, s, U, s, s);
  if (s <= 16) return eig_sym_reg<16>(A, s, U, s, s);
  if (s <= 24) return eig_sym_reg<24>(A, s, U, s, s);
  if (s <= 32) return eig_sym_reg<32>(A, s, U, s, s);
  return false;
}

// single block: eig(BB) -> E, D = Q2 U_R with the sign rule, Uf = U_R * sign / E
__global__ void __launch_bounds__(256) stage2_final_kernel(double* BB, int s, const double* Q2, int64_t J,
                                                            int R, double* D, double* E, double* Uf,
                                                            double* Ubuf, int64_t* status, int eig_smem) {
  __shared__ double cs[3 * 80];
  __shared__ int flag;
  __shared__ int perm[160];
  __shared__ double babs[256];
  __shared__ int64_t brow[256];
  __shared__ int bneg[256];
  __shared__ double sgn[64];
  __shared__ double ev[64];
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ int reg_ok;
  if (tid < 32) {
    const bool okk = eig_reg_any(BB, s, Ubuf);
    if (tid == 0) reg_ok = okk;
  }
  __syncthreads();
  if (!reg_ok) {
    // block Jacobi on shared-memory copies (ld s + 1) when they fit (s2 <= ~110)
    extern __shared__ __align__(16) double esm[];
    const bool in_sm = (size_t)2 * s * (s + 1) * 8 <= (size_t)eig_smem;
    double* A = in_sm ? esm : BB;
    double* U = in_sm ? esm + (size_t)s * (s + 1) : Ubuf;
    const int la = in_sm ? s + 1 : s;
    if (in_sm) {
      for (int e = tid; e < s * s; e += nt) A[(e / s) * la + e % s] = BB[e];
      __syncthreads();
    }
    const int sw = jacobi_eig_block(A, la, U, la, s, cs, &flag);
    if (sw > 40 && tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
    if (in_sm) {
      for (int e = tid; e < s * s; e += nt) {
        BB[e] = A[(e / s) * la + e % s];
        Ubuf[e] = U[(e / s) * la + e % s];
      }
      __syncthreads();
    }
  }
  sort_desc_perm(BB, s, s, perm);
  for (int r = tid; r < R; r += nt) {
    const double mu = BB[perm[r] * s + perm[r]];
    ev[r] = mu > 0.0 ? sqrt(mu) : 0.0;
    E[r] = ev[r];
  }
  __syncthreads();
  // D = Q2 U[:, perm[:R]]
  for (int64_t e = tid; e < J * R; e += nt) {
    const int64_t j = e / R;
    const int r = (int)(e % R);
    double acc = 0.0;
    for (int c = 0; c < s; ++c) acc = fma(Q2[j * s + c], Ubuf[c * s + perm[r]], acc);
    D[e] = acc;
  }
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    double ba = -1.0;
    int64_t br = INT64_MAX;
    int bn = 0;
    for (int64_t j = tid; j < J; j += nt) {
      const double v = D[j * R + r], a = fabs(v);
      if (a > ba) { ba = a; br = j; bn = v < 0.0; }
    }
    babs[tid] = ba;
    brow[tid] = br;
    bneg[tid] = bn;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (tid < o) {
        const double va = babs[tid], vb = babs[tid + o];
        const int64_t ra = brow[tid], rb = brow[tid + o];
        if (vb > va || (vb == va && rb < ra)) { babs[tid] = vb; brow[tid] = rb; bneg[tid] = bneg[tid + o]; }
      }
      __syncthreads();
    }
    if (tid == 0) sgn[r] = bneg[0] ? -1.0 : 1.0;
    __syncthreads();
  }
  for (int64_t e = tid; e < J * R; e += nt) D[e] *= sgn[e % R];
  for (int e = tid; e < s * R; e += nt) {
    const int c = e / R, r = e % R;
    Uf[e] = ev[r] > 0.0 ? (Ubuf[c * s + perm[r]] * sgn[r]) / ev[r] : 0.0;
  }
}

// F[n][r] = sum_c C[n][c] Uf[c][r]
__global__ void f_kernel(const double* C, int64_t N, int s, const double* Uf, int R, double* F) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * R;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / R;
    const int r = (int)(e % R);
    double acc = 0.0;
    for (int c = 0; c < s; ++c) acc = fma(C[n * s + c], Uf[c * R + r], acc);
    F[e] = acc;
  }
}

int gemm_tn_splits(int64_t m, int64_t K, int n);
cudaError_t run_gemm_tn(const double* A, int64_t m, int64_t K, const double* B, int n, double* out,
                        cudaStream_t st, double* parts);

namespace {
// split of the reduction dimension for the split-K products: about two CTAs
// per SM in total, chunks of >= 256
int splits_for(int64_t red, int64_t tiles, int sms) {
  const int64_t want = (2 * (int64_t)sms + tiles - 1) / tiles;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (red + 255) / 256));
}
int64_t chunk_for(int64_t red, int splits) { return ((red + splits - 1) / splits + 3) / 4 * 4; }

struct S2Layout {
  size_t parts, Y, Z, Y2, C, BB, Uf, Ubuf, total;
  int ks_nn, ms_g;
};
S2Layout s2_layout(int64_t J, int64_t KR, int s2, int R) {
  S2Layout L{};
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ng = (s2 + 23) / 24;
  L.ks_nn = splits_for(KR, ((J + 63) / 64) * ng, sms);
  L.ms_g = splits_for(KR, ((s2 + 63) / 64) * ng, sms);
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
  L.parts = take(std::max({(size_t)L.ks_nn * J * s2, (size_t)L.ms_g * s2 * s2,
                           (size_t)gemm_tn_splits(J, KR, s2) * KR * s2}) * 8);
  L.Y = take(J * s2 * 8);
  L.Z = take(KR * s2 * 8);
  L.Y2 = take(J * s2 * 8);
  L.C = take(KR * s2 * 8);
  L.BB = take(s2 * s2 * 8);
  L.Uf = take(s2 * R * 8);
  L.Ubuf = take(s2 * s2 * 8);
  L.total = off;
  return L;
}
}  // namespace

size_t stage2_bytes(int64_t J, int64_t KR, int s2, int R) { return s2_layout(J, KR, s2, R).total; }

// out (K x n) = A^T B for row-major A (m x K) and B (m x n): the tall-skinny
// DMMA product of stage 2 (also the fit's M^T V for the zero-pass fitness).
// The reduction over m is split so that ~4 CTAs per SM keep enough loads of A
// in flight; the splits' partials (in ``parts``, >= ms K n doubles, or written
// straight to ``out`` when ms = 1) are summed in order.
int gemm_tn_splits(int64_t m, int64_t K, int n) {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ctas = ((K + 63) / 64) * ((n + 23) / 24);
  const int64_t want = (4 * (int64_t)sms + ctas - 1) / ctas;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (m + 63) / 64));
}

cudaError_t run_gemm_tn(const double* A, int64_t m, int64_t K, const double* B, int n, double* out,
                        cudaStream_t st, double* parts) {
  const int ms = parts ? gemm_tn_splits(m, K, n) : 1;
  const int64_t mc = ((m + ms - 1) / ms + 3) / 4 * 4;
  const int msr = (int)((m + mc - 1) / mc);
  tn_dmma_kernel<<<dim3((unsigned)((K + 63) / 64), msr, (unsigned)((n + 23) / 24)), 256, 0, st>>>(
      A, K, m, K, B, n, n, mc, msr == 1 ? out : parts);
  if (msr > 1)
    reduce_parts_kernel<<<(unsigned)std::min<int64_t>((K * n + 255) / 256, 4096), 256, 0, st>>>(parts, msr, K * n,
                                                                                                  out);
  return cudaGetLastError();
}

// out (m x n) = A B, A row-major (m x K), B row-major (K x n), for the ALS's
// slice-stack products: split over K for ~4 CTAs per SM (gemm_nn_splits),
// the partials (``parts``, >= splits m n doubles) summed in order.
int gemm_nn_splits(int64_t m, int64_t K, int n) {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ctas = ((m + 63) / 64) * ((n + 23) / 24);
  const int64_t want = (4 * (int64_t)sms + ctas - 1) / ctas;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (K + 63) / 64));
}

cudaError_t run_gemm_nn(const double* A, int64_t m, int64_t K, const double* B, int n, double* out, cudaStream_t st,
                        double* parts) {
  const int ks = parts ? gemm_nn_splits(m, K, n) : 1;
  const int64_t kc = ((K + ks - 1) / ks + 3) / 4 * 4;
  const int ksr = (int)((K + kc - 1) / kc);
  nn_dmma_kernel<<<dim3((unsigned)((m + 63) / 64), ksr, (unsigned)((n + 23) / 24)), 256, 0, st>>>(
      A, K, m, K, B, n, n, kc, ksr == 1 ? out : parts);
  if (ksr > 1)
    reduce_parts_kernel<<<(unsigned)std::min<int64_t>((m * n + 255) / 256, 4096), 256, 0, st>>>(parts, ksr, m * n,
                                                                                                  out);
  return cudaGetLastError();
}

cudaError_t run_stage2(const double* M, int64_t J, int64_t KR, const double* omega2, int s2, int R,
                       double* D, double* E, double* F, char* ws, int64_t* status, cudaStream_t st,
                       int power_iters) {
  const S2Layout L = s2_layout(J, KR, s2, R);
  double* parts = reinterpret_cast<double*>(ws + L.parts);
  double* Y = reinterpret_cast<double*>(ws + L.Y);
  double* Z = reinterpret_cast<double*>(ws + L.Z);
  double* Y2 = reinterpret_cast<double*>(ws + L.Y2);
  double* C = reinterpret_cast<double*>(ws + L.C);
  double* BB = reinterpret_cast<double*>(ws + L.BB);
  double* Uf = reinterpret_cast<double*>(ws + L.Uf);
  double* Ubuf = reinterpret_cast<double*>(ws + L.Ubuf);
  const unsigned ng = (unsigned)((s2 + 23) / 24);
  // out (J x s2) = M B (B: KR x s2): split over KR, ordered reduction
  auto nn = [&](const double* B, double* out) {
    const int64_t kc = chunk_for(KR, L.ks_nn);
    const int ks = (int)((KR + kc - 1) / kc);
    nn_dmma_kernel<<<dim3((unsigned)((J + 63) / 64), ks, ng), 256, 0, st>>>(M, KR, J, KR, B, s2, s2, kc, parts);
    reduce_parts_kernel<<<(unsigned)((J * s2 + 255) / 256), 256, 0, st>>>(parts, ks, J * s2, out);
  };
  // out (KR x s2) = M^T B (B: J x s2): split over J so that ~4 CTAs per SM
  // stream M (a latency-bound read otherwise), ordered reduction
  auto tn = [&](const double* B, double* out) { run_gemm_tn(M, J, KR, B, s2, out, st, parts); };
  // Y2 = (M M^T)^q M Omega2 (P/linalg.py:124-126; no re-orthonormalisation,
  // as the reference), ping-ponging between Y and Y2
  const int q = power_iters < 0 ? 0 : power_iters;
  if (q == 0) {
    nn(omega2, Y2);
  } else {
    nn(omega2, Y);
    for (int it = 0; it < q; ++it) {
      double* src = (it % 2 == 0) ? Y : Y2;
      double* dst = (it % 2 == 0) ? Y2 : Y;
      tn(src, Z);
      nn(Z, dst);
    }
    if (q % 2 == 0) cudaMemcpyAsync(Y2, Y, (size_t)J * s2 * 8, cudaMemcpyDeviceToDevice, st);
  }
  if (!run_orth2(Y2, J, s2, st)) cgs2_cols_kernel<<<1, 256, 0, st>>>(Y2, J, s2, Y);  // Y is dead: column-major copy
  tn(Y2, C);
  // BB = C^T C (s2 x s2): split over the KR rows of C, ordered reduction
  {
    const int64_t mc = chunk_for(KR, L.ms_g);
    const int ms = (int)((KR + mc - 1) / mc);
    tn_dmma_kernel<<<dim3((unsigned)((s2 + 63) / 64), ms, ng), 256, 0, st>>>(C, s2, KR, s2, C, s2, s2, mc, parts);
    reduce_parts_kernel<<<(s2 * s2 + 255) / 256, 256, 0, st>>>(parts, ms, (int64_t)s2 * s2, BB);
  }
  {
    const size_t esm = (size_t)2 * s2 * (s2 + 1) * 8;
    const int eb = esm <= 200 * 1024 ? (int)esm : 0;
    if (eb) {
      const cudaError_t ea = cudaFuncSetAttribute(stage2_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, eb);
      if (ea != cudaSuccess) return ea;
    }
    stage2_final_kernel<<<1, 256, eb, st>>>(BB, s2, Y2, J, R, D, E, Uf, Ubuf, status, eb);
  }
  f_kernel<<<(unsigned)imin64((KR * R + 255) / 256, 4096), 256, 0, st>>>(C, KR, s2, Uf, R, F);
  return cudaGetLastError();
}

}  // namespace dp2
