// Stage 2: randomized SVD of the concatenated right parts
// M = [V_1 S_1 | ... | V_K S_K] (J x KR, P/compress.py:108-111), fp64.
//
//   Y  = M Omega2           (J x s2)     nn split-K partials + ordered reduce
//   Z  = M^T Y              (KR x s2)    tn
//   Y2 = M Z                (J x s2)     = the reference's M (M^T M Omega2)
//   Q2 = orth(Y2)                        CholQR2 in one CTA (CGS2 fallback; the reference's np.linalg.qr)
//   C  = M^T Q2             (KR x s2)    B2 = Q2^T M = C^T
//   B2 B2^T = C^T C = U mu U^T           register Jacobi (block Jacobi fallback); E = sqrt(mu_R)
//   D = Q2 U_R (sign rule, P/linalg.py:62-70), F = C U_R / E (same flips)
#include <dlfcn.h>

#include "dp2_common.cuh"
#include "dp2_internal.h"
#include "dp2_small_linalg.cuh"

namespace dp2 {

// ---------------------------------------------------------------- cuBLAS
// The four products with M and the Gram C^T C are plain dense fp64 GEMMs
// (M is J x KR, e.g. 512 x 10^4): cuBLAS DGEMM (fp64 tensor cores) when the
// library can be opened at run time, else the kernels below.  Loaded with
// dlopen so libdpar2 has no link-time dependency on it; cuBLAS results are
// bitwise reproducible on a given GPU.
namespace {
typedef int (*blas_create_t)(void**);
typedef int (*blas_stream_t)(void*, cudaStream_t);
typedef int (*blas_dgemm_t)(void*, int, int, int, int, int, const double*, const double*, int, const double*, int,
                            const double*, double*, int);
struct Blas {
  bool tried = false;
  blas_create_t create = nullptr;
  blas_stream_t stream = nullptr;
  blas_dgemm_t dgemm = nullptr;
  void* handle[64] = {};
};
Blas& blas() {
  static Blas b;
  if (!b.tried) {
    b.tried = true;
    const char* names[] = {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12", "libcublas.so"};
    void* lib = nullptr;
    for (const char* n : names)
      if ((lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (lib) {
      b.create = reinterpret_cast<blas_create_t>(dlsym(lib, "cublasCreate_v2"));
      b.stream = reinterpret_cast<blas_stream_t>(dlsym(lib, "cublasSetStream_v2"));
      b.dgemm = reinterpret_cast<blas_dgemm_t>(dlsym(lib, "cublasDgemm_v2"));
      if (!b.create || !b.stream || !b.dgemm) b.create = nullptr;
    }
  }
  return b;
}
// column-major C (m x n) = op(A) op(B); false when cuBLAS is unavailable
bool dgemm_cm(cudaStream_t st, bool ta, bool tb, int m, int n, int k, const double* A, int lda, const double* B,
              int ldb, double* C, int ldc) {
  Blas& b = blas();
  if (!b.create) return false;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  if (!b.handle[dev] && b.create(&b.handle[dev]) != 0) {
    b.handle[dev] = nullptr;
    return false;
  }
  if (b.stream(b.handle[dev], st) != 0) return false;
  const double one = 1.0, zero = 0.0;
  return b.dgemm(b.handle[dev], ta ? 1 : 0, tb ? 1 : 0, m, n, k, &one, A, lda, B, ldb, &zero, C, ldc) == 0;
}
}  // namespace

bool stage2_uses_blas() { return blas().create != nullptr; }

constexpr int kChunk = 1024;  // split-K chunk of the KR dimension

// out_part[chunk][i][c] = sum_{n in chunk} A[i][n] * B[n][c],  c in [32g, 32g+32) & < sb
__global__ void __launch_bounds__(256) nn_partial_kernel(const double* A, int64_t lda, int64_t N,
                                                          const double* B, int ldb, int sb,
                                                          double* out_part, int64_t m) {
  __shared__ double red[32];
  const int64_t i = blockIdx.x;
  const int chunk = blockIdx.y, g = blockIdx.z;
  const int64_t n0 = (int64_t)chunk * kChunk, n1 = imin64(N, n0 + kChunk);
  const int c0 = g * 32, cw = min(32, sb - c0);
  double acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.0;
  for (int64_t n = n0 + threadIdx.x; n < n1; n += blockDim.x) {
    const double a = A[i * lda + n];
    const double* b = B + n * ldb + c0;
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c < cw) acc[c] = fma(a, b[c], acc[c]);
  }
  for (int c = 0; c < cw; ++c) {
    const double s = block_sum(acc[c], red);
    if (threadIdx.x == 0) out_part[((size_t)chunk * m + i) * sb + c0 + c] = s;
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

// out[n][c] = sum_i A[i][n] * B[i][c]   (A m x N row-major, B m x sb), c group g
__global__ void __launch_bounds__(256) tn_kernel(const double* A, int64_t lda, int64_t m, int64_t N,
                                                  const double* B, int ldb, int sb, double* out,
                                                  int ldo) {
  __shared__ double bt[32 * 32];
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c0 = blockIdx.y * 32, cw = min(32, sb - c0);
  double acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.0;
  for (int64_t i0 = 0; i0 < m; i0 += 32) {
    const int ir = (int)imin64(32, m - i0);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
      const int r = e / 32, c = e % 32;
      bt[e] = (r < ir && c < cw) ? B[(i0 + r) * ldb + c0 + c] : 0.0;
    }
    __syncthreads();
    if (n < N) {
      for (int r = 0; r < ir; ++r) {
        const double a = A[(i0 + r) * lda + n];
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = fma(a, bt[r * 32 + c], acc[c]);
      }
    }
  }
  if (n < N)
    for (int c = 0; c < cw; ++c) out[n * ldo + c0 + c] = acc[c];
}

// partial Gram over row chunks: part[chunk][a][b] = sum_{n in chunk} C[n][a] C[n][b]
__global__ void __launch_bounds__(256) gram_partial_kernel(const double* C, int64_t N, int ld, int s,
                                                            double* part) {
  __shared__ double tile[1056];
  const int chunk = blockIdx.x;
  const int64_t n0 = (int64_t)chunk * kChunk, n1 = imin64(N, n0 + kChunk);
  const int ntri = s * (s + 1) / 2;
  const int trows = max(1, 1056 / s);
  for (int e0 = 0; e0 < ntri; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    int a = 0, b = 0;
    if (e < ntri) {
      int rem = e;
      while (rem >= s - a) { rem -= s - a; ++a; }
      b = a + rem;
    }
    double acc = 0.0;
    for (int64_t r0 = n0; r0 < n1; r0 += trows) {
      const int rr = (int)imin64(trows, n1 - r0);
      __syncthreads();
      for (int i = threadIdx.x; i < rr * s; i += blockDim.x) tile[i] = C[(r0 + i / s) * ld + (i % s)];
      __syncthreads();
      if (e < ntri)
        for (int r = 0; r < rr; ++r) acc = fma(tile[r * s + a], tile[r * s + b], acc);
    }
    if (e < ntri) {
      part[(size_t)chunk * s * s + a * s + b] = acc;
      part[(size_t)chunk * s * s + b * s + a] = acc;
    }
  }
}

// single block: eig(BB) -> E, D = Q2 U_R with the sign rule, Uf = U_R * sign / E
// Q2 = orth(Y2) (J x s, row-major, in place), one CTA: the J x SP slab in
// shared memory, CholQR twice (G = Y^T Y on DMMA, register Cholesky, row
// substitution) -- orthonormal to rounding for kappa(Y2) below ~1e6 (first
// pivot floor 1e-12); otherwise CGS2 with re-randomisation, like cgs2_kernel.
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

__global__ void __launch_bounds__(256) stage2_final_kernel(double* BB, int s, const double* Q2, int64_t J,
                                                            int R, double* D, double* E, double* Uf,
                                                            double* Ubuf, int64_t* status) {
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
    const int sw = jacobi_eig_block(BB, s, Ubuf, s, s, cs, &flag);
    if (sw > 40 && tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
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

namespace {
struct S2Layout {
  size_t parts, Y, Z, Y2, C, bbp, BB, Uf, Ubuf, total;
};
S2Layout s2_layout(int64_t J, int64_t KR, int s2, int R) {
  S2Layout L{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
  const size_t nch = (KR + kChunk - 1) / kChunk;
  L.parts = take(nch * J * s2 * 8);
  L.Y = take(J * s2 * 8);
  L.Z = take(KR * s2 * 8);
  L.Y2 = take(J * s2 * 8);
  L.C = take(KR * s2 * 8);
  L.bbp = take(nch * s2 * s2 * 8);
  L.BB = take(s2 * s2 * 8);
  L.Uf = take(s2 * R * 8);
  L.Ubuf = take(s2 * s2 * 8);
  L.total = off;
  return L;
}
}  // namespace

size_t stage2_bytes(int64_t J, int64_t KR, int s2, int R) { return s2_layout(J, KR, s2, R).total; }

cudaError_t run_stage2(const double* M, int64_t J, int64_t KR, const double* omega2, int s2, int R,
                       double* D, double* E, double* F, char* ws, int64_t* status, cudaStream_t st) {
  const S2Layout L = s2_layout(J, KR, s2, R);
  double* parts = reinterpret_cast<double*>(ws + L.parts);
  double* Y = reinterpret_cast<double*>(ws + L.Y);
  double* Z = reinterpret_cast<double*>(ws + L.Z);
  double* Y2 = reinterpret_cast<double*>(ws + L.Y2);
  double* C = reinterpret_cast<double*>(ws + L.C);
  double* bbp = reinterpret_cast<double*>(ws + L.bbp);
  double* BB = reinterpret_cast<double*>(ws + L.BB);
  double* Uf = reinterpret_cast<double*>(ws + L.Uf);
  double* Ubuf = reinterpret_cast<double*>(ws + L.Ubuf);
  const int nch = (int)((KR + kChunk - 1) / kChunk);
  const int ng = (s2 + 31) / 32;
  // row-major M (J x KR) is column-major (KR x J); row-major B (KR x s2) is
  // column-major (s2 x KR): Y = M B  <=>  Y_cm (s2 x J) = B_cm M_cm
  auto nn = [&](const double* B, double* out) {
    if (dgemm_cm(st, false, false, s2, (int)J, (int)KR, B, s2, M, (int)KR, out, s2)) return;
    nn_partial_kernel<<<dim3((unsigned)J, nch, ng), 256, 0, st>>>(M, KR, KR, B, s2, s2, parts, J);
    reduce_parts_kernel<<<(unsigned)((J * s2 + 255) / 256), 256, 0, st>>>(parts, nch, J * s2, out);
  };
  // Z = M^T Y  <=>  Z_cm (s2 x KR) = Y_cm M_cm^T
  auto tn = [&](const double* B, double* out) {
    if (dgemm_cm(st, false, true, s2, (int)KR, (int)J, B, s2, M, (int)KR, out, s2)) return;
    tn_kernel<<<dim3((unsigned)((KR + 255) / 256), ng), 256, 0, st>>>(M, KR, J, KR, B, s2, s2, out, s2);
  };
  nn(omega2, Y);
  tn(Y, Z);
  nn(Z, Y2);
  if (!run_orth2(Y2, J, s2, st)) cgs2_kernel<<<1, 256, 0, st>>>(Y2, J, s2, s2, 0);
  tn(Y2, C);
  // BB = C^T C  <=>  C_cm C_cm^T (symmetric, so layout-neutral)
  if (!dgemm_cm(st, false, true, s2, s2, (int)KR, C, s2, C, s2, BB, s2)) {
    gram_partial_kernel<<<nch, 256, 0, st>>>(C, KR, s2, s2, bbp);
    reduce_parts_kernel<<<(s2 * s2 + 255) / 256, 256, 0, st>>>(bbp, nch, (int64_t)s2 * s2, BB);
  }
  stage2_final_kernel<<<1, 256, 0, st>>>(BB, s2, Y2, J, R, D, E, Uf, Ubuf, status);
  f_kernel<<<(unsigned)imin64((KR * R + 255) / 256, 4096), 256, 0, st>>>(C, KR, s2, Uf, R, F);
  return cudaGetLastError();
}

}  // namespace dp2
