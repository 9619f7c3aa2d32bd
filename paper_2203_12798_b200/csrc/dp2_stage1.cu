// Stage 1: per-slice randomized SVD of every X_k (P/linalg.py:97-132 as
// driven by P/compress.py:93-105), restated as two streaming passes over the
// packed store plus small per-slice factorizations.
//
//   pass 1  Z_k  = X_k^T (X_k Omega_k)            (sketch_kernel, no Y store)
//   orth    Q_Z  = CGS2(Z_k)                      (range-preserving: range(X Q_Z)
//                                                  = range(X X^T X Omega) = the
//                                                  reference's Y after q = 1)
//   pass 2  Y_k  = X_k Q_Z (stored), C_k^T = X_k^T Y_k
//   factor  G = Y^T Y = W L W^T, T = W L^-1/2 (Q = Y T orthonormal),
//           B B^T = T^T (C C^T) T = U mu U^T,  P = T U_R, S = sqrt(mu_R),
//           V_k = C_k^T P / S                     (= Q^T X's truncated SVD,
//                                                  P/linalg.py:128-129)
//   signs   A_k = Y_k P, largest-|.| entry of each column >= 0, first index
//           on ties (P/linalg.py:62-70); M[:, kR:(k+1)R] = V_k S_k
//           (P/compress.py:108)
//
// Work decomposition: the global row space is cut into equal segments, one
// persistent CTA each; a CTA walks its pieces (segment x slice) tile by tile
// and emits one partial per piece; per-slice reductions then sum the
// partials in piece order, so results are deterministic for a fixed plan.
#include "dp2_common.cuh"
#include "dp2_internal.h"

namespace dp2 {

// ============================================================ sketch pass
struct SketchParams {
  const void* X;
  int64_t ldx;
  int J, sp, lds, njs;
  const double* B;          // K x J x sp (Omega or Q_Z)
  const int32_t* piece_slice;
  const int64_t* piece_row0;
  const int32_t* piece_rows;
  const int32_t* seg_begin;
  double* out_part;         // npieces x J x sp
  double* y_out;            // total_rows x sp or null
  double* xsq_part;         // npieces x njs or null
  double* g_part;           // npieces x sp x sp (G = Y^T Y per piece) or null
  int64_t* status;
};

template <typename T, int TM, int MT, int NT>
__global__ void __launch_bounds__(256, 1) sketch_kernel(SketchParams prm) {
  constexpr int SG = 8 * NT, YP = SG + 2, YS = SG + 1, NW = 8;
  extern __shared__ __align__(16) unsigned char smem[];
  const int LDS = prm.lds, J = prm.J, sp = prm.sp;
  T* xs = reinterpret_cast<T*>(smem);
  const size_t xbytes = (((size_t)2 * TM * LDS * sizeof(T)) + 15) & ~(size_t)15;
  double* ypart = reinterpret_cast<double*>(smem + xbytes);
  double* ys = ypart + NW * TM * YP;
  double* red = ys + TM * YS;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int seg = blockIdx.x, col0 = blockIdx.y * SG, jsplit = blockIdx.z;
  const int jbase = jsplit * 64 * MT;
  const bool stats = (blockIdx.y == 0) && prm.xsq_part != nullptr;
  const int J4 = (J + 3) / 4;
  const int cpr = (int)((J * (int)sizeof(T) + 15) / 16);        // 16B chunks per row
  const int loaded_cols = cpr * 16 / (int)sizeof(T);

  // zero the never-loaded pad columns of both buffers once
  for (int i = tid; i < 2 * TM * LDS; i += blockDim.x)
    if (i % LDS >= loaded_cols) xs[i] = T(0);

  const int pbeg = prm.seg_begin[seg], pend = prm.seg_begin[seg + 1];
  if (pbeg >= pend) return;
  const char* Xb = reinterpret_cast<const char*>(prm.X);

  auto issue = [&](int buf, int p, int t) {
    const int64_t row0 = prm.piece_row0[p] + (int64_t)t * TM;
    const int rows = min(TM, prm.piece_rows[p] - t * TM);
    char* dst = reinterpret_cast<char*>(xs + (size_t)buf * TM * LDS);
    for (int i = tid; i < TM * cpr; i += blockDim.x) {
      const int r = i / cpr, c = i % cpr;
      const bool ok = r < rows;
      const char* src = ok ? Xb + ((row0 + r) * prm.ldx) * (int64_t)sizeof(T) + (int64_t)c * 16 : Xb;
      cp_async16(dst + ((size_t)r * LDS) * sizeof(T) + (size_t)c * 16, src, ok ? 16 : 0);
    }
  };

  int p = pbeg, t = 0, buf = 0;
  issue(0, p, 0);
  cp_async_commit();

  double zacc[MT][NT][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) zacc[a][b][0] = zacc[a][b][1] = 0.0;
  double sq = 0.0;
  int bad = 0;
  constexpr int GPT = (SG * SG + 255) / 256;
  double gacc[GPT];
#pragma unroll
  for (int q = 0; q < GPT; ++q) gacc[q] = 0.0;
  const bool do_g = prm.g_part != nullptr && jsplit == 0;

  while (true) {
    int np = p, ntl = t + 1;
    if (ntl * TM >= prm.piece_rows[p]) { np = p + 1; ntl = 0; }
    const bool has_next = np < pend;
    if (has_next) issue(buf ^ 1, np, ntl);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    const T* X = xs + (size_t)buf * TM * LDS;
    const int ks = prm.piece_slice[p];
    const double* Bm = prm.B + (size_t)ks * J * sp + col0;

    // ---- phase A: Y_t = X_t B (split-K over warps)
    double ya[TM / 8][NT][2];
#pragma unroll
    for (int a = 0; a < TM / 8; ++a)
#pragma unroll
      for (int b = 0; b < NT; ++b) ya[a][b][0] = ya[a][b][1] = 0.0;
    for (int kk = warp; kk < J4; kk += NW) {
      const int kr = kk * 4 + (lane & 3);
      double bf[NT];
#pragma unroll
      for (int b = 0; b < NT; ++b) bf[b] = kr < J ? __ldg(Bm + (size_t)kr * sp + b * 8 + (lane >> 2)) : 0.0;
#pragma unroll
      for (int a = 0; a < TM / 8; ++a) {
        const double av = (double)X[(a * 8 + (lane >> 2)) * LDS + kr];
#pragma unroll
        for (int b = 0; b < NT; ++b) dmma_8x8x4(ya[a][b][0], ya[a][b][1], av, bf[b]);
      }
    }
#pragma unroll
    for (int a = 0; a < TM / 8; ++a)
#pragma unroll
      for (int b = 0; b < NT; ++b) {
        double* dst = ypart + (warp * TM + a * 8 + (lane >> 2)) * YP + b * 8 + 2 * (lane & 3);
        dst[0] = ya[a][b][0];
        dst[1] = ya[a][b][1];
      }
    __syncthreads();
    for (int i = tid; i < TM * SG; i += blockDim.x) {
      const int r = i / SG, c = i % SG;
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += ypart[(w * TM + r) * YP + c];
      ys[r * YS + c] = s;
    }
    __syncthreads();
    const int rows = min(TM, prm.piece_rows[p] - t * TM);
    if (prm.y_out != nullptr && jsplit == 0) {
      const int64_t grow = prm.piece_row0[p] + (int64_t)t * TM;
      for (int i = tid; i < rows * SG; i += blockDim.x) {
        const int r = i / SG, c = i % SG;
        prm.y_out[(grow + r) * sp + col0 + c] = ys[r * YS + c];
      }
    }
    if (do_g) {  // G += Y_t^T Y_t (rows past the piece are zero)
#pragma unroll
      for (int q = 0; q < GPT; ++q) {
        const int e = tid + q * 256;
        if (e < SG * SG) {
          const int a = e / SG, b = e % SG;
          double acc = gacc[q];
          for (int r = 0; r < TM; ++r) acc = fma(ys[r * YS + a], ys[r * YS + b], acc);
          gacc[q] = acc;
        }
      }
    }

    // ---- phase B: Z += X_t^T Y_t (each warp owns MT 8-row blocks of J)
#pragma unroll
    for (int kq = 0; kq < TM / 4; ++kq) {
      const int kr = kq * 4 + (lane & 3);
      double bf[NT];
#pragma unroll
      for (int b = 0; b < NT; ++b) bf[b] = ys[kr * YS + b * 8 + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        const int m = jbase + (warp * MT + a) * 8 + (lane >> 2);
        double av = 0.0;
        if (m < J) {
          av = (double)X[kr * LDS + m];
          if (stats) {
            sq = fma(av, av, sq);
            bad |= !isfinite(av);
          }
        }
#pragma unroll
        for (int b = 0; b < NT; ++b) dmma_8x8x4(zacc[a][b][0], zacc[a][b][1], av, bf[b]);
      }
    }

    if ((t + 1) * TM >= prm.piece_rows[p]) {  // piece complete: flush partial
      if (do_g) {
#pragma unroll
        for (int q = 0; q < GPT; ++q) {
          const int e = tid + q * 256;
          if (e < SG * SG) prm.g_part[(size_t)p * SG * SG + e] = gacc[q];
          gacc[q] = 0.0;
        }
      }
      double* out = prm.out_part + (size_t)p * J * sp + col0;
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        const int m = jbase + (warp * MT + a) * 8 + (lane >> 2);
        if (m < J) {
#pragma unroll
          for (int b = 0; b < NT; ++b) {
            double* d = out + (size_t)m * sp + b * 8 + 2 * (lane & 3);
            d[0] = zacc[a][b][0];
            d[1] = zacc[a][b][1];
          }
        }
#pragma unroll
        for (int b = 0; b < NT; ++b) zacc[a][b][0] = zacc[a][b][1] = 0.0;
      }
      if (stats) {
        const double tot = block_sum(sq, red);
        if (tid == 0) prm.xsq_part[(size_t)p * prm.njs + jsplit] = tot;
        sq = 0.0;
        if (__syncthreads_or(bad) && tid == 0) status_min(prm.status, ST_NONFINITE, ks);
        bad = 0;
      }
    }
    __syncthreads();
    if (!has_next) break;
    p = np;
    t = ntl;
    buf ^= 1;
  }
}

// ============================================================ partial sum + CGS2
// Sum the slice's piece partials (piece order) into Q, then orthonormalise the
// first s_k columns with classical Gram-Schmidt + one reorthogonalisation.
// Exactly-zero columns are replaced by unit vectors (the reference's
// Householder QR likewise returns a full orthonormal Q for a zero sketch).
// Element (r, c) of Q is Q[r * rs + c * cs]: cs = 1 for row-major Q, rs = 1
// (columns contiguous) for coalesced column sweeps.
__device__ void cgs2_columns(double* Q, int64_t rows, int64_t rs, int64_t cs, int ncols, double* h, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int c = 0; c < ncols; ++c) {
    double* qc = Q + c * cs;
    for (int attempt = 0;; ++attempt) {
      if (attempt > 0) {  // replacement unit vector e_{(c + attempt - 1) mod rows}
        const int64_t e = (int64_t)(c + attempt - 1) % rows;
        for (int64_t i = tid; i < rows; i += nt) qc[i * rs] = (i == e) ? 1.0 : 0.0;
        __syncthreads();
      }
      for (int pass = 0; pass < 2; ++pass) {
        for (int i = warp; i < c; i += nw) {
          const double* qi = Q + i * cs;
          double s = 0.0;
          for (int64_t r = lane; r < rows; r += 32) s = fma(qi[r * rs], qc[r * rs], s);
          s = warp_sum(s);
          if (lane == 0) h[i] = s;
        }
        __syncthreads();
        for (int64_t r = tid; r < rows; r += nt) {
          double acc = qc[r * rs];
          for (int i = 0; i < c; ++i) acc = fma(-h[i], Q[r * rs + i * cs], acc);
          qc[r * rs] = acc;
        }
        __syncthreads();
      }
      double part = 0.0;
      for (int64_t r = tid; r < rows; r += nt) part = fma(qc[r * rs], qc[r * rs], part);
      const double nrm2 = block_sum(part, red);
      const bool ok = attempt == 0 ? (nrm2 > 1e-300) : (nrm2 > 0.25);
      if (ok || attempt > rows + 1) {
        const double inv = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
        for (int64_t r = tid; r < rows; r += nt) qc[r * rs] *= inv;
        __syncthreads();
        break;
      }
    }
  }
}

// The CGS2 runs on a column-major copy of the slice's Q (coalesced dot
// products and updates; row-major Q would touch one sector per row) held in
// the slice's first piece partial, which is dead once summed.
__global__ void __launch_bounds__(256) orth_kernel(double* part, const int32_t* slice_piece,
                                                    const int32_t* s_k, int J, int sp, double* Q) {
  __shared__ double h[256];
  __shared__ double red[32];
  const int k = blockIdx.x;
  const int p0 = slice_piece[k], p1 = slice_piece[k + 1];
  const int s = s_k[k];
  double* Qk = Q + (size_t)k * J * sp;
  for (int64_t i = threadIdx.x; i < (int64_t)J * sp; i += blockDim.x) {
    double acc = 0.0;
    for (int p = p0; p < p1; ++p) acc += part[(size_t)p * J * sp + i];
    Qk[i] = acc;
  }
  __syncthreads();
  if (p1 == p0) {  // no piece (empty slice): row-major in place
    cgs2_columns(Qk, J, sp, 1, s, h, red);
    return;
  }
  double* Qc = part + (size_t)p0 * J * sp;  // s x J, column c at Qc + c J
  for (int64_t i = threadIdx.x; i < (int64_t)J * s; i += blockDim.x) {
    const int64_t c = i / J, r = i - c * J;
    Qc[i] = Qk[r * sp + c];
  }
  __syncthreads();
  cgs2_columns(Qc, J, 1, J, s, h, red);
  for (int64_t i = threadIdx.x; i < (int64_t)J * s; i += blockDim.x) {
    const int64_t r = i / s, c = i - r * s;
    Qk[r * sp + c] = Qc[c * J + r];
  }
}

// CGS2 of one tall row-major Q (rows x ncols) through a column-major copy in
// ``scr`` (rows x ncols doubles): the stage-2 orthonormalisation for s2 > 32.
__global__ void __launch_bounds__(256) cgs2_cols_kernel(double* Q, int64_t rows, int ncols, double* scr) {
  __shared__ double h[256];
  __shared__ double red[32];
  for (int64_t i = threadIdx.x; i < rows * ncols; i += blockDim.x) {
    const int64_t c = i / rows, r = i - c * rows;
    scr[i] = Q[r * ncols + c];
  }
  __syncthreads();
  cgs2_columns(scr, rows, 1, rows, ncols, h, red);
  for (int64_t i = threadIdx.x; i < rows * ncols; i += blockDim.x) {
    const int64_t r = i / ncols, c = i - r * ncols;
    Q[i] = scr[c * rows + r];
  }
}


// ============================================================ per-slice factor
// Two s x s work matrices (ld = s + 1) in shared memory when they fit in the
// dynamic allocation (s <= ~105), else in the slice's global scratch
// (3*sp*(sp+1) + 4*sp doubles per slice, which also holds T = W / sqrt(lam)).
struct FactorParams {
  const double* part;       // npieces x J x sp (C^T partials)
  const int32_t* slice_piece;
  const int64_t* row_off;
  const int32_t* s_k;
  const double* y2;         // total_rows x sp
  double* ct;               // K x J x sp  (out: C^T)
  double* Pm;               // K x sp x R
  double* Sv;               // K x R
  double* Vt;               // K x J x R
  int32_t* rank_out;        // K
  double* scr;              // global scratch
  int64_t* status;
  int J, sp, R, smem_bytes;
};

constexpr int kGramRows = 32;   // row tile of the streamed grams
constexpr int kGramBlk = 4;     // upper-triangle 4 x 4 output blocks per thread (s <= 160 at 256 threads)

// dst (s x s, ld) = src^T src over nrows rows of src (row stride lds, first s
// columns), full symmetric.  Rows stream once through ``tile`` (kGramRows x
// s4 doubles); thread t accumulates the upper-triangle 4 x 4 output blocks t,
// t + nt, ... in registers, each summed in row order.
DP2_DEV void gram_cols_cta(const double* src, int64_t nrows, int lds, int s, double* dst, int ld, double* tile) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nb4 = (s + 3) / 4, s4 = nb4 * 4, nbt = nb4 * (nb4 + 1) / 2;
  int bi[kGramBlk], bj[kGramBlk];
#pragma unroll
  for (int m = 0; m < kGramBlk; ++m) {
    const int e = tid + m * nt;
    bi[m] = -1;
    bj[m] = 0;
    if (e < nbt) {
      int a = 0, rem = e;
      while (rem >= nb4 - a) {
        rem -= nb4 - a;
        ++a;
      }
      bi[m] = a;
      bj[m] = a + rem;
    }
  }
  double acc[kGramBlk][16];
#pragma unroll
  for (int m = 0; m < kGramBlk; ++m)
#pragma unroll
    for (int x = 0; x < 16; ++x) acc[m][x] = 0.0;
  for (int64_t r0 = 0; r0 < nrows; r0 += kGramRows) {
    const int rr = (int)(nrows - r0 < kGramRows ? nrows - r0 : kGramRows);
    __syncthreads();
    for (int i = tid; i < kGramRows * s4; i += nt) {
      const int r = i / s4, c = i - r * s4;
      tile[i] = (r < rr && c < s) ? src[(r0 + r) * lds + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < kGramBlk; ++m) {
      if (bi[m] < 0) continue;
      const double* ta = tile + bi[m] * 4;
      const double* tb = tile + bj[m] * 4;
      for (int r = 0; r < rr; ++r) {
        const double2 a01 = *reinterpret_cast<const double2*>(ta + r * s4);
        const double2 a23 = *reinterpret_cast<const double2*>(ta + r * s4 + 2);
        const double2 b01 = *reinterpret_cast<const double2*>(tb + r * s4);
        const double2 b23 = *reinterpret_cast<const double2*>(tb + r * s4 + 2);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[m][x * 4 + y] = fma(av[x], bv[y], acc[m][x * 4 + y]);
      }
    }
  }
#pragma unroll
  for (int m = 0; m < kGramBlk; ++m) {
    if (bi[m] < 0) continue;
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int a = bi[m] * 4 + x, b = bj[m] * 4 + y;
        if (a < s && b < s) {
          dst[a * ld + b] = acc[m][x * 4 + y];
          dst[b * ld + a] = acc[m][x * 4 + y];
        }
      }
  }
  __syncthreads();
}

// Cholesky G = L L^T of the s x s symmetric matrix in A (lower triangle
// overwritten by L), one column per step over the CTA; false (uniformly) when
// a pivot is not above rel_floor * max_i G_ii or not finite.
DP2_DEV bool cta_chol_lower(double* A, int ld, int s, double rel_floor, int* flag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double gmax_s;
  if (tid == 0) {
    double g = 0.0;
    for (int i = 0; i < s; ++i) g = fmax(g, A[i * ld + i]);
    gmax_s = g;
    *flag = g > 0.0 && isfinite(g) ? 0 : 1;
  }
  __syncthreads();
  if (*flag) return false;
  const double floor = rel_floor * gmax_s;
  for (int j = 0; j < s; ++j) {
    if (tid == 0) {
      const double d = A[j * ld + j];
      if (d > floor && isfinite(d)) A[j * ld + j] = sqrt(d);
      else *flag = 1;
    }
    __syncthreads();
    if (*flag) return false;
    const double il = 1.0 / A[j * ld + j];
    for (int i = j + 1 + tid; i < s; i += nt) A[i * ld + j] *= il;
    __syncthreads();
    const int n = s - j - 1;
    for (int e = tid; e < n * n; e += nt) {  // trailing lower triangle
      const int i = j + 1 + e / n, c = j + 1 + e % n;
      if (c <= i) A[i * ld + c] = fma(-A[i * ld + j], A[c * ld + j], A[i * ld + c]);
    }
    __syncthreads();
  }
  return true;
}

// tmp = CC T in place: rows a0 .. a0 + 3 of A (s x s, stride ld) per warp
// pass, read in full before the warp overwrites their first rp columns;
// T (s x rp) is Tg with row stride s.  Covers rp <= 32 MC columns.
template <int MC>
DP2_DEV void cc_times_t(double* A, int ld, const double* Tg, int s, int rp, int warp, int nw, int lane) {
  for (int a0 = warp * 4; a0 < s; a0 += nw * 4) {
    double o[4][MC];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int m = 0; m < MC; ++m) o[x][m] = 0.0;
    for (int b = 0; b < s; ++b) {
      double t[MC];
#pragma unroll
      for (int m = 0; m < MC; ++m) {
        const int c = lane + 32 * m;
        t[m] = c < rp ? Tg[b * s + c] : 0.0;
      }
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const double cab = a0 + x < s ? A[(a0 + x) * ld + b] : 0.0;
#pragma unroll
        for (int m = 0; m < MC; ++m) o[x][m] = fma(cab, t[m], o[x][m]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int m = 0; m < MC; ++m) {
        const int c = lane + 32 * m;
        if (a0 + x < s && c < rp) A[(a0 + x) * ld + c] = o[x][m];
      }
    __syncwarp();
  }
}

__host__ __device__ inline size_t factor_smem_bytes(int s) {
  return (2 * (size_t)s * (s + 1) + (size_t)kGramRows * ((s + 3) / 4 * 4) + 4 * (size_t)s + 8) * 8;
}

__global__ void __launch_bounds__(256) factor_kernel(FactorParams prm) {
  extern __shared__ __align__(16) double fsm[];
  const int k = blockIdx.x, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int J = prm.J, sp = prm.sp, R = prm.R, s = prm.s_k[k];
  const int ld = s + 1;
  const bool in_smem = factor_smem_bytes(s) <= (size_t)prm.smem_bytes;
  double* gscr = prm.scr + (size_t)k * (3 * (size_t)sp * (sp + 1) + 4 * sp);
  double* A = in_smem ? fsm : gscr;
  double* B = A + (size_t)s * ld;
  double* tile = in_smem ? B + (size_t)s * ld : fsm;          // kGramRows x s4
  double* lam = tile + (size_t)kGramRows * ((s + 3) / 4 * 4);  // s
  double* cs = lam + s;                                        // 3*(s/2+1)
  double* Tg = gscr + 2 * (size_t)sp * (sp + 1);               // s x s (ld = s), global: T = W[:, perm] / sqrt(lam)
  __shared__ int perm[256];  // s <= sp <= 256 (dp2_stage1)
  __shared__ int flag;
  __shared__ double Sloc[64];

  // 1. C^T = sum of piece partials
  const int p0 = prm.slice_piece[k], p1 = prm.slice_piece[k + 1];
  double* Ct = prm.ct + (size_t)k * J * sp;
  for (int64_t i = tid; i < (int64_t)J * sp; i += nt) {
    double acc = 0.0;
    for (int p = p0; p < p1; ++p) acc += prm.part[(size_t)p * J * sp + i];
    Ct[i] = acc;
  }
  __syncthreads();
  // 2. G = Y^T Y over the slice rows (A); 3. eig(G) -> eigenvectors (B), lambda (descending)
  gram_cols_cta(prm.y2 + prm.row_off[k] * sp, prm.row_off[k + 1] - prm.row_off[k], sp, s, A, ld, tile);
  int rp = 0, sw = 0;
  // 3. whitening T (Y T orthonormal): T = L^-T from the Cholesky factor of G
  //    (the small-sketch path's relative pivot floor 1e-13, s sequential
  //    column steps over the CTA); a rank-deficient sketch (pivot below the
  //    floor) takes the eigen basis of G instead, dropping lambda <=
  //    1e-13 lambda_max: T = W[:, perm] / sqrt(lambda)
  if (cta_chol_lower(A, ld, s, 1e-13, &flag)) {
    rp = s;
    for (int c = tid; c < s; c += nt)  // L^-1 by forward substitution, column c per thread, into B
      for (int i = 0; i < s; ++i) {
        if (i < c) {
          B[i * ld + c] = 0.0;
          continue;
        }
        double t = i == c ? 1.0 : 0.0;
        for (int m = c; m < i; ++m) t = fma(-A[i * ld + m], B[m * ld + c], t);
        B[i * ld + c] = t / A[i * ld + i];
      }
    __syncthreads();
    for (int i = tid; i < s * s; i += nt) {
      const int a = i / s, c = i - a * s;
      Tg[a * s + c] = B[c * ld + a];
    }
    __syncthreads();
  } else {
    gram_cols_cta(prm.y2 + prm.row_off[k] * sp, prm.row_off[k + 1] - prm.row_off[k], sp, s, A, ld, tile);
    sw = jacobi_eig_block(A, ld, B, ld, s, cs, &flag);
    if (sw > 40 && tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(prm.status + ST_SWEEPCAP), 1ull);
    sort_desc_perm(A, ld, s, perm);
    for (int i = tid; i < s; i += nt) lam[i] = A[perm[i] * ld + perm[i]];
    __syncthreads();
    const double lmax = lam[0] > 0.0 ? lam[0] : 0.0;
    for (int i = 0; i < s; ++i) rp += (lam[i] > 1e-13 * lmax && lam[i] > 0.0) ? 1 : 0;
    for (int i = tid; i < s * rp; i += nt) {
      const int a = i / rp, c = i - a * rp;
      Tg[a * s + c] = B[a * ld + perm[c]] / sqrt(lam[c]);
    }
    __syncthreads();
  }
  // 4. CC = C C^T over J (A), then tmp = CC T in place (A[:, :rp]), 4 rows per
  // warp pass; a lane holds columns lane + 32 m, m < MC (MC = 8 when rp > 128)
  gram_cols_cta(Ct, J, sp, s, A, ld, tile);
  if (rp <= 128) cc_times_t<4>(A, ld, Tg, s, rp, warp, nw, lane);
  else cc_times_t<8>(A, ld, Tg, s, rp, warp, nw, lane);
  __syncthreads();
  // Bg = T^T tmp (rp x rp, B), symmetrised
  for (int i = tid; i < rp * rp; i += nt) {
    const int a = i / rp, c = i - a * rp;
    double acc = 0.0;
    for (int b = 0; b < s; ++b) acc = fma(Tg[b * s + a], A[b * ld + c], acc);
    B[a * ld + c] = acc;
  }
  __syncthreads();
  for (int i = tid; i < rp * rp; i += nt) {
    const int a = i / rp, c = i - a * rp;
    if (a < c) {
      const double m = 0.5 * (B[a * ld + c] + B[c * ld + a]);
      B[a * ld + c] = m;
      B[c * ld + a] = m;
    }
  }
  __syncthreads();
  sw = jacobi_eig_block(B, ld, A, ld, rp, cs, &flag);
  if (sw > 40 && tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(prm.status + ST_SWEEPCAP), 1ull);
  sort_desc_perm(B, ld, rp, perm);
  // 5. P = T U[:, :R], S = sqrt(mu)
  double* Pk = prm.Pm + (size_t)k * sp * R;
  double* Sk = prm.Sv + (size_t)k * R;
  for (int i = tid; i < sp * R; i += nt) {
    const int a = i / R, r = i - a * R;
    double acc = 0.0;
    if (a < s && r < rp) {
      const int col = perm[r];
      for (int b = 0; b < rp; ++b) acc = fma(Tg[a * s + b], A[b * ld + col], acc);
    }
    Pk[a * R + r] = acc;
  }
  for (int r = tid; r < R; r += nt) {
    const double mu = r < rp ? B[perm[r] * ld + perm[r]] : 0.0;
    Sloc[r] = mu > 0.0 ? sqrt(mu) : 0.0;
    Sk[r] = Sloc[r];
  }
  __syncthreads();
  // 6. V = C^T P / S
  double* Vk = prm.Vt + (size_t)k * J * R;
  for (int64_t i = tid; i < (int64_t)J * R; i += nt) {
    const int64_t j = i / R;
    const int r = (int)(i % R);
    double acc = 0.0;
    for (int a = 0; a < s; ++a) acc = fma(Ct[j * sp + a], Pk[a * R + r], acc);
    Vk[i] = Sloc[r] > 0.0 ? acc / Sloc[r] : 0.0;
  }
  int rk = 0;
  for (int r = 0; r < R; ++r) rk += Sloc[r] > 0.0 ? 1 : 0;
  if (tid == 0) {
    prm.rank_out[k] = rk;
    if (rk < R) status_min(prm.status, ST_RANKDEF, k);
  }
}

// ============================================================ signs and A
// a_r(i) = sum_c y2[i][c] P[c][r] (large-sketch path: arows_kernel)
struct RowsParams {
  const double* y2;
  const int64_t* row_off;
  const int32_t* piece_slice;
  const int64_t* piece_row0;
  const int32_t* piece_rows;
  const int32_t* s_k;
  const double* Pm;     // K x sp x R
  int sp, R;
  double* cand_abs;     // npieces x R
  int64_t* cand_row;    // npieces x R
  int32_t* cand_neg;    // npieces x R
  double* A;            // total_rows x R
};

// Combine candidates, fold the signs into P, write M's column block k.
__global__ void __launch_bounds__(128) signs_kernel(const int32_t* slice_piece, const double* cand_abs,
                                                     const int64_t* cand_row, const int32_t* cand_neg,
                                                     double* Pm, const double* Sv, const double* Vt,
                                                     int K, int J, int sp, int R, double* M,
                                                     double* sgn_out = nullptr) {
  const int k = blockIdx.x, tid = threadIdx.x;
  __shared__ double sgn[64];
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
    if (sgn_out) sgn_out[(size_t)k * R + r] = sgn[r];
  }
  __syncthreads();
  double* Pk = Pm + (size_t)k * sp * R;
  for (int i = tid; i < sp * R; i += blockDim.x) Pk[i] *= sgn[i % R];
  const double* Vk = Vt + (size_t)k * J * R;
  const double* Sk = Sv + (size_t)k * R;
  const int64_t KR = (int64_t)K * R;
  for (int64_t i = tid; i < (int64_t)J * R; i += blockDim.x) {
    const int64_t j = i / R;
    const int r = (int)(i % R);
    M[j * KR + (int64_t)k * R + r] = (sgn[r] * Vk[i]) * Sk[r];
  }
}

// Large-sketch path, one pass over Y: A = Y P (unsigned) for the rows of
// piece p and the piece's argmax candidates of |A[:, c]| (first row on ties).
// One warp per row (rows r0 + w, r0 + w + 8, ...: ascending per warp), lanes
// over the columns c = lane, lane + 32; the y row is read coalesced into
// registers and broadcast by shuffle, P (s x R) is staged in shared memory;
// accumulation over a ascending.  The stored A is the exact array the
// candidates saw (the signs are applied after, apply_signs_kernel).
__global__ void __launch_bounds__(256) arows_kernel(RowsParams prm) {
  extern __shared__ __align__(16) double Ps[];  // s x R
  __shared__ double wabs[8][64];
  __shared__ int64_t wrow[8][64];
  __shared__ int wneg[8][64];
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, R = prm.R, sp = prm.sp;
  const int k = prm.piece_slice[p], s = prm.s_k[k];
  const double* Pk = prm.Pm + (size_t)k * sp * R;
  for (int i = tid; i < s * R; i += blockDim.x) Ps[i] = Pk[i];
  __syncthreads();
  const int64_t r0 = prm.piece_row0[p], nr = prm.piece_rows[p];
  const int64_t base = prm.row_off[k];
  const int c0 = lane, c1 = lane + 32;
  double best0 = -1.0, best1 = -1.0;
  int64_t brw0 = INT64_MAX, brw1 = INT64_MAX;
  int bng0 = 0, bng1 = 0;
  for (int64_t i = r0 + warp; i < r0 + nr; i += 8) {
    const double* y = prm.y2 + i * sp;
    double yv[8];  // s <= 256 (dp2_stage1's sketch-width bound)
#pragma unroll
    for (int t = 0; t < 8; ++t) yv[t] = lane + 32 * t < s ? __ldg(y + lane + 32 * t) : 0.0;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (32 * t >= s) break;
      const int n = min(32, s - 32 * t);
      for (int q = 0; q < n; ++q) {
        const double ya = __shfl_sync(0xffffffffu, yv[t], q);
        const double* pr = Ps + (32 * t + q) * R;
        if (c0 < R) a0 = fma(ya, pr[c0], a0);
        if (c1 < R) a1 = fma(ya, pr[c1], a1);
      }
    }
    double* arow = prm.A + i * R;
    if (c0 < R) {
      arow[c0] = a0;
      const double v = fabs(a0);
      if (v > best0) { best0 = v; brw0 = i - base; bng0 = a0 < 0.0; }
    }
    if (c1 < R) {
      arow[c1] = a1;
      const double v = fabs(a1);
      if (v > best1) { best1 = v; brw1 = i - base; bng1 = a1 < 0.0; }
    }
  }
  wabs[warp][c0] = best0;
  wrow[warp][c0] = brw0;
  wneg[warp][c0] = bng0;
  wabs[warp][c1] = best1;
  wrow[warp][c1] = brw1;
  wneg[warp][c1] = bng1;
  __syncthreads();
  if (tid < R) {  // across the warps: larger |a|, then lower row
    double v = -1.0;
    int64_t rw = INT64_MAX;
    int ng = 0;
    for (int w = 0; w < 8; ++w)
      if (wabs[w][tid] > v || (wabs[w][tid] == v && wrow[w][tid] < rw)) {
        v = wabs[w][tid];
        rw = wrow[w][tid];
        ng = wneg[w][tid];
      }
    prm.cand_abs[(size_t)p * R + tid] = v;
    prm.cand_row[(size_t)p * R + tid] = rw;
    prm.cand_neg[(size_t)p * R + tid] = ng;
  }
}

// A[i][c] *= sgn[k][c] for the rows of piece p (coalesced rows)
__global__ void __launch_bounds__(256) apply_signs_kernel(RowsParams prm, const double* sgn) {
  const int p = blockIdx.x, R = prm.R;
  const int k = prm.piece_slice[p];
  const int64_t r0 = prm.piece_row0[p], n = (int64_t)prm.piece_rows[p] * R;
  double* a = prm.A + r0 * R;
  const double* sg = sgn + (size_t)k * R;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) a[e] *= sg[e % R];
}

__global__ void fill_kernel(double* x, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// Rank-deficient slices: complete A_k's trailing columns to an orthonormal set.
__global__ void __launch_bounds__(256) complete_kernel(const int64_t* row_off, const int32_t* rank_out,
                                                        int R, double* A) {
  __shared__ double h[256];
  __shared__ double red[32];
  const int k = blockIdx.x;
  const int rk = rank_out[k];
  if (rk >= R) return;
  const int64_t rows = row_off[k + 1] - row_off[k];
  double* Ak = A + row_off[k] * R;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int c = rk; c < R; ++c) {
    for (int64_t e = 0; e < rows; ++e) {
      for (int64_t i = tid; i < rows; i += nt) Ak[i * R + c] = (i == (e + c) % rows) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int i = warp; i < c; i += nw) {
          double sacc = 0.0;
          for (int64_t r = lane; r < rows; r += 32) sacc = fma(Ak[r * R + i], Ak[r * R + c], sacc);
          sacc = warp_sum(sacc);
          if (lane == 0) h[i] = sacc;
        }
        __syncthreads();
        for (int64_t r = tid; r < rows; r += nt) {
          double acc = Ak[r * R + c];
          for (int i = 0; i < c; ++i) acc = fma(-h[i], Ak[r * R + i], acc);
          Ak[r * R + c] = acc;
        }
        __syncthreads();
      }
      double part = 0.0;
      for (int64_t r = tid; r < rows; r += nt) part = fma(Ak[r * R + c], Ak[r * R + c], part);
      const double n2 = block_sum(part, red);
      if (n2 > 0.25) {
        const double inv = 1.0 / sqrt(n2);
        for (int64_t r = tid; r < rows; r += nt) Ak[r * R + c] *= inv;
        __syncthreads();
        break;
      }
    }
  }
}

// ============================================================ host side
namespace {

int pick_lds(int J, int elem) {
  const int J4 = ((J + 3) / 4) * 4;
  int lds = J4;
  if (elem == 8) {
    while (lds % 16 != 4) ++lds;
  } else {
    while (lds % 32 != 8) ++lds;
  }
  return lds;
}

template <typename T, int TM, int MT, int NT>
cudaError_t launch_sketch(const SketchParams& prm, int nseg, int ng, int njs, cudaStream_t st) {
  constexpr int SG = 8 * NT;
  const size_t xbytes = (((size_t)2 * TM * prm.lds * sizeof(T)) + 15) & ~(size_t)15;
  const size_t smem = xbytes + (size_t)(8 * TM * (SG + 2) + TM * (SG + 1) + 32) * sizeof(double);
  auto kern = sketch_kernel<T, TM, MT, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(nseg, ng, njs), 256, smem, st>>>(prm);
  return cudaGetLastError();
}

template <typename T, int TM, int MT>
cudaError_t dispatch_nt(const SketchParams& prm, int nt, int nseg, int ng, int njs, cudaStream_t st) {
  switch (nt) {
    case 1: return launch_sketch<T, TM, MT, 1>(prm, nseg, ng, njs, st);
    case 2: return launch_sketch<T, TM, MT, 2>(prm, nseg, ng, njs, st);
    case 3: return launch_sketch<T, TM, MT, 3>(prm, nseg, ng, njs, st);
    default: return launch_sketch<T, TM, MT, 4>(prm, nseg, ng, njs, st);
  }
}

template <typename T, int TM>
cudaError_t dispatch_mt(const SketchParams& prm, int mt, int nt, int nseg, int ng, int njs, cudaStream_t st) {
  switch (mt) {
    case 1: return dispatch_nt<T, TM, 1>(prm, nt, nseg, ng, njs, st);
    case 2: return dispatch_nt<T, TM, 2>(prm, nt, nseg, ng, njs, st);
    case 4: return dispatch_nt<T, TM, 4>(prm, nt, nseg, ng, njs, st);
    default: return dispatch_nt<T, TM, 8>(prm, nt, nseg, ng, njs, st);
  }
}

}  // namespace

// Smem budget per CTA for the X tiles (both buffers).
static constexpr size_t kXTileBudget = 150 * 1024;

// The generic streaming pass (per-tile DMMA, B from L2 each k-step: no
// J-sized shared-memory image): fp64 storage outside the warp-specialised
// pass's shapes, and fp32 storage whose B image does not fit the FFMA pass
// (J above ~1300) -- fp64 products on the exactly upcast values.
cudaError_t run_sketch_generic(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                               double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part) {
  const int J = (int)st->J;
  const int elem = st->dtype == DP2_F64 ? 8 : 4;
  SketchParams prm{};
  prm.X = st->X;
  prm.ldx = st->ldx;
  prm.J = J;
  prm.sp = sp;
  prm.lds = pick_lds(J, elem);
  prm.B = B;
  prm.piece_slice = st->piece_slice;
  prm.piece_row0 = st->piece_row0;
  prm.piece_rows = st->piece_rows;
  prm.seg_begin = st->seg_begin;
  prm.out_part = out_part;
  prm.y_out = y_out;
  prm.xsq_part = xsq_part;
  prm.g_part = sp <= 32 ? g_part : nullptr;
  prm.status = status;
  const int nt = sp >= 32 ? 4 : sp / 8;
  const int ng = sp >= 32 ? sp / 32 : 1;
  int mt = 1;
  while (mt < 8 && 64 * mt < J) mt *= 2;
  const int njs = (J + 64 * mt - 1) / (64 * mt);
  prm.njs = njs;
  const int tm = (size_t)2 * 16 * prm.lds * elem <= kXTileBudget ? 16 : 8;
  if ((size_t)2 * tm * prm.lds * elem > 200 * 1024) return cudaErrorInvalidValue;
  const int nseg = st->nseg;
  if (elem == 4)
    return tm == 16 ? dispatch_mt<float, 16>(prm, mt, nt, nseg, ng, njs, stream)
                    : dispatch_mt<float, 8>(prm, mt, nt, nseg, ng, njs, stream);
  return tm == 16 ? dispatch_mt<double, 16>(prm, mt, nt, nseg, ng, njs, stream)
                  : dispatch_mt<double, 8>(prm, mt, nt, nseg, ng, njs, stream);
}

cudaError_t run_sketch(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                       double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part) {
  if (st->dtype == DP2_F32) return run_sketch_f32(st, B, sp, out_part, y_out, xsq_part, status, stream, g_part);
  if (sketch64_eligible(st, sp, xsq_part != nullptr, g_part != nullptr))
    return run_sketch64(st, B, sp, out_part, y_out, status, stream, g_part);
  return run_sketch_generic(st, B, sp, out_part, y_out, xsq_part, status, stream, g_part);
}

int sketch_njs(int J) {
  int mt = 1;
  while (mt < 8 && 64 * mt < J) mt *= 2;
  return (J + 64 * mt - 1) / (64 * mt);
}

Stage1Layout stage1_layout(const dp2_store* st, int sp, int R) {
  Stage1Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t J = st->J, K = st->K, P = st->npieces, N = st->total_rows;
  L.part = take(P * J * sp * 8);
  L.qz = take(K * J * sp * 8);
  L.y2 = take(N * sp * 8);
  L.Pm = take(K * sp * R * 8);
  L.Sv = take(K * R * 8);
  L.Vt = take(K * J * R * 8);
  L.cand_abs = take(P * R * 8);
  L.cand_row = take(P * R * 8);
  L.cand_neg = take(P * R * 4);
  L.xsq = take(P * sketch_njs((int)J) * 8);
  L.gpart = take(P * sp * sp * 8);
  L.CCg = take(K * sp * sp * 8);
  L.Gg = take(K * sp * sp * 8);
  L.sgn = take(K * R * 8);
  L.scr = take(K * (3 * (size_t)sp * (sp + 1) + 4 * sp) * 8);
  L.total = off;
  return L;
}

cudaError_t run_stage1(const dp2_store* st, const double* omega, const int32_t* s_dev, int sp, int R,
                       double* A_out, double* M_out, int32_t* rank_out, char* ws, int64_t* status,
                       float* timing, cudaStream_t stream, double* a_signs, int power_iters) {
  const Stage1Layout L = stage1_layout(st, sp, R);
  double* part = reinterpret_cast<double*>(ws + L.part);
  double* qz = reinterpret_cast<double*>(ws + L.qz);
  double* y2 = reinterpret_cast<double*>(ws + L.y2);
  double* Pm = reinterpret_cast<double*>(ws + L.Pm);
  double* Sv = reinterpret_cast<double*>(ws + L.Sv);
  double* Vt = reinterpret_cast<double*>(ws + L.Vt);
  double* xsq = reinterpret_cast<double*>(ws + L.xsq);
  const int K = (int)st->K, J = (int)st->J;
  cudaEvent_t ev[8];
  if (timing) {
    for (int i = 0; i < 7; ++i) cudaEventCreate(&ev[i]);
    cudaEventRecord(ev[0], stream);
  }
  // the per-piece sums of squares are not consumed by stage 1 (the fitness
  // uses dp2_slice_stats); the tensor-core pass flags non-finite input from Y
  // (the tensor-core and DMMA passes flag non-finite input from Y instead)
  const bool s64 = (st->dtype == DP2_F64 || sketch_engine() == 2) && sketch64_eligible(st, sp, false, false);
  // power iterations (P/linalg.py:124-126): q sketch passes Z = X^T (X B),
  // each followed by B <- orth(Z) (range-preserving; it also keeps the
  // iteration well conditioned), then the final pass Y = X B.  q = 0: the
  // final pass runs on Omega itself (range(X Omega)).
  const int q = power_iters < 0 ? 0 : power_iters;
  cudaError_t e = cudaSuccess;
  if (q > 0) {
    e = run_sketch(st, omega, sp, part, nullptr, (sketch_tc_eligible(st, sp) || s64) ? nullptr : xsq, status,
                   stream);
    if (e != cudaSuccess) return e;
  }
  if (timing) cudaEventRecord(ev[1], stream);
  // orth of pass partials -> qz; then the extra power iterations (q > 1)
  auto orth_and_more = [&](auto&& orth) -> cudaError_t {
    if (q == 0) return cudaMemcpyAsync(qz, omega, (size_t)K * J * sp * 8, cudaMemcpyDeviceToDevice, stream);
    cudaError_t eo = orth();
    for (int it = 1; it < q && eo == cudaSuccess; ++it) {
      eo = run_sketch(st, qz, sp, part, nullptr, nullptr, status, stream);
      if (eo == cudaSuccess) eo = orth();
    }
    return eo;
  };
  if (sp <= 32) {
    double* gpart = reinterpret_cast<double*>(ws + L.gpart);
    double* CCg = reinterpret_cast<double*>(ws + L.CCg);
    double* Gg = reinterpret_cast<double*>(ws + L.Gg);
    double* sgn = reinterpret_cast<double*>(ws + L.sgn);
    // the tensor-core pass leaves G to gram_y_piece_kernel (run_stage1_small; partials into gpart)
    const bool tc = sketch_tc_eligible(st, sp);
    // G = Y^T Y comes from pass 2 unless that pass cannot form it (the
    // tensor-core pass, or the DMMA pass split into column groups at J > 512):
    // then small(1) forms it from the stored Y rows
    const bool dmma_nog = !tc && s64 && !sketch64_eligible(st, sp, false, true);
    double* gp = (tc || dmma_nog) ? nullptr : gpart;
    auto small = [&](int phase) {
      return run_stage1_small(st, s_dev, sp, R, part, part, gp, qz, qz, CCg, Gg, y2, Pm, Sv, sgn,
                              reinterpret_cast<double*>(ws + L.cand_abs), reinterpret_cast<int64_t*>(ws + L.cand_row),
                              reinterpret_cast<int32_t*>(ws + L.cand_neg), A_out, M_out, rank_out, status, phase,
                              stream, tc, gpart, a_signs);
    };
    e = orth_and_more([&]() -> cudaError_t {
      if ((size_t)J * (sp + 1) * 8 <= 200 * 1024) return small(0);
      orth_kernel<<<K, 256, 0, stream>>>(part, st->slice_piece, s_dev, J, sp, qz);
      return cudaGetLastError();
    });
    if (e != cudaSuccess) return e;
    if (timing) cudaEventRecord(ev[2], stream);
    // the tensor-core pass stores Y in fp32: its accumulator precision, half the bytes
    e = tc ? run_sketch_tc(st, qz, sp, part, y2, nullptr, status, stream, nullptr, true)
           : run_sketch(st, qz, sp, part, y2, nullptr, status, stream, gp);
    if (e != cudaSuccess) return e;
    if (timing) cudaEventRecord(ev[3], stream);
    e = small(1);
    if (e != cudaSuccess) return e;
    if (timing) cudaEventRecord(ev[4], stream);
    complete_kernel<<<K, 256, 0, stream>>>(st->row_off, rank_out, R, A_out);
    e = cudaGetLastError();
    if (timing) {
      cudaEventRecord(ev[5], stream);
      cudaEventSynchronize(ev[5]);
      cudaEventElapsedTime(&timing[0], ev[0], ev[1]);
      cudaEventElapsedTime(&timing[1], ev[1], ev[2]);
      cudaEventElapsedTime(&timing[2], ev[2], ev[3]);
      cudaEventElapsedTime(&timing[3], ev[3], ev[4]);
      cudaEventElapsedTime(&timing[4], ev[4], ev[5]);
      cudaEventElapsedTime(&timing[5], ev[0], ev[5]);
      for (int i = 0; i < 7; ++i) cudaEventDestroy(ev[i]);
    }
    return e;
  }
  e = orth_and_more([&]() -> cudaError_t {
    orth_kernel<<<K, 256, 0, stream>>>(part, st->slice_piece, s_dev, J, sp, qz);
    return cudaGetLastError();
  });
  if (e != cudaSuccess) return e;
  if (timing) cudaEventRecord(ev[2], stream);
  e = run_sketch(st, qz, sp, part, y2, nullptr, status, stream);
  if (e != cudaSuccess) return e;
  if (timing) cudaEventRecord(ev[3], stream);
  FactorParams fp{};
  fp.part = part;
  fp.slice_piece = st->slice_piece;
  fp.row_off = st->row_off;
  fp.s_k = s_dev;
  fp.y2 = y2;
  fp.ct = qz;
  fp.Pm = Pm;
  fp.Sv = Sv;
  fp.Vt = Vt;
  fp.rank_out = rank_out;
  fp.scr = reinterpret_cast<double*>(ws + L.scr);
  fp.status = status;
  fp.J = J;
  fp.sp = sp;
  fp.R = R;
  // the two work matrices in shared memory for every s up to sp when they fit
  // (s <= ~105), else per slice in the global scratch (the gram tile stays)
  size_t fsm = factor_smem_bytes(sp);
  if (fsm > 210 * 1024) fsm = 210 * 1024;
  fp.smem_bytes = (int)fsm;
  e = cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  if (e != cudaSuccess) return e;
  factor_kernel<<<K, 256, fsm, stream>>>(fp);
  if (timing) cudaEventRecord(ev[4], stream);
  RowsParams rp{};
  rp.y2 = y2;
  rp.row_off = st->row_off;
  rp.piece_slice = st->piece_slice;
  rp.piece_row0 = st->piece_row0;
  rp.piece_rows = st->piece_rows;
  rp.s_k = s_dev;
  rp.Pm = Pm;
  rp.sp = sp;
  rp.R = R;
  rp.cand_abs = reinterpret_cast<double*>(ws + L.cand_abs);
  rp.cand_row = reinterpret_cast<int64_t*>(ws + L.cand_row);
  rp.cand_neg = reinterpret_cast<int32_t*>(ws + L.cand_neg);
  rp.A = A_out;
  const int P = (int)st->npieces;
  const size_t psm = (size_t)sp * R * 8;  // P staged in shared memory (<= 128 x 64 doubles)
  e = cudaFuncSetAttribute(arows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
  if (e != cudaSuccess) return e;
  // one pass over Y: unsigned A + candidates; signs into P, M and sgn; signed A
  double* sgn = reinterpret_cast<double*>(ws + L.sgn);
  arows_kernel<<<P, 256, psm, stream>>>(rp);
  signs_kernel<<<K, 128, 0, stream>>>(st->slice_piece, rp.cand_abs, rp.cand_row, rp.cand_neg, Pm, Sv, Vt,
                                      K, J, sp, R, M_out, sgn);
  apply_signs_kernel<<<P, 256, 0, stream>>>(rp, sgn);
  complete_kernel<<<K, 256, 0, stream>>>(st->row_off, rank_out, R, A_out);
  if (a_signs) fill_kernel<<<(K * R + 255) / 256, 256, 0, stream>>>(a_signs, (int64_t)K * R, 1.0);  // A is signed
  e = cudaGetLastError();
  if (timing) {
    cudaEventRecord(ev[5], stream);
    cudaEventSynchronize(ev[5]);
    cudaEventElapsedTime(&timing[0], ev[0], ev[1]);
    cudaEventElapsedTime(&timing[1], ev[1], ev[2]);
    cudaEventElapsedTime(&timing[2], ev[2], ev[3]);
    cudaEventElapsedTime(&timing[3], ev[3], ev[4]);
    cudaEventElapsedTime(&timing[4], ev[4], ev[5]);
    cudaEventElapsedTime(&timing[5], ev[0], ev[5]);
    for (int i = 0; i < 7; ++i) cudaEventDestroy(ev[i]);
  }
  return e;
}

}  // namespace dp2
