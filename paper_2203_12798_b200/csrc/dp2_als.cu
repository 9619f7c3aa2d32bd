// Compressed-space ALS (P/solver.py:39-190), fp64.
//
// One iteration = 9 stream-ordered, graph-capturable launches:
//   rotate  (warp/slice) T_k = (F_k cc) diag(w_k) H^T; polar Pi_k = Z_k P_k^T by
//           one-sided Jacobi warm-started from the previous iteration's P_k;
//           Theta_k = Pi_k^T F_k; mode-1 and gram(W) partials.  16 < R <= 56:
//           one CTA per slice, polar factor by Newton-Schulz on DMMA R x R
//           matmuls (CTA-parallel Jacobi fallback)
//   reduce  (n/32 CTAs)  ordered sum of the per-CTA mode-1 / gram(W) slots
//   solve_h (1 CTA)      H = G1 pinv(W'W * V'V); column norms -> nh
//   mode2   (warp/slice) sum_k (w_k nh) (Theta_k^T H), gram(W nh) partials
//   reduce  (n/32 CTAs)  the same for the mode-2 slots
//   solve_v (1 CTA)      V = D (E * summed) pinv(...); norms; V'V, cc', pinv3
//   mode3   (warp/slice) G3 row, W_k = G3_k pinv3; L_k = [Theta_k E | -H W_k]
//   metric  (DMMA)       e = ||L N^T||_F^2 with N = [D V] (J x 2R): the
//           reference's sum_k ||Theta_k E D^T - H S_k V^T||^2 as one tall GEMM
//           with a fused sum-of-squares epilogue (the R x J products are never
//           stored)
//   finish  (1 warp)     e = ordered sum of partials, trace, device stop rule
// Partials go to per-CTA slots (warps combined in warp order, slots reduced in
// slot order by a fixed warp tree): deterministic for a given device.  Every
// kernel returns at once when the device stop flag is set, so the whole loop
// is one CUDA graph (P/solver.py:180-184 evaluated on the device).
#include "dp2_common.cuh"
#include "dp2_internal.h"
#include "dp2_als_persist.cuh"
#include <cstdio>
#include <cstdlib>
// #define DP2_ROT_DEBUG 1

namespace dp2 {

// ------------------------------------------------------------ helpers
__global__ void reduce_parts_dev(const double* part, int nparts, int64_t size, double* out) {
  for (int64_t idx = threadIdx.x; idx < size; idx += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < nparts; ++c) acc += part[(size_t)c * size + idx];
    out[idx] = acc;
  }
}

// out = D (E * summed)   (P/solver.py:100)
__global__ void g2_kernel(const double* D, const double* E, const double* summed, int64_t J, int R,
                          double* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= J * R) return;
  const int64_t j = e / R;
  const int r = (int)(e % R);
  double acc = 0.0;
  for (int a = 0; a < R; ++a) acc = fma(D[j * R + a], E[a] * summed[a * R + r], acc);
  out[e] = acc;
}

// Ordered reduction of per-CTA slots, latency-first: warp w handles entries
// w, w+nw, ...; each lane issues its (up to 8) slot loads before summing, the
// 32 lane partials combine by a fixed xor tree.  Deterministic for a given
// nslots.
DP2_DEV void reduce_slots_warp(const double* slots, int nslots, int n, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = warp; e < n; e += nw) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int w = lane + 32 * u;
      v[u] = w < nslots ? slots[(size_t)w * n + e] : 0.0;
    }
    double s = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    for (int w = lane + 256; w < nslots; w += 32) s += slots[(size_t)w * n + e];
    s = warp_sum(s);
    if (lane == 0) out[e] = s;
  }
}

// In-place ordered reduction of nslots per-CTA slots (n doubles each) into
// slot 0, two slot arrays at once (blockIdx.y): CTA x sums entries
// 32x .. 32x+31 (coalesced rows), warp w slots w, w + 8, ... in order, and the
// 8 warp partials combine in warp order -- deterministic, and spread over
// n/32 SMs instead of the single solve CTA.
__global__ void __launch_bounds__(256) reduce_slots_kernel(const int32_t* ctl, double* s0, double* s1, int nslots,
                                                           int n) {
  if (ctl[0]) return;
  double* slots = blockIdx.y ? s1 : s0;
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (e < n) {
    int w = warp;
    for (; w + 24 < nslots; w += 32) {
      const double a = slots[(size_t)w * n + e], b = slots[(size_t)(w + 8) * n + e];
      const double c = slots[(size_t)(w + 16) * n + e], d = slots[(size_t)(w + 24) * n + e];
      acc += (a + b) + (c + d);
    }
    for (; w < nslots; w += 8) acc += slots[(size_t)w * n + e];
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && e < n) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    slots[e] = t;
  }
}

// cc = E * (D^T V) and VtV = V^T V, one warp per entry
DP2_DEV void gram_dv_warps(const double* D, const double* E, const double* V, int64_t J, int R, double* cc,
                           double* VtV, double* Mv, const double* HtH) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = warp; e < R * R; e += nw) {
    const int a = e / R, r = e % R;
    double s1 = 0.0, s2 = 0.0;
    for (int64_t j = lane; j < J; j += 32) {
      const double v = V[j * R + r];
      s1 = fma(D[j * R + a], v, s1);
      s2 = fma(V[j * R + a], v, s2);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      cc[e] = E[a] * s1;
      VtV[e] = s2;
      if (Mv) Mv[e] = s2 * HtH[e];
    }
  }
}

// CTA combine of per-warp smem partials (warp order) into the CTA's slot.
DP2_DEV void combine_warps(const double* wbase, size_t wstride, int nwarps, int n, double* slot) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) s += wbase[w * wstride + e];
    slot[e] = s;
  }
}

// ------------------------------------------------------------ prep / finish
__global__ void als_prep_kernel(const double* D, const double* E, const double* V, int64_t J, int R,
                                AlsBufs b, int64_t* tstamp, int reset) {
  gram_dv_warps(D, E, V, J, R, b.cc, b.VtV, nullptr, nullptr);
  if (b.GD) {  // G_D = D^T D for the persistent loop's implicit V = D C
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int e = warp; e < R * R; e += nw) {
      const int a = e / R, c = e % R;
      double s = 0.0;
      for (int64_t j = lane; j < J; j += 32) s = fma(D[j * R + a], D[j * R + c], s);
      s = warp_sum(s);
      if (lane == 0) b.GD[e] = s;
    }
  }
  if (b.ps_gcnt && threadIdx.x < 64) b.ps_gcnt[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    b.ctl[8] = 0;
    for (int r = 0; r < R; ++r) b.nh[r] = 1.0;
    if (reset) {
      b.ctl[0] = 0;
      b.ctl[1] = 0;
      if (b.pwarm)
        for (int i = 0; i < 3; ++i) b.pwarm[i * (R * R + 8) + R * R] = 0.0;  // no warm pinv bases yet
    }
    if (tstamp) tstamp[0] = (int64_t)globaltimer_ns();
  }
}

__global__ void als_finish_kernel(AlsBufs b, int it, double tol, double* trace, int64_t* tstamp,
                                  int32_t* iters) {
  if (b.ctl[0]) return;
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int w = lane; w < b.nbm; w += 32) s += b.s_e[w];
  const double e = warp_sum(s);
  if (lane != 0) return;
  trace[it] = e;
  if (tstamp) tstamp[it + 1] = (int64_t)globaltimer_ns();
  *iters = it + 1;
  b.ctl[1] = 1;  // warm start valid from now on
  if (it > 0) {
    const double prev = trace[it - 1];
    if (prev == 0.0 || fabs(prev - e) <= tol * prev) b.ctl[0] = 1;
  }
}

// ------------------------------------------------------------ per-slice kernels
struct SliceArgs {
  const double *F, *D, *E, *H, *V, *W;
  double *polar, *theta, *Wout;
  int64_t K, J;
  int R;
  int mode1;      // rotate: also emit mode-1 and gram(W) partials
  int warm;       // rotate: warm start from b.pprev when b.ctl[1]
  int write_w;    // mode3: W_k = G3_k pinv3 (else write G3 into Wout)
  int write_l;    // mode3: emit L_k rows for the metric GEMM
  const double* g3_in;  // mode3: precomputed G3 (K x R), else formed per slice
  int64_t* status;
};

DP2_DEV void load_cta_common(const SliceArgs& a, const AlsBufs& b, CtaShared& s, bool needH, bool needPinv) {
  const int R = a.R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    s.cc[e] = b.cc[e];
    if (needH) s.H[e] = a.H[e];
    if (needPinv) s.aux[e] = b.pinv3[e];
  }
  for (int e = threadIdx.x; e < R; e += blockDim.x) {
    s.E[e] = a.E[e];
    s.vec[e] = b.nh[e];
  }
  __syncthreads();
}


// ------------------------------------------------------------ large R (R > 32)
// One CTA per slice: the one-sided Jacobi SVD of T_k parallel over the CTA --
// each round's independent column pairs (round-robin ordering) spread over
// the warps, each pair's three dot products and its column updates spread
// over the lanes -- instead of one warp doing all pairs and elements serially
// (the generic kernel above: ~25 ms per iteration at K = 1000, R = 50).
// ``pt``: the round-robin pairs, pt[r * np + i] = (p << 16) | q (rr_pair_table).
DP2_DEV void rr_pair_table(int n, int* pt) {
  const int ne = n + (n & 1), np = ne / 2;
  for (int e = threadIdx.x; e < (ne - 1) * np; e += blockDim.x) {
    int p, q;
    rr_pair(ne, e / np, e % np, p, q);
    pt[e] = (p << 16) | q;
  }
}

DP2_DEV int jacobi_onesided_cta(double* T, int ldt, double* V, int ldv, int n, const int* pt, int* flag,
                                int max_sweeps = 60) {
  // a pair per 8-lane group (4 per warp): a round of <= 28 pairs (n <= 56) is
  // one pass over the 256-thread CTA; lane `sub` of a group holds elements
  // sub, sub + 8, ... of the pair's two columns in registers between the dot
  // products (3 shuffle levels) and the rotation
  constexpr int KM = 7;
  const int sub = threadIdx.x & 7, grp = threadIdx.x >> 3;
  if (n < 2) return 0;
  const int ne = n + (n & 1), np = ne / 2;
  const double tol = n * kEps;  // rounding floor of the length-n dot products
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < ne - 1; ++r) {
      int p = 0, q = n;
      if (grp < np) {
        const int pq = pt[r * np + grp];
        p = pq >> 16;
        q = pq & 0xffff;
      }
      const bool live = q < n;
      double* tp = T + p * ldt;
      double* tq = T + (live ? q : p) * ldt;
      double x[KM], y[KM];
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int m = 0; m < KM; ++m) {
        const int k = sub + 8 * m;
        x[m] = (live && k < n) ? tp[k] : 0.0;
        y[m] = (live && k < n) ? tq[k] : 0.0;
        al = fma(x[m], x[m], al);
        be = fma(y[m], y[m], be);
        ga = fma(x[m], y[m], ga);
      }
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
#ifdef DP2_ROT_DEBUG
      if (live && sub == 0 && blockIdx.x == 0) {
        const float rel = (float)(ga * ga / (al * be + 1e-300));
        atomicMax(flag + 1, __float_as_int(rel));
        if (ga != 0.0 && ga * ga > (tol * tol) * (al * be)) atomicAdd(flag + 2, 1);
      }
#endif
      if (live && ga != 0.0 && ga * ga > (tol * tol) * (al * be)) {
        double c, sn;
        rot_params(be - al, ga, c, sn);
        double* vp = V + p * ldv;
        double* vq = V + q * ldv;
#pragma unroll
        for (int m = 0; m < KM; ++m) {
          const int k = sub + 8 * m;
          if (k < n) {
            tp[k] = c * x[m] - sn * y[m];
            tq[k] = sn * x[m] + c * y[m];
            const double a = vp[k], b = vq[k];
            vp[k] = c * a - sn * b;
            vq[k] = sn * a + c * b;
          }
        }
        if (sub == 0) *flag = 1;
      }
      __syncthreads();
    }
#ifdef DP2_ROT_DEBUG
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      printf("  sweep %d maxrel %.3e rots %d\n", sweep, __int_as_float(flag[1]), flag[2]);
      flag[1] = flag[2] = 0;
    }
#endif
    if (*flag == 0) break;
    __syncthreads();  // everyone has read the flag before it is reset
  }
  return sweep + 1;
}

__host__ __device__ inline size_t rotate_cta_doubles(int R) {
  return (size_t)2 * R * R /* Fs, Pi */ + (size_t)2 * R * (R + 1) /* Ts, Vr */ + (size_t)R + 16 /* norms, flag */ +
         (size_t)(R + 1) * (R + 2) / 4 + 1 /* pair table */;
}

// Polar factor of the R x R matrix T (row-major, ld R, in shared memory) by
// the CTA-parallel one-sided Jacobi SVD T V = Z Sigma (round-robin pairs over
// the warps, each pair's dot products and updates over 8 lanes), with the
// orthonormal completion of warp_polar for a (numerically) singular T:
// Pi = Z V^T (row-major, ld R).  Ts / Vr: R x (R + 1) scratch; nrm: R + 16
// doubles (flag after them); pt: the round-robin pair table.  The fallback of
// als_rotate_ns_kernel (R <= 56).
DP2_DEV void cta_polar_jacobi(const double* T, double* Pi, double* Ts, double* Vr, double* nrm, int* flag,
                              const int* pt, int R, int64_t k, int64_t* status) {
  const int RR = R * R, ldt = R + 1, tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < RR; e += nt) {  // columns of T, V = I
    const int c = e / R, i = e - c * R;
    Ts[c * ldt + i] = T[i * R + c];
    Vr[c * ldt + i] = c == i ? 1.0 : 0.0;
  }
  __syncthreads();
  const int sw = jacobi_onesided_cta(Ts, ldt, Vr, ldt, R, pt, flag);
  if (sw > 60 && tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
  for (int i = tid >> 5; i < R; i += nt >> 5) {  // column norms
    double sq = 0.0;
    for (int d = tid & 31; d < R; d += 32) sq = fma(Ts[i * ldt + d], Ts[i * ldt + d], sq);
    sq = warp_sum(sq);
    if ((tid & 31) == 0) nrm[i] = sqrt(sq);
  }
  __syncthreads();
  for (int e = tid; e < RR; e += nt) {
    const int i = e / R, d = e - i * R;
    const double n = nrm[i];
    Ts[i * ldt + d] = n > 1e-300 ? Ts[i * ldt + d] / n : 0.0;
  }
  __syncthreads();
  if (tid == 0) {  // (numerically) singular T_k: complete Z orthonormally, as warp_polar
    for (int i = 0; i < R; ++i) {
      if (nrm[i] > 1e-300) continue;
      for (int t = 0; t < R; ++t) {
        double* z = Ts + i * ldt;
        for (int d = 0; d < R; ++d) z[d] = (d == t) ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
          for (int c = 0; c < R; ++c) {
            if (c == i || !(nrm[c] > 1e-300)) continue;
            double dd = 0.0;
            for (int d = 0; d < R; ++d) dd = fma(Ts[c * ldt + d], z[d], dd);
            for (int d = 0; d < R; ++d) z[d] = fma(-dd, Ts[c * ldt + d], z[d]);
          }
        double n2 = 0.0;
        for (int d = 0; d < R; ++d) n2 = fma(z[d], z[d], n2);
        if (n2 > 0.25) {
          const double inv = 1.0 / sqrt(n2);
          for (int d = 0; d < R; ++d) z[d] *= inv;
          nrm[i] = 1.0;
          break;
        }
      }
      if (!(nrm[i] > 1e-300)) status_min(status, ST_POLAR, k);
    }
  }
  __syncthreads();
  for (int e = tid; e < RR; e += nt) {  // Pi[d][c] = sum_i Z[d][i] V[c][i]
    const int d = e / R, c = e - d * R;
    double s = 0.0;
    for (int i = 0; i < R; ++i) s = fma(Ts[i * ldt + d], Vr[i * ldt + c], s);
    Pi[e] = s;
  }
  __syncthreads();
}

// ---- CTA matmuls on the fp64 tensor pipe (DMMA m8n8k4) for 16 < R <= 56.
// Square NP x NP operands (NP = R rounded up to 8), C = op(A) op(B); shared
// operands are zero-padded to NP with row stride ld = 4 (mod 16) doubles
// (conflict-free fragment loads), global operands (ld R) are read with
// predicates.  Warp w owns the 8 x 8 output tiles w, w + 8, ... (two at a
// time: independent accumulator chains); every lane calls epi(m, n, c0, c1)
// for its elements (m, n), (m, n + 1) -- the ownership is static, so
// per-element read-modify-writes across calls are race-free.
__host__ __device__ inline bool rot_ns(int R) { return R > 16 && R <= 56; }  // als_rotate_ns_kernel range
__host__ __device__ inline int ns_np(int R) { return (R + 7) & ~7; }
__host__ __device__ inline int ns_ld(int R) { return ((ns_np(R) + 15) & ~15) + 4; }
__host__ __device__ inline size_t rotate_ns_doubles(int R) {
  const size_t mat = (size_t)ns_np(R) * ns_ld(R), ns = 3 * mat + 32, jac = rotate_cta_doubles(R) + (size_t)R * R;
  return ns > jac ? ns : jac;
}

template <bool TA, bool GA, bool TB, bool GB>
struct MmOp {
  const double* A;
  int lda;
  const double* B;
  int ldb;
  int R;
  DP2_DEV double a(int m, int k) const {
    if (GA && (m >= R || k >= R)) return 0.0;
    return TA ? A[k * lda + m] : A[m * lda + k];
  }
  DP2_DEV double b(int k, int n) const {
    if (GB && (k >= R || n >= R)) return 0.0;
    return TB ? B[n * ldb + k] : B[k * ldb + n];
  }
};

// A = X (shared, ld), B = Y = a (3I - a^2 S) / 2 from the shared S (scaled
// Newton-Schulz step)
struct MmOpY {
  const double* X;
  const double* S;
  int ld, R;
  double sa, sa2;
  DP2_DEV double a(int m, int k) const { return X[m * ld + k]; }
  DP2_DEV double b(int k, int n) const { return sa * ((k == n && k < R ? 1.5 : 0.0) - 0.5 * sa2 * S[k * ld + n]); }
};

template <int NP, class Op, class Epi>
DP2_DEV void cta_mm(const Op& op, Epi epi) {  // 256 threads; warp w owns tiles w, w + 8, ...
  constexpr int NT = NP / 8, NTILES = NT * NT, MT = (NTILES + 7) / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  double c[MT][2];
  int m0[MT], n0[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int t = warp + 8 * i < NTILES ? warp + 8 * i : 0;
    m0[i] = (t / NT) * 8;
    n0[i] = (t % NT) * 8;
    c[i][0] = c[i][1] = 0.0;
  }
  // all of the warp's tiles at once: MT independent accumulator chains
#pragma unroll 2
  for (int k0 = 0; k0 < NP; k0 += 4) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
      if (warp + 8 * i < NTILES) dmma_8x8x4(c[i][0], c[i][1], op.a(m0[i] + r, k0 + q), op.b(k0 + q, n0[i] + r));
  }
#pragma unroll
  for (int i = 0; i < MT; ++i)
    if (warp + 8 * i < NTILES) epi(m0[i] + r, n0[i] + 2 * q, c[i][0], c[i][1]);
}

// One CTA per slice (CTA-strided), 16 < R <= 56: T_k = (F_k cc) diag(w_k) H^T
// (P/solver.py:55-58) and its orthogonal polar factor Pi_k = Z_k P_k^T -- the
// only part of SVD(T_k) the reference consumes (P/solver.py:59, :71) -- by
// the Newton-Schulz iteration X <- X (3I - X^T X) / 2 from X0 = T / sqrt(m),
// m = min(||T^T T||_1, ||T^T T||_F) >= sigma_max^2 (so every singular value
// of X0 is in (0, 1]): R x R matmuls on the fp64 tensor pipe only, no
// divisions or data-dependent rotations on the critical path.  It stops when
// ||I - X^T X||_F < 1e-12 after one more step (quadratic convergence: the
// result is orthogonal to rounding).  A singular or extremely ill-conditioned
// T_k (no convergence in 100 steps) falls back to the CTA-parallel one-sided
// Jacobi with orthonormal completion (cta_polar_jacobi).  Then Theta_k =
// Pi_k^T F_k (P/solver.py:67-75) and the mode-1 partials into this CTA's
// slots (ordered by slice within the CTA).
template <int NP>
__global__ void __launch_bounds__(256, 2) als_rotate_ns_kernel(SliceArgs a, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  constexpr int LD = ((NP + 15) & ~15) + 4;
  const int R = a.R, RR = R * R, tid = threadIdx.x, nt = blockDim.x;
  const size_t MAT = (size_t)NP * LD;
  double* X = sm;
  double* S = X + MAT;
  double* Xn = S + MAT;
  double* red = Xn + MAT;  // [1] col-sum max, [2] ||S||_F^2, [4 + (it & 1)] ||I - S||_F^2 of step it
  const double* __restrict__ cc = b.cc;
  const double* __restrict__ H = a.H;
  double* acc1 = a.mode1 ? b.s_g1 + (size_t)blockIdx.x * RR : nullptr;  // this CTA's partial slots
  double* acc2 = a.mode1 ? b.s_wtw + (size_t)blockIdx.x * RR : nullptr;
  if (a.mode1)
    for (int e = tid; e < RR; e += nt) acc1[e] = acc2[e] = 0.0;
  for (int e = tid; e < 3 * (int)MAT; e += nt) sm[e] = 0.0;  // zero padding stays zero
  __syncthreads();
  for (int64_t k = blockIdx.x; k < a.K; k += gridDim.x) {
    const double* Fk = a.F + k * RR;
    const double* wk = a.W + k * R;
    // Th = (F_k cc) diag(w_k) -> S
    cta_mm<NP>(MmOp<false, true, false, true>{Fk, R, cc, R, R}, [&](int m, int n, double c0, double c1) {
      S[m * LD + n] = n < R ? c0 * __ldg(wk + n) : 0.0;
      S[m * LD + n + 1] = n + 1 < R ? c1 * __ldg(wk + n + 1) : 0.0;
    });
    if (tid < 6) red[tid] = 0.0;
    __syncthreads();
    // T = Th H^T -> X
    cta_mm<NP>(MmOp<false, false, true, true>{S, LD, H, R, R}, [&](int m, int n, double c0, double c1) {
      X[m * LD + n] = c0;
      X[m * LD + n + 1] = c1;
    });
    __syncthreads();
    // S = T^T T; m = min(max column |.| sum, Frobenius norm) of S >= sigma_max(T)^2
    cta_mm<NP>(MmOp<true, false, false, false>{X, LD, X, LD, R}, [&](int m, int n, double c0, double c1) {
      S[m * LD + n] = c0;
      S[m * LD + n + 1] = c1;
    });
    __syncthreads();
    {
      double f = 0.0;
      for (int e = tid; e < NP * NP; e += nt) {
        const double v = S[(e / NP) * LD + e % NP];
        f = fma(v, v, f);
      }
      f = warp_sum(f);
      if ((tid & 31) == 0) atomicAdd(red + 2, f);
      if (tid < NP) {
        double cs = 0.0;
        for (int i = 0; i < NP; ++i) cs += fabs(S[i * LD + tid]);
        atomicMax(reinterpret_cast<unsigned long long*>(red + 1), (unsigned long long)__double_as_longlong(cs));
      }
    }
    __syncthreads();
    const double mb = fmin(red[1], sqrt(red[2]));
    bool done = false;
    if (mb > 0.0 && isfinite(mb)) {
      const double al = 1.0 / sqrt(mb), al2 = 1.0 / mb;
      for (int e = tid; e < NP * NP; e += nt) {  // X0 = al T, S0 = X0^T X0
        const int i = e / NP, j = e % NP;
        X[i * LD + j] *= al;
        S[i * LD + j] *= al2;
      }
      __syncthreads();
      double* Xc = X;
      double* Xo = Xn;
      bool last = false;
      // scaled Newton-Schulz (the optimally scaled cubic of Chen & Chow):
      // with every singular value of X in [lb, 1], X <- a X (3I - a^2 X^T X) / 2,
      // a^2 = 3 / (1 + lb + lb^2), maps [lb, 1] into [lb', 1],
      // lb' = a lb (3 - a^2 lb^2) / 2 (~2.6 lb for small lb against 1.5 lb
      // unscaled).  lb starts at 1e-7 (a smaller true sigma_min only grows more
      // slowly) and is raised to the bound sqrt(1 - ||I - X^T X||_F) once
      // that is < 1, so the last steps are the plain quadratic iteration.
      double lb = 1e-7;
      for (int it = 0; it < 100; ++it) {
        const double a2 = 3.0 / (1.0 + lb + lb * lb), a = sqrt(a2);
        // Xo = Xc Y, Y = a (3I - a^2 S) / 2 formed in the fragment loads
        cta_mm<NP>(MmOpY{Xc, S, LD, R, a, a2}, [&](int m, int n, double c0, double c1) {
          Xo[m * LD + n] = c0;
          Xo[m * LD + n + 1] = c1;
        });
        __syncthreads();
        // every thread has read the previous step's error: recycle its slot
        if (tid == 0) red[4 + ((it + 1) & 1)] = 0.0;
        lb = fmin(1.0, 0.5 * a * lb * (3.0 - a2 * lb * lb));
        double* t = Xc;
        Xc = Xo;
        Xo = t;
        if (last) { done = true; break; }
        // S = Xc^T Xc, with ||I - S||_F^2
        double ep = 0.0;
        cta_mm<NP>(MmOp<true, false, false, false>{Xc, LD, Xc, LD, R}, [&](int m, int n, double c0, double c1) {
          const double d0 = (m == n && m < R ? 1.0 : 0.0) - c0, d1 = (m == n + 1 && m < R ? 1.0 : 0.0) - c1;
          ep = fma(d0, d0, fma(d1, d1, ep));
          S[m * LD + n] = c0;
          S[m * LD + n + 1] = c1;
        });
        ep = warp_sum(ep);
        if ((tid & 31) == 0) atomicAdd(red + 4 + (it & 1), ep);
        __syncthreads();
        const double e2 = red[4 + (it & 1)];
        if (!isfinite(e2)) break;
        if (e2 < 1.0) lb = fmax(lb, sqrt(1.0 - sqrt(e2)));
        if (e2 < 1e-24) last = true;  // one more step squares the error
#ifdef DP2_NS_DEBUG
        if (tid == 0 && blockIdx.x < 2 && (it % 5 == 0 || last)) printf("k %lld it %d e2 %.3e lb %.3e\n", (long long)k, it, e2, lb);
#endif
      }
      if (done && Xc != X) {  // result into X
        for (int e = tid; e < NP * NP; e += nt) X[(e / NP) * LD + e % NP] = Xc[(e / NP) * LD + e % NP];
        __syncthreads();
      }
    }
    double* Pi = X;  // polar factor, padded layout (ld LD)
    if (!done) {     // fallback: T again (row-major, ld R) -> Jacobi -> Pi (ld R) -> padded X
      double* Tr = sm;
      double* Pr = Tr + RR;
      double* Ts = Pr + RR;
      double* Vr = Ts + R * (R + 1);
      double* nrm = Vr + R * (R + 1);
      int* flag = reinterpret_cast<int*>(nrm + R + 8);
      int* pt = flag + 16;
      __syncthreads();
      for (int e = tid; e < RR; e += nt) {  // Th = (F_k cc) diag(w_k) into Pr
        const int i = e / R, c = e - i * R;
        double s = 0.0;
        for (int q = 0; q < R; ++q) s = fma(__ldg(Fk + i * R + q), __ldg(cc + q * R + c), s);
        Pr[e] = s * __ldg(wk + c);
      }
      rr_pair_table(R, pt);
      __syncthreads();
      for (int e = tid; e < RR; e += nt) {  // T = Th H^T
        const int i = e / R, d = e - i * R;
        double s = 0.0;
        for (int c = 0; c < R; ++c) s = fma(Pr[i * R + c], __ldg(H + d * R + c), s);
        Tr[e] = s;
      }
      __syncthreads();
      cta_polar_jacobi(Tr, Pr, Ts, Vr, nrm, flag, pt, R, k, a.status);
      double pv[(56 * 56 + 255) / 256];
#pragma unroll
      for (int u = 0; u < (56 * 56 + 255) / 256; ++u) {
        const int e = tid + 256 * u;
        pv[u] = e < RR ? Pr[e] : 0.0;
      }
      __syncthreads();
      for (int e = tid; e < 3 * (int)MAT; e += nt) sm[e] = 0.0;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < (56 * 56 + 255) / 256; ++u) {
        const int e = tid + 256 * u;
        if (e < RR) X[(e / R) * LD + e % R] = pv[u];
      }
      __syncthreads();
    }
    if (a.polar)
      for (int e = tid; e < RR; e += nt) a.polar[k * RR + e] = Pi[(e / R) * LD + e % R];
    // Theta = Pi^T F_k -> S (and out)
    cta_mm<NP>(MmOp<true, false, false, true>{Pi, LD, Fk, R, R}, [&](int m, int n, double c0, double c1) {
      S[m * LD + n] = c0;
      S[m * LD + n + 1] = c1;
      if (m < R) {
        if (n < R) a.theta[k * RR + m * R + n] = c0;
        if (n + 1 < R) a.theta[k * RR + m * R + n + 1] = c1;
      }
    });
    __syncthreads();
    if (a.mode1)  // g1[i][r] += w[k][r] (Theta cc)[i][r];  wtw[i][r] += w[k][i] w[k][r]
      cta_mm<NP>(MmOp<false, false, false, true>{S, LD, cc, R, R}, [&](int m, int n, double c0, double c1) {
        if (m < R) {
          const double wm = __ldg(wk + m);
          if (n < R) {
            const double wn = __ldg(wk + n);
            acc1[m * R + n] += wn * c0;
            acc2[m * R + n] += wm * wn;
          }
          if (n + 1 < R) {
            const double wn = __ldg(wk + n + 1);
            acc1[m * R + n + 1] += wn * c1;
            acc2[m * R + n + 1] += wm * wn;
          }
        }
      });
    __syncthreads();
  }
}

// Rotation kernel with compile-time R (R <= 16), one warp per slice: the polar
// factor of T_k by the Newton-Schulz iteration (R x R warp matmuls only) --
// the unique orthogonal polar factor of the nonsingular T_k, i.e. the
// reference's Z_k P_k^T (P/solver.py:59).  A singular or extremely
// ill-conditioned T_k (no convergence in 80 steps) falls back to one-sided
// Jacobi with orthonormal completion (warp_polar).
template <int R>
__host__ __device__ constexpr int grp_doubles() { return 13 * R * R + 2 * R * (R | 1) + 8 * R; }
template <int R>
__host__ __device__ constexpr int grp_per_warp() { return 1; }

// Gauss-Jordan inverse with partial pivoting of the R x R matrix in aug[:, :R]
// (aug is R x 2R); result in aug[:, R:].  Returns false on a zero pivot.
template <int R>
DP2_DEV bool wgj_inverse(double* aug, double* fac) {
  const int lane = threadIdx.x & 31;
  constexpr int W = 2 * R;
#pragma unroll
  for (int it = 0; it < (R * R + 31) / 32; ++it) {
    const int e = lane + 32 * it;
    if (e < R * R) aug[(e / R) * W + R + e % R] = (e / R == e % R) ? 1.0 : 0.0;
  }
  __syncwarp();
  for (int c = 0; c < R; ++c) {
    double best = lane >= c && lane < R ? fabs(aug[lane * W + c]) : -1.0;
    int bi = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (!(best > 0.0)) return false;
    if (bi != c)
      for (int j = lane; j < W; j += 32) {
        const double t = aug[c * W + j];
        aug[c * W + j] = aug[bi * W + j];
        aug[bi * W + j] = t;
      }
    __syncwarp();
    const double inv = 1.0 / aug[c * W + c];
    if (lane < R) fac[lane] = aug[lane * W + c];
    __syncwarp();
    for (int j = lane; j < W; j += 32) aug[c * W + j] *= inv;
    __syncwarp();
    for (int e = lane; e < R * W; e += 32) {
      const int i = e / W, j = e % W;
      if (i != c) aug[e] = fma(-fac[i], aug[c * W + j], aug[e]);
    }
    __syncwarp();
  }
  return true;
}

template <int R>
__global__ void __launch_bounds__(128) als_rotate_group_kernel(SliceArgs a, AlsBufs b, int wpb_r) {
  if (b.ctl[0]) return;
  constexpr int LDT = R | 1, PER = grp_doubles<R>(), RR = R * R;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* cc = sm;
  double* Hs = cc + RR;
  double* base = sm + 2 * RR + (size_t)wib * PER;
  double* Fs = base;
  double* Th = Fs + RR;
  double* T = Th + RR;
  double* Pp = T + RR;
  double* X = Pp + RR;
  double* Y = X + RR;
  double* Pi = Y + RR;
  double* aug = Pi + RR;      // R x 2R
  double* acc1 = aug + 2 * RR;
  double* acc2 = acc1 + RR;
  double* Ts = acc2 + RR;     // Jacobi fallback: R x LDT each
  double* Vr = Ts + R * LDT;
  double* tmp = Vr + R * LDT;  // 8R
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    cc[e] = b.cc[e];
    Hs[e] = a.H[e];
  }
  __syncthreads();
  for (int e = lane; e < RR; e += 32) { acc1[e] = 0.0; acc2[e] = 0.0; }
  const bool warm = a.warm && b.ctl[1];
  const int64_t gw = (int64_t)blockIdx.x * wpb_r + wib, nwr = (int64_t)gridDim.x * wpb_r;
  for (int64_t k = gw; k < a.K; k += nwr) {
    const double* wk = a.W + k * R;
    for (int e = lane; e < RR; e += 32) {
      Fs[e] = a.F[k * RR + e];
      if (warm) Pp[e] = b.pprev[k * RR + e];
    }
    __syncwarp();
    wmm<R, false, false>(Fs, cc, Th);  // Th = F_k cc
    for (int e = lane; e < RR; e += 32) Th[e] *= wk[e % R];
    __syncwarp();
    wmm<R, false, true>(Th, Hs, T);  // T = Th H^T
    // Newton-Schulz iteration for the polar factor: X0 = T / ||T||_F (all
    // singular values in (0, 1]), X <- X (3I - X^T X) / 2; converges to the
    // orthogonal polar factor of any nonsingular T (quadratically once the
    // singular values approach 1).  Stop when the update is < 3e-8 (the next
    // step's error is ~ the square of that).  Only R x R matmuls: no inverse,
    // no divisions on the critical path.
    bool done = false;
    {
      double nt = 0.0;
      for (int e = lane; e < RR; e += 32) nt = fma(T[e], T[e], nt);
      nt = warp_sum(nt);
      if (nt > 0.0 && isfinite(nt)) {
        const double inv = 1.0 / sqrt(nt);
        for (int e = lane; e < RR; e += 32) X[e] = T[e] * inv;
        __syncwarp();
        double* Xc = X;
        double* Xn = Pi;
        for (int it = 0; it < 80; ++it) {
          wmm<R, true, false>(Xc, Xc, Y);  // Y = X^T X
          for (int e = lane; e < RR; e += 32) Y[e] = ((e / R == e % R) ? 1.5 : 0.0) - 0.5 * Y[e];
          __syncwarp();
          wmm<R, false, false>(Xc, Y, Xn);  // Xn = X (3I - X^T X) / 2
          double d = 0.0;
          for (int e = lane; e < RR; e += 32) {
            const double t = Xn[e] - Xc[e];
            d = fma(t, t, d);
          }
          d = warp_sum(d);
          double* t = Xc;
          Xc = Xn;
          Xn = t;
          if (d < 9e-16) { done = true; break; }
        }
        if (done && Xc != Pi) {
          for (int e = lane; e < RR; e += 32) Pi[e] = Xc[e];
          __syncwarp();
        }
      }
    }
    if (!done) {  // cold start / fallback: one-sided Jacobi on T
      for (int e = lane; e < RR; e += 32) {
        const int i = e / R, c = e % R;
        Ts[c * LDT + i] = T[e];
        Vr[c * LDT + i] = (i == c) ? 1.0 : 0.0;
      }
      __syncwarp();
      warp_polar(Ts, Vr, LDT, R, Pi, tmp, a.status, k);
    }
    for (int e = lane; e < RR; e += 32) {
      b.pprev[k * RR + e] = Pi[e];
      if (a.polar) a.polar[k * RR + e] = Pi[e];
    }
    wmm<R, true, false>(Pi, Fs, Th);  // Theta = Pi^T F
    for (int e = lane; e < RR; e += 32) a.theta[k * RR + e] = Th[e];
    if (a.mode1)
      for (int e = lane; e < RR; e += 32) {
        const int i = e / R, r = e % R;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) s = fma(Th[i * R + q], cc[q * R + r], s);
        acc1[e] += wk[r] * s;
        acc2[e] += wk[i] * wk[r];
      }
    __syncwarp();
  }
  if (a.mode1) {
    __syncthreads();
    const double* g0 = sm + 2 * RR;
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
      double s1 = 0.0, s2 = 0.0;
      for (int w = 0; w < wpb_r; ++w) {
        const double* gb = g0 + (size_t)w * PER + 9 * RR;  // acc1 (acc2 follows)
        s1 += gb[e];
        s2 += gb[RR + e];
      }
      b.s_g1[(size_t)blockIdx.x * RR + e] = s1;
      b.s_wtw[(size_t)blockIdx.x * RR + e] = s2;
    }
  }
}

// mode-1 partials from a given Theta stack (kernel-granular API)
__global__ void als_mode1_kernel(SliceArgs a, AlsBufs b) {
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CtaShared cs = carve_cta(sm, R);
  const size_t wstride = 3 * (size_t)R * R;
  double* wbase = sm + cta_shared_doubles(R);
  double* acc1 = wbase + wib * wstride;
  double* acc2 = acc1 + R * R;
  load_cta_common(a, b, cs, false, false);
  for (int e = lane; e < R * R; e += 32) { acc1[e] = 0.0; acc2[e] = 0.0; }
  const int gw = blockIdx.x * b.wpb + wib;
  for (int64_t k = gw; k < a.K; k += b.nwt) {
    const double* Th = a.theta + k * R * R;
    const double* wk = a.W + k * R;
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, r = e % R;
      double s = 0.0;
      for (int q = 0; q < R; ++q) s = fma(Th[i * R + q], cs.cc[q * R + r], s);
      acc1[e] += wk[r] * s;
      acc2[e] += wk[i] * wk[r];
    }
  }
  __syncthreads();
  combine_warps(wbase, wstride, b.wpb, R * R, b.s_g1 + (size_t)blockIdx.x * R * R);
  combine_warps(wbase + R * R, wstride, b.wpb, R * R, b.s_wtw + (size_t)blockIdx.x * R * R);
}

__global__ void als_mode2_kernel(SliceArgs a, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CtaShared cs = carve_cta(sm, R);
  const size_t wstride = 3 * (size_t)R * R;
  double* wbase = sm + cta_shared_doubles(R);
  double* acc1 = wbase + wib * wstride;
  double* acc2 = acc1 + R * R;
  double* Th = acc2 + R * R;  // Theta_k staged in smem
  load_cta_common(a, b, cs, true, false);
  for (int e = lane; e < R * R; e += 32) { acc1[e] = 0.0; acc2[e] = 0.0; }
  const int gw = blockIdx.x * b.wpb + wib;
  for (int64_t k = gw; k < a.K; k += b.nwt) {
    for (int e = lane; e < R * R; e += 32) Th[e] = a.theta[k * R * R + e];
    __syncwarp();
    const double* wk = a.W + k * R;
    for (int e = lane; e < R * R; e += 32) {
      const int ai = e / R, r = e % R;
      double s = 0.0;  // (Theta^T H)[ai][r]
      for (int q = 0; q < R; ++q) s = fma(Th[q * R + ai], cs.H[q * R + r], s);
      const double wr = wk[r] * cs.vec[r], wa = wk[ai] * cs.vec[ai];
      acc1[e] += wr * s;
      acc2[e] += wa * wr;
    }
    __syncwarp();
  }
  __syncthreads();
  combine_warps(wbase, wstride, b.wpb, R * R, b.s_m2 + (size_t)blockIdx.x * R * R);
  combine_warps(wbase + R * R, wstride, b.wpb, R * R, b.s_wtw2 + (size_t)blockIdx.x * R * R);
}

// ---- R > 16: modes 2 and 3 as GEMMs over the Theta stack (K x R^2):
//   mode 2: T = Theta^T W (R^2 x R, T[(q, a)][r] = sum_k w_kr Theta_k[q][a]), then
//           summed[a][r] = nh_r sum_q H[q][r] T[(q, a)][r] and gram(W nh)
//           (the reference's sum_k w_k nh (Theta_k^T H), P/solver.py:93-101,
//           summed over k first)
//   mode 3: G3 = Theta Z (K x R), Z[(i, j)][r] = H[i][r] cc[j][r]
//           (P/solver.py:104-111)
// on the DMMA skinny-GEMM kernels of stage 2 (ordered split-K reductions).
__global__ void als_m2_finish_kernel(const int32_t* ctl, const double* t3, const double* wtw, const double* H,
                                     const double* nh, int R, double* summed, double* wtw2) {
  if (ctl[0]) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * R; e += gridDim.x * blockDim.x) {
    const int a = e / R, r = e % R;
    double s = 0.0;
    for (int q = 0; q < R; ++q) s = fma(H[q * R + r], t3[((size_t)q * R + a) * R + r], s);
    summed[e] = nh[r] * s;
    wtw2[e] = (nh[a] * nh[r]) * wtw[e];
  }
}

__global__ void als_z_kernel(const int32_t* ctl, const double* H, const double* cc, int R, double* zz) {
  if (ctl[0]) return;
  const int n = R * R * R;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int r = e % R, ij = e / R, i = ij / R, j = ij % R;
    zz[e] = H[i * R + r] * cc[j * R + r];
  }
}

// G3 row, new W row, and the metric operator rows L_k = [Theta_k E | -H W_k]
__global__ void als_mode3_kernel(SliceArgs a, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CtaShared cs = carve_cta(sm, R);
  double* g3 = sm + cta_shared_doubles(R) + (size_t)wib * ((size_t)R * R + 2 * R);
  double* wn = g3 + R;
  double* Th = wn + R;  // Theta_k staged in smem
  load_cta_common(a, b, cs, true, a.write_w != 0);
  const int gw = blockIdx.x * b.wpb + wib;
  const int ldl = 2 * R;
  for (int64_t k = gw; k < a.K; k += b.nwt) {
    for (int e = lane; e < R * R; e += 32) Th[e] = a.theta[k * R * R + e];
    __syncwarp();
    // G3[r] = sum_i H[i][r] sum_j Theta[i][j] cc[j][r]   (P/solver.py:109-111)
    for (int r = lane; r < R; r += 32) {
      if (a.g3_in) {
        g3[r] = a.g3_in[k * R + r];
        continue;
      }
      double s = 0.0;
      for (int i = 0; i < R; ++i) {
        double h = 0.0;
        for (int j = 0; j < R; ++j) h = fma(Th[i * R + j], cs.cc[j * R + r], h);
        s = fma(cs.H[i * R + r], h, s);
      }
      g3[r] = s;
    }
    __syncwarp();
    for (int c = lane; c < R; c += 32) {
      double s;
      if (a.write_w) {
        s = 0.0;
        for (int r = 0; r < R; ++r) s = fma(g3[r], cs.aux[r * R + c], s);
      } else {
        s = g3[c];
      }
      wn[c] = s;
      if (a.Wout) a.Wout[k * R + c] = s;
    }
    __syncwarp();
    if (a.write_l) {
      const double* wk = a.write_w ? wn : a.W + k * R;
      for (int e = lane; e < R * ldl; e += 32) {
        const int i = e / ldl, c = e % ldl;
        b.L[(k * R + i) * ldl + c] = c < R ? Th[i * R + c] * cs.E[c] : -(cs.H[i * R + (c - R)] * wk[c - R]);
      }
    }
    __syncwarp();
  }
}

// e partials: ||L N^T||_F^2 over row tiles of L (rows = K*R, cols = 2R) with
// N = [D V] (J x 2R).  Warp tile: 8 rows of L x all J in 8-column DMMA tiles;
// A fragments (L rows) stay in registers, N streams through shared memory.
template <int KS>  // k-steps of 4 covering 2R (padded)
__global__ void __launch_bounds__(256) als_metric_kernel(AlsBufs b, const double* D, const double* V, int64_t J,
                                                         int R, int64_t rowsL) {
  if (b.ctl[0]) return;
  constexpr int JC = KS <= 12 ? 64 : 32;
  __shared__ double ns[JC][4 * KS + 1];
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ldl = 2 * R;
  const int64_t mtiles = (rowsL + 7) / 8;
  double acc = 0.0;
  for (int64_t mt0 = (int64_t)blockIdx.x * 8; mt0 < mtiles; mt0 += (int64_t)gridDim.x * 8) {
    const int64_t mt = mt0 + warp;
    double af[KS];
    const int64_t row = mt * 8 + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int c = ks * 4 + (lane & 3);
      af[ks] = (mt < mtiles && row < rowsL && c < ldl) ? b.L[row * ldl + c] : 0.0;
    }
    for (int64_t j0 = 0; j0 < J; j0 += JC) {
      __syncthreads();
      for (int e = threadIdx.x; e < JC * 4 * KS; e += blockDim.x) {
        const int jj = e / (4 * KS), c = e % (4 * KS);
        const int64_t j = j0 + jj;
        double v = 0.0;
        if (j < J && c < ldl) v = c < R ? D[j * R + c] : V[j * R + (c - R)];
        ns[jj][c] = v;
      }
      __syncthreads();
      if (mt < mtiles) {
        const int nj = (int)imin64(JC, J - j0);
        for (int nt = 0; nt * 8 < nj; ++nt) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) dmma_8x8x4(c0, c1, af[ks], ns[nt * 8 + (lane >> 2)][ks * 4 + (lane & 3)]);
          acc = fma(c0, c0, acc);
          acc = fma(c1, c1, acc);
        }
      }
    }
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) b.s_e[blockIdx.x] = tot;
}

// rows per staged chunk of D / V in als_solve_v_kernel's large-J path (227 KB cap)
__host__ __device__ inline int solve_v_jt(int R) { return R <= 50 ? 32 : 8; }

struct SolveArgs {
  const double *D, *E;
  double *H, *V, *W;
  int64_t J;
  int R, normalize, nslots, nslots_h, dsm;
  int64_t* status;
};

__global__ void __launch_bounds__(512) als_solve_h_kernel(SolveArgs s, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = s.R;
  double* G1 = sm;
  double* WtW = G1 + R * R;
  double* Mh = WtW + R * R;
  double* U = Mh + R * R;
  double* Pv = U + R * R;
  double* Hn = Pv + R * R;
  double* cs = Hn + R * R;  // 3*(R/2+1)
  __shared__ double nrm[64];
  reduce_slots_warp(b.s_g1, s.nslots_h, R * R, G1);
  reduce_slots_warp(b.s_wtw, s.nslots_h, R * R, WtW);
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    Mh[e] = WtW[e] * b.VtV[e];
    b.G1[e] = G1[e];
    b.WtW[e] = WtW[e];
  }
  __syncthreads();
  block_pinv_sym(Mh, U, Pv, R, cs, s.status, b.pwarm);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, c = e % R;
    double acc = 0.0;
    for (int q = 0; q < R; ++q) acc = fma(G1[i * R + q], Pv[q * R + c], acc);
    Hn[e] = acc;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < R; c += blockDim.x) {
    double n2 = 0.0;
    for (int i = 0; i < R; ++i) n2 = fma(Hn[i * R + c], Hn[i * R + c], n2);
    const double n = sqrt(n2);
    nrm[c] = (s.normalize && !(n < 1e-300)) ? n : 1.0;
    b.nh[c] = nrm[c];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    Hn[e] = Hn[e] / nrm[e % R];
    s.H[e] = Hn[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, c = e % R;
    double acc = 0.0;
    for (int q = 0; q < R; ++q) acc = fma(Hn[q * R + i], Hn[q * R + c], acc);
    b.HtH[e] = acc;
  }
}

__global__ void __launch_bounds__(512) als_solve_v_kernel(SolveArgs s, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = s.R;
  const int64_t J = s.J;
  double* summed = sm;
  double* WtW2 = summed + R * R;
  double* Mv = WtW2 + R * R;
  double* U = Mv + R * R;
  double* Pv = U + R * R;
  double* es = Pv + R * R;  // E * summed
  double* cs = es + R * R;
  __shared__ double nrm[64];
  double* EP = cs + 3 * (R / 2 + 1) + 8;
  double* Ds = EP + R * R;
  double* Vs = s.dsm ? Ds + J * R : b.G2;
  const double* Dp = s.dsm ? Ds : s.D;
  // stage D first: its load overlaps the slot reductions and warp 0's pinv
  if (s.dsm)
    for (int64_t e = threadIdx.x; e < J * R; e += blockDim.x) Ds[e] = s.D[e];
  reduce_slots_warp(b.s_m2, s.nslots, R * R, summed);
  reduce_slots_warp(b.s_wtw2, s.nslots, R * R, WtW2);
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    Mv[e] = WtW2[e] * b.HtH[e];
    es[e] = s.E[e / R] * summed[e];
    b.summed[e] = summed[e];
    b.WtW2[e] = WtW2[e];
  }
  __syncthreads();
  block_pinv_sym(Mv, U, Pv, R, cs, s.status, b.pwarm ? b.pwarm + (R * R + 8) : nullptr);
  // V = D (E * summed) pinv = D EP with EP = (E * summed) pinv (R x R), so the
  // J-sized work is one product; D and V stay in smem when they fit
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int q = e / R, r = e % R;
    double acc = 0.0;
    for (int a2 = 0; a2 < R; ++a2) acc = fma(es[q * R + a2], Pv[a2 * R + r], acc);
    EP[e] = acc;
  }
  __syncthreads();
  if (s.dsm) {
    for (int64_t e = threadIdx.x; e < J * R; e += blockDim.x) {
      const int64_t j = e / R;
      const int r = (int)(e % R);
      double acc = 0.0;
      for (int q = 0; q < R; ++q) acc = fma(Dp[j * R + q], EP[q * R + r], acc);
      Vs[e] = acc;
    }
    __syncthreads();
    {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int c = warp; c < R; c += nw) {
        double part = 0.0;
        for (int64_t j = lane; j < J; j += 32) part = fma(Vs[j * R + c], Vs[j * R + c], part);
        const double n = sqrt(warp_sum(part));
        if (lane == 0) nrm[c] = (s.normalize && !(n < 1e-300)) ? n : 1.0;
      }
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < J * R; e += blockDim.x) {
      const double v = Vs[e] / nrm[e % R];
      Vs[e] = v;
      s.V[e] = v;
    }
    __syncthreads();
    gram_dv_warps(Dp, s.E, Vs, J, R, b.cc, b.VtV, Mv, b.HtH);
    __syncthreads();
  } else {
    // D and V do not fit in shared memory: one sweep over row chunks of D
    // (staged coalesced) computes V = D EP (unnormalised, into G2) and the
    // unnormalised grams D^T V and V^T V in registers (thread entries e = tid
    // + 512 u, rows in ascending order); the column norms are the diagonal of
    // V^T V, and the normalised V, cc = E * (D^T V) and V^T V follow by
    // scaling (P/solver.py:126-128, push_col_norms then the grams).
    constexpr int MAXU = 8;  // R * R <= 4096 entries over 512 threads
    const int JT = solve_v_jt(R);
    double* Dc = EP + R * R;          // JT x R
    double* Vc = Dc + JT * R;         // JT x R
    double g1[MAXU], g2[MAXU];
#pragma unroll
    for (int u = 0; u < MAXU; ++u) g1[u] = g2[u] = 0.0;
    const int nt = blockDim.x, tid = threadIdx.x;
    for (int64_t j0 = 0; j0 < J; j0 += JT) {
      const int nj = (int)(J - j0 < JT ? J - j0 : JT);
      for (int e = tid; e < nj * R; e += nt) Dc[e] = Dp[j0 * R + e];
      __syncthreads();
      for (int e = tid; e < nj * R; e += nt) {
        const int jj = e / R, r = e - jj * R;
        double acc = 0.0;
        for (int q = 0; q < R; ++q) acc = fma(Dc[jj * R + q], EP[q * R + r], acc);
        Vc[e] = acc;
        Vs[j0 * R + e] = acc;
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < MAXU; ++u) {
        const int e = tid + nt * u;
        if (e < R * R) {
          const int a = e / R, r = e - a * R;
          double t1 = g1[u], t2 = g2[u];
          for (int jj = 0; jj < nj; ++jj) {
            const double v = Vc[jj * R + r];
            t1 = fma(Dc[jj * R + a], v, t1);
            t2 = fma(Vc[jj * R + a], v, t2);
          }
          g1[u] = t1;
          g2[u] = t2;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < MAXU; ++u) {
      const int e = tid + nt * u;
      if (e < R * R && e / R == e % R) {
        const double n = sqrt(g2[u]);
        nrm[e / R] = (s.normalize && !(n < 1e-300)) ? n : 1.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < MAXU; ++u) {
      const int e = tid + nt * u;
      if (e < R * R) {
        const int a = e / R, r = e - a * R;
        const double vtv = g2[u] / (nrm[a] * nrm[r]);
        b.cc[e] = s.E[a] * (g1[u] / nrm[r]);
        b.VtV[e] = vtv;
        Mv[e] = vtv * b.HtH[e];
      }
    }
    for (int64_t e = tid; e < J * R; e += nt) s.V[e] = Vs[e] / nrm[e % R];
    __syncthreads();
  }
  block_pinv_sym(Mv, U, Pv, R, cs, s.status, b.pwarm ? b.pwarm + 2 * (R * R + 8) : nullptr);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) b.pinv3[e] = Pv[e];
}


// ------------------------------------------------------------ host side
namespace {

struct AlsLayout {
  size_t theta, pprev, cc, nh, HtH, VtV, pinv3, G1, WtW, summed, WtW2, L, s_g1, s_wtw, s_m2, s_wtw2, s_e, G2, g3,
      GD, ps_slots, ps_e, ps_C, ps_stamps, ps_gslots, ps_gcnt, pwarm, t3, zz, gp, ctl, total;
};

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int total_warps(int64_t K, int R) {
  const int wpb = wpb_for(R);
  const int64_t maxw = (int64_t)sm_count() * 4 * wpb;
  int64_t w = K < maxw ? K : maxw;
  w = ((w + wpb - 1) / wpb) * wpb;
  return (int)(w < wpb ? wpb : w);
}

int metric_blocks(int64_t K, int R) {
  const int64_t mtiles = (K * R + 7) / 8;
  const int64_t b = (mtiles + 7) / 8;
  const int64_t cap = (int64_t)sm_count() * 4;
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

// compile-time-R rotation kernel configuration (R <= 16); nbr = 0 -> generic kernel
template <int R>
void rot_cfg_t(int64_t K, int& wpbr, int& nbr) {
  constexpr int NG = grp_per_warp<R>();
  const size_t per_warp = (size_t)NG * grp_doubles<R>() * 8 + 2 * R * R * 8;
  wpbr = (int)(160 * 1024 / per_warp);
  wpbr = wpbr < 1 ? 1 : (wpbr > 4 ? 4 : wpbr);
  int64_t warps = (K + NG - 1) / NG;
  const int64_t cap = (int64_t)sm_count() * 8;
  warps = warps < cap ? warps : cap;
  nbr = (int)((warps + wpbr - 1) / wpbr);
}
void rot_cfg(int64_t K, int R, int& wpbr, int& nbr) {
  wpbr = 0;
  nbr = 0;
  switch (R) {
#define DP2_ROT_CASE(N) \
  case N: rot_cfg_t<N>(K, wpbr, nbr); break;
    DP2_ROT_CASE(1) DP2_ROT_CASE(2) DP2_ROT_CASE(3) DP2_ROT_CASE(4) DP2_ROT_CASE(5) DP2_ROT_CASE(6)
    DP2_ROT_CASE(7) DP2_ROT_CASE(8) DP2_ROT_CASE(9) DP2_ROT_CASE(10) DP2_ROT_CASE(11) DP2_ROT_CASE(12)
    DP2_ROT_CASE(13) DP2_ROT_CASE(14) DP2_ROT_CASE(15) DP2_ROT_CASE(16)
#undef DP2_ROT_CASE
    default: break;
  }
}

AlsLayout als_layout(int64_t K, int64_t J, int R) {
  AlsLayout L{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
  const size_t RR = (size_t)R * R * 8, nb = total_warps(K, R) / wpb_for(R), nbm = metric_blocks(K, R);
  L.theta = take(K * RR);
  L.pprev = take(K * RR);
  L.cc = take(RR);
  L.nh = take(R * 8);
  L.HtH = take(RR);
  L.VtV = take(RR);
  L.pinv3 = take(RR);
  L.G1 = take(RR);
  L.WtW = take(RR);
  L.summed = take(RR);
  L.WtW2 = take(RR);
  L.L = take(K * RR * 2);
  int wr = 0, nr = 0;
  rot_cfg(K, R, wr, nr);
  size_t ns = nr > (int)nb ? (size_t)nr : nb;
  if (rot_ns(R) && ns < 2 * (size_t)sm_count()) ns = 2 * (size_t)sm_count();  // als_rotate_ns_kernel slots
  L.s_g1 = take(ns * RR);
  L.s_wtw = take(ns * RR);
  L.s_m2 = take(nb * RR);
  L.s_wtw2 = take(nb * RR);
  L.s_e = take(nbm * 8);
  L.G2 = take(J * R * 8);
  L.g3 = take(K * R * 8);
  const size_t ps_cap = (size_t)sm_count() * PS_CAP_PER_SM;
  L.GD = take(RR);
  L.ps_slots = take(ps_cap * 2 * RR);
  L.ps_e = take(ps_cap * 8);
  L.ps_C = take(RR);
  L.ps_stamps = take(64 * 16 * 8);
  L.ps_gslots = take(64 * 2 * RR);
  L.ps_gcnt = take(64 * 4);
  L.pwarm = take(3 * (RR + 64));
  {  // R > 16: R^3 buffers and the split-K partials of the mode-2 stack products
    const size_t r3 = (size_t)R * R * R * 8;
    const int sp = std::max(gemm_tn_splits(K, (int64_t)R * R, R), gemm_tn_splits(K, R, R));
    const size_t nnp = (size_t)gemm_nn_splits(K, (int64_t)R * R, R) * K * R * 8;
    L.t3 = take(R > 16 ? r3 : 8);
    L.zz = take(R > 16 ? r3 : 8);
    L.gp = take(R > 16 ? std::max((size_t)sp * r3, nnp) : 8);
  }
  L.ctl = take(64);
  L.total = off;
  return L;
}

AlsBufs make_bufs(char* ws, int64_t K, int64_t J, int R) {
  const AlsLayout L = als_layout(K, J, R);
  AlsBufs b{};
  auto d = [&](size_t o) { return reinterpret_cast<double*>(ws + o); };
  b.theta = d(L.theta);
  b.pprev = d(L.pprev);
  b.cc = d(L.cc);
  b.nh = d(L.nh);
  b.HtH = d(L.HtH);
  b.VtV = d(L.VtV);
  b.pinv3 = d(L.pinv3);
  b.G1 = d(L.G1);
  b.WtW = d(L.WtW);
  b.summed = d(L.summed);
  b.WtW2 = d(L.WtW2);
  b.L = d(L.L);
  b.s_g1 = d(L.s_g1);
  b.s_wtw = d(L.s_wtw);
  b.s_m2 = d(L.s_m2);
  b.s_wtw2 = d(L.s_wtw2);
  b.s_e = d(L.s_e);
  b.G2 = d(L.G2);
  b.g3 = d(L.g3);
  b.GD = d(L.GD);
  b.ps_slots = d(L.ps_slots);
  b.ps_e = d(L.ps_e);
  b.ps_C = d(L.ps_C);
  b.ps_stamps = reinterpret_cast<int64_t*>(ws + L.ps_stamps);
  b.ps_gslots = d(L.ps_gslots);
  b.ps_gcnt = reinterpret_cast<unsigned*>(ws + L.ps_gcnt);
  b.pwarm = d(L.pwarm);
  b.t3 = d(L.t3);
  b.zz = d(L.zz);
  b.gp = d(L.gp);
  b.ctl = reinterpret_cast<int32_t*>(ws + L.ctl);
  b.nwt = total_warps(K, R);
  b.wpb = wpb_for(R);
  b.nb = b.nwt / b.wpb;
  b.nbm = metric_blocks(K, R);
  rot_cfg(K, R, b.wpbr, b.nbr);
  if (b.nbr <= 0) { b.nbr = b.nb; b.wpbr = b.wpb; }
  if (rot_ns(R)) {  // als_rotate_ns_kernel: two CTAs per SM, CTA-strided slices
    const int64_t cap = 2 * (int64_t)sm_count();
    b.nbr = (int)(K < cap ? K : cap);
    b.wpbr = 8;
  }
  return b;
}

size_t acc2_smem(int R, int wpb) { return (cta_shared_doubles(R) + wpb * 3 * (size_t)R * R) * 8; }
size_t mode3_smem(int R, int wpb) { return (cta_shared_doubles(R) + wpb * ((size_t)R * R + 2 * (size_t)R)) * 8; }
size_t solve_smem(int R) { return (7 * (size_t)R * R + 3 * (R / 2 + 1) + 8) * 8; }
// solve_v: + EP (R x R) + D, V (J x R each) when they fit in shared memory
bool solve_v_dsm(int64_t J, int R) { return (solve_smem(R) + ((size_t)R * R + 2 * (size_t)J * R) * 8) <= 200 * 1024; }
size_t solve_v_smem(int64_t J, int R) {  // EP, then D and V, or two solve_v_jt(R)-row chunks of them
  return solve_smem(R) + ((size_t)R * R + (solve_v_dsm(J, R) ? 2 * (size_t)J * R : 2 * (size_t)solve_v_jt(R) * R)) * 8;
}

cudaError_t set_smem(const void* f, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    char buf[96];
    snprintf(buf, sizeof(buf), "dynamic smem attribute %zu bytes", bytes);
    note_error(buf);
    (void)cudaGetLastError();  // reported here: do not leave it for later launch checks
  }
  return e;
}

template <int KS>
void metric_t(const AlsBufs& b, const double* D, const double* V, int64_t J, int R, int64_t K, cudaStream_t st) {
  als_metric_kernel<KS><<<b.nbm, 256, 0, st>>>(b, D, V, J, R, K * R);
}

cudaError_t launch_metric(const AlsBufs& b, const double* D, const double* V, int64_t J, int R, int64_t K,
                          cudaStream_t st) {
  const int ks = (2 * R + 3) / 4;
  if (ks <= 1) metric_t<1>(b, D, V, J, R, K, st);
  else if (ks <= 2) metric_t<2>(b, D, V, J, R, K, st);
  else if (ks <= 3) metric_t<3>(b, D, V, J, R, K, st);
  else if (ks <= 4) metric_t<4>(b, D, V, J, R, K, st);
  else if (ks <= 5) metric_t<5>(b, D, V, J, R, K, st);
  else if (ks <= 6) metric_t<6>(b, D, V, J, R, K, st);
  else if (ks <= 8) metric_t<8>(b, D, V, J, R, K, st);
  else if (ks <= 10) metric_t<10>(b, D, V, J, R, K, st);
  else if (ks <= 12) metric_t<12>(b, D, V, J, R, K, st);
  else if (ks <= 16) metric_t<16>(b, D, V, J, R, K, st);
  else if (ks <= 24) metric_t<24>(b, D, V, J, R, K, st);
  else metric_t<32>(b, D, V, J, R, K, st);
  return cudaGetLastError();
}

template <int R>
size_t rot_group_smem(int wpbr) { return ((size_t)2 * R * R + (size_t)wpbr * grp_per_warp<R>() * grp_doubles<R>()) * 8; }

template <int R>
cudaError_t rotate_t(const SliceArgs& a, const AlsBufs& b, cudaStream_t st, bool setattr) {
  const size_t sm = rot_group_smem<R>(b.wpbr);
  if (setattr) return set_smem((const void*)als_rotate_group_kernel<R>, sm);
  als_rotate_group_kernel<R><<<b.nbr, 32 * b.wpbr, sm, st>>>(a, b, b.wpbr);
  return cudaGetLastError();
}

// rotation step: compile-time-R lane-group kernel for R <= 16, else generic
cudaError_t launch_rotate(const SliceArgs& a, const AlsBufs& b, cudaStream_t st, bool setattr = false) {
  switch (a.R) {
#define DP2_ROT_CASE(N) \
  case N: return rotate_t<N>(a, b, st, setattr);
    DP2_ROT_CASE(1) DP2_ROT_CASE(2) DP2_ROT_CASE(3) DP2_ROT_CASE(4) DP2_ROT_CASE(5) DP2_ROT_CASE(6)
    DP2_ROT_CASE(7) DP2_ROT_CASE(8) DP2_ROT_CASE(9) DP2_ROT_CASE(10) DP2_ROT_CASE(11) DP2_ROT_CASE(12)
    DP2_ROT_CASE(13) DP2_ROT_CASE(14) DP2_ROT_CASE(15) DP2_ROT_CASE(16)
#undef DP2_ROT_CASE
    default:
      if (rot_ns(a.R)) {  // CTA Newton-Schulz on the fp64 tensor pipe (Jacobi fallback)
        const size_t smc = rotate_ns_doubles(a.R) * 8;
        const void* f = nullptr;
        switch (ns_np(a.R)) {
          case 24: f = (const void*)als_rotate_ns_kernel<24>; break;
          case 32: f = (const void*)als_rotate_ns_kernel<32>; break;
          case 40: f = (const void*)als_rotate_ns_kernel<40>; break;
          case 48: f = (const void*)als_rotate_ns_kernel<48>; break;
          default: f = (const void*)als_rotate_ns_kernel<56>; break;
        }
        if (setattr) return set_smem(f, smc);
        void* args[] = {(void*)&a, (void*)&b};
        return cudaLaunchKernel(f, dim3(b.nbr), dim3(256), args, smc, st);
      }
      note_error("rank above the device limit of 56");
      return cudaErrorInvalidValue;
  }
}

cudaError_t prepare(int R, const AlsBufs& b) {
  cudaError_t e = set_smem((const void*)als_mode2_kernel, acc2_smem(R, b.wpb));
  if (e == cudaSuccess) e = set_smem((const void*)als_mode1_kernel, acc2_smem(R, b.wpb));
  if (e == cudaSuccess) e = set_smem((const void*)als_mode3_kernel, mode3_smem(R, b.wpb));
  if (e == cudaSuccess) e = set_smem((const void*)als_solve_h_kernel, solve_smem(R));
  if (e == cudaSuccess) e = set_smem((const void*)als_solve_v_kernel, 225 * 1024);  // + static smem <= 227 KB
  if (e == cudaSuccess) {
    SliceArgs a{};
    a.R = R;
    e = launch_rotate(a, b, nullptr, true);
  }
  return e;
}

cudaError_t launch_iteration(const SliceArgs& base, const SolveArgs& sv, const AlsBufs& b, int it, double tol,
                             double* trace, int64_t* tstamp, int32_t* iters, cudaStream_t st) {
  const int R = base.R, nt = 32 * b.wpb;
  SliceArgs a = base;
  a.mode1 = 1;
  a.warm = 1;
  cudaError_t e0 = launch_rotate(a, b, st);
  if (e0 != cudaSuccess) return e0;
  SolveArgs s1 = sv;  // slots pre-reduced into slot 0 on n/32 CTAs
  const int RR = R * R, gx = (RR + 31) / 32;
  reduce_slots_kernel<<<dim3(gx, 2), 256, 0, st>>>(b.ctl, b.s_g1, b.s_wtw, sv.nslots_h, RR);
  s1.nslots_h = 1;
  als_solve_h_kernel<<<1, 512, solve_smem(R), st>>>(s1, b);
  const bool gemm = R > 16;  // modes 2 / 3 on the stack GEMMs (als_m2_finish_kernel)
  if (gemm) {
    cudaError_t eg = run_gemm_tn(a.theta, a.K, (int64_t)RR, a.W, R, b.t3, st, b.gp);
    if (eg == cudaSuccess) eg = run_gemm_tn(a.W, a.K, R, a.W, R, b.zz, st, b.gp);
    if (eg != cudaSuccess) return eg;
    als_m2_finish_kernel<<<(RR + 255) / 256, 256, 0, st>>>(b.ctl, b.t3, b.zz, a.H, b.nh, R, b.s_m2, b.s_wtw2);
  } else {
    als_mode2_kernel<<<b.nb, nt, acc2_smem(R, b.wpb), st>>>(a, b);
    reduce_slots_kernel<<<dim3(gx, 2), 256, 0, st>>>(b.ctl, b.s_m2, b.s_wtw2, sv.nslots, RR);
  }
  s1.nslots = 1;
  als_solve_v_kernel<<<1, 512, solve_v_smem(sv.J, R), st>>>(s1, b);
  a.write_w = 1;
  a.write_l = 1;
  a.Wout = sv.W;
  if (gemm) {
    als_z_kernel<<<(RR * R + 255) / 256, 256, 0, st>>>(b.ctl, a.H, b.cc, R, b.zz);
    cudaError_t eg = run_gemm_nn(a.theta, a.K, (int64_t)RR, b.zz, R, b.g3, st, b.gp);
    if (eg != cudaSuccess) return eg;
    a.g3_in = b.g3;
  }
  als_mode3_kernel<<<b.nb, nt, mode3_smem(R, b.wpb), st>>>(a, b);
  cudaError_t e = launch_metric(b, a.D, sv.V, a.J, R, a.K, st);
  if (e != cudaSuccess) return e;
  als_finish_kernel<<<1, 32, 0, st>>>(b, it, tol, trace, tstamp, iters);
  return cudaGetLastError();
}

SliceArgs slice_args(const double* F, const double* D, const double* E, const double* H, const double* V,
                     const double* W, int64_t K, int64_t J, int R, int64_t* status) {
  SliceArgs a{};
  a.F = F;
  a.D = D;
  a.E = E;
  a.H = H;
  a.V = V;
  a.W = W;
  a.K = K;
  a.J = J;
  a.R = R;
  a.status = status;
  return a;
}

SolveArgs solve_args(const double* D, const double* E, double* H, double* V, double* W, int64_t J, int R,
                     int normalize, const AlsBufs& b, int64_t* status) {
  SolveArgs sv{};
  sv.D = D;
  sv.E = E;
  sv.H = H;
  sv.V = V;
  sv.W = W;
  sv.J = J;
  sv.R = R;
  sv.normalize = normalize;
  sv.nslots = b.nb;
  sv.nslots_h = b.nbr;
  sv.dsm = solve_v_dsm(J, R);
  sv.status = status;
  return sv;
}

bool persist_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("DP2_ALS_PERSIST");
    v = (s && s[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

cudaError_t launch_persist(int R, const PsArgs& p, const AlsBufs& b, cudaStream_t st) {
  const int sms = sm_count();
  if (R >= 1 && R <= 4) return launch_persist_a(R, p, b, sms, st);
  if (R <= 8) return launch_persist_b(R, p, b, sms, st);
  if (R <= 12) return launch_persist_c(R, p, b, sms, st);
  if (R <= 16) return launch_persist_d(R, p, b, sms, st);
  if (R == 20) return launch_persist_e(R, p, b, sms, st);
  if (R == 24) return launch_persist_f(R, p, b, sms, st);
  return cudaErrorInvalidValue;
}

}  // namespace

size_t als_bytes(int64_t K, int64_t J, int R) { return als_layout(K, J, R).total; }
// byte offset of the persistent loop's phase stamps inside the workspace (profiling)
size_t als_stamp_offset(int64_t K, int64_t J, int R) { return als_layout(K, J, R).ps_stamps; }

cudaError_t als_run(const double* F, const double* D, const double* E, int64_t K, int64_t J, int R,
                    double* H, double* V, double* W, double* polar, int max_iters, double tol,
                    int normalize, double* trace, int64_t* tstamp, int32_t* iters, int use_graph,
                    char* ws, int64_t* status, cudaStream_t st, int64_t* launches) {
  if (launches) *launches = 1 + 9 * (int64_t)max_iters;
  AlsBufs b = make_bufs(ws, K, J, R);
  SliceArgs a = slice_args(F, D, E, H, V, W, K, J, R, status);
  a.polar = polar;
  a.theta = b.theta;
  SolveArgs sv = solve_args(D, E, H, V, W, J, R, normalize, b, status);
  if (persist_enabled() && (R <= 16 || R == 20 || R == 24)) {  // instantiated ranks (dp2_als_ps*.cu)
    PsArgs p{};
    p.F = F;
    p.D = D;
    p.E = E;
    p.H = H;
    p.V = V;
    p.W = W;
    p.polar = polar;
    p.trace = trace;
    p.tstamp = tstamp;
    p.iters = iters;
    p.K = K;
    p.J = J;
    p.max_iters = max_iters;
    p.normalize = normalize;
    p.tol = tol;
    p.slots = b.ps_slots;
    p.eslots = b.ps_e;
    p.C = b.ps_C;
    p.GD = b.GD;
    p.bar = reinterpret_cast<unsigned*>(b.ctl + 8);
    p.status = status;
    p.gslots = b.ps_gslots;
    p.gcnt = b.ps_gcnt;
    p.stamps = getenv("DP2_ALS_STAMPS") ? reinterpret_cast<int64_t*>(b.ps_stamps) : nullptr;
    als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, tstamp, 1);
    const cudaError_t pe = launch_persist(R, p, b, st);
    if (pe == cudaSuccess) {
      if (launches) *launches = 2;
      return cudaSuccess;
    }
    (void)cudaGetLastError();  // not co-resident here: the multi-kernel loop below
  }
  b.GD = nullptr;
  cudaError_t e = prepare(R, b);
  if (e != cudaSuccess) return e;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, tstamp, 1);
  if (!use_graph) {
    for (int it = 0; it < max_iters; ++it) {
      e = launch_iteration(a, sv, b, it, tol, trace, tstamp, iters, st);
      if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
  }
  // Capture on a private stream (the caller's may be the legacy stream, which
  // cannot capture), then launch the instantiated graph on the caller's stream.
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  cudaStream_t cs;
  e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) { cudaStreamDestroy(cs); return e; }
  for (int it = 0; it < max_iters && e == cudaSuccess; ++it)
    e = launch_iteration(a, sv, b, it, tol, trace, tstamp, iters, cs);
  cudaError_t e2 = cudaStreamEndCapture(cs, &graph);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess) return e;
  if (e2 != cudaSuccess) return e2;
  e = cudaGraphInstantiate(&exec, graph, 0);
  if (e == cudaSuccess) {
    e = cudaGraphLaunch(exec, st);
    cudaGraphExecDestroy(exec);
  }
  cudaGraphDestroy(graph);
  return e;
}

// ------------------------------------------------------------ granular API
cudaError_t als_rotations(const double* F, const double* D, const double* E, int64_t K, int64_t J, int R,
                          const double* H, const double* V, const double* W, double* polar,
                          double* theta, char* ws, int64_t* status, cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R);
  SliceArgs a = slice_args(F, D, E, H, V, W, K, J, R, status);
  a.polar = polar;
  a.theta = theta;
  cudaError_t e = prepare(R, b);
  if (e != cudaSuccess) return e;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  return launch_rotate(a, b, st);
}

cudaError_t als_mttkrp(int mode, const double* theta, const double* D, const double* E, int64_t K,
                       int64_t J, int R, const double* H, const double* V, const double* W, double* out,
                       char* ws, cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R);
  SliceArgs a = slice_args(nullptr, D, E, H, V, W, K, J, R, nullptr);
  a.theta = const_cast<double*>(theta);
  cudaError_t e = prepare(R, b);
  if (e != cudaSuccess) return e;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  const int nt = 32 * b.wpb;
  if (mode == 1) {
    als_mode1_kernel<<<b.nb, nt, acc2_smem(R, b.wpb), st>>>(a, b);
    reduce_parts_dev<<<1, 256, 0, st>>>(b.s_g1, b.nb, (int64_t)R * R, out);
  } else if (mode == 2) {
    als_mode2_kernel<<<b.nb, nt, acc2_smem(R, b.wpb), st>>>(a, b);  // nh == 1 after prep
    reduce_parts_dev<<<1, 256, 0, st>>>(b.s_m2, b.nb, (int64_t)R * R, b.summed);
    g2_kernel<<<(unsigned)((J * R + 255) / 256), 256, 0, st>>>(D, E, b.summed, J, R, out);
  } else {
    a.write_w = 0;
    a.Wout = out;
    als_mode3_kernel<<<b.nb, nt, mode3_smem(R, b.wpb), st>>>(a, b);
  }
  return cudaGetLastError();
}

cudaError_t als_update_factors(const double* theta, const double* D, const double* E, int64_t K,
                               int64_t J, int R, double* H, double* V, double* W, int normalize,
                               char* ws, int64_t* status, cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R);
  SliceArgs a = slice_args(nullptr, D, E, H, V, W, K, J, R, status);
  a.theta = const_cast<double*>(theta);
  SolveArgs sv = solve_args(D, E, H, V, W, J, R, normalize, b, status);
  cudaError_t e = prepare(R, b);
  if (e != cudaSuccess) return e;
  const int nt = 32 * b.wpb;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  als_mode1_kernel<<<b.nb, nt, acc2_smem(R, b.wpb), st>>>(a, b);
  sv.nslots_h = b.nb;
  als_solve_h_kernel<<<1, 512, solve_smem(R), st>>>(sv, b);
  als_mode2_kernel<<<b.nb, nt, acc2_smem(R, b.wpb), st>>>(a, b);
  als_solve_v_kernel<<<1, 512, solve_v_smem(sv.J, R), st>>>(sv, b);
  a.write_w = 1;
  a.Wout = W;
  als_mode3_kernel<<<b.nb, nt, mode3_smem(R, b.wpb), st>>>(a, b);
  return cudaGetLastError();
}

cudaError_t als_metric(const double* theta, const double* D, const double* E, int64_t K, int64_t J,
                       int R, const double* H, const double* V, const double* W, double* out, char* ws,
                       cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R);
  SliceArgs a = slice_args(nullptr, D, E, H, V, W, K, J, R, nullptr);
  a.theta = const_cast<double*>(theta);
  a.write_w = 0;
  a.write_l = 1;
  a.Wout = nullptr;
  cudaError_t e = prepare(R, b);
  if (e != cudaSuccess) return e;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  als_mode3_kernel<<<b.nb, 32 * b.wpb, mode3_smem(R, b.wpb), st>>>(a, b);
  e = launch_metric(b, D, V, J, R, K, st);
  if (e != cudaSuccess) return e;
  reduce_parts_dev<<<1, 32, 0, st>>>(b.s_e, b.nbm, 1, out);
  return cudaGetLastError();
}

}  // namespace dp2

namespace dp2 {
// ------------------------------------------------------------ phase API (multi-GPU)
// One ALS iteration split at its three reduction points so that the caller can
// allreduce the R x R partials across GPUs between phases:
//   0 prep | 1 rotate -> red_out = [G1 | W'W] | 2 solve_h(red_in)
//   3 mode2 -> red_out = [summed | W''W''] | 4 solve_v(red_in)
//   5 mode3 + metric -> red_out[0] = e_local | 6 finish(red_in[0])
cudaError_t als_phase(int phase, const double* F, const double* D, const double* E, int64_t K, int64_t J, int R,
                      double* H, double* V, double* W, double* polar, int it, double tol, int normalize,
                      double* trace, int64_t* tstamp, int32_t* iters, const double* red_in, double* red_out,
                      char* ws, int64_t* status, cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R);
  SliceArgs a = slice_args(F, D, E, H, V, W, K, J, R, status);
  a.polar = polar;
  a.theta = b.theta;
  SolveArgs sv = solve_args(D, E, H, V, W, J, R, normalize, b, status);
  const int nt = 32 * b.wpb;
  const size_t RR = (size_t)R * R;
  cudaError_t e = cudaSuccess;
  switch (phase) {
    case 0:
      e = prepare(R, b);
      if (e != cudaSuccess) return e;
      als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, tstamp, 1);
      break;
    case 1:
      a.mode1 = 1;
      a.warm = 1;
      e = launch_rotate(a, b, st);
      if (e != cudaSuccess) return e;
      reduce_parts_dev<<<1, 256, 0, st>>>(b.s_g1, b.nbr, (int64_t)RR, red_out);
      reduce_parts_dev<<<1, 256, 0, st>>>(b.s_wtw, b.nbr, (int64_t)RR, red_out + RR);
      break;
    case 2:
      cudaMemcpyAsync(b.s_g1, red_in, RR * 8, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(b.s_wtw, red_in + RR, RR * 8, cudaMemcpyDeviceToDevice, st);
      sv.nslots_h = 1;
      als_solve_h_kernel<<<1, 512, solve_smem(R), st>>>(sv, b);
      break;
    case 3:
      als_mode2_kernel<<<b.nb, nt, acc2_smem(R, b.wpb), st>>>(a, b);
      reduce_parts_dev<<<1, 256, 0, st>>>(b.s_m2, b.nb, (int64_t)RR, red_out);
      reduce_parts_dev<<<1, 256, 0, st>>>(b.s_wtw2, b.nb, (int64_t)RR, red_out + RR);
      break;
    case 4:
      cudaMemcpyAsync(b.s_m2, red_in, RR * 8, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(b.s_wtw2, red_in + RR, RR * 8, cudaMemcpyDeviceToDevice, st);
      sv.nslots = 1;
      als_solve_v_kernel<<<1, 512, solve_v_smem(sv.J, R), st>>>(sv, b);
      break;
    case 5:
      a.write_w = 1;
      a.write_l = 1;
      a.Wout = W;
      als_mode3_kernel<<<b.nb, nt, mode3_smem(R, b.wpb), st>>>(a, b);
      e = launch_metric(b, D, V, J, R, K, st);
      if (e != cudaSuccess) return e;
      reduce_parts_dev<<<1, 32, 0, st>>>(b.s_e, b.nbm, 1, red_out);
      break;
    case 6: {
      cudaMemcpyAsync(b.s_e, red_in, 8, cudaMemcpyDeviceToDevice, st);
      AlsBufs b1 = b;
      b1.nbm = 1;
      als_finish_kernel<<<1, 32, 0, st>>>(b1, it, tol, trace, tstamp, iters);
      break;
    }
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
}  // namespace dp2
