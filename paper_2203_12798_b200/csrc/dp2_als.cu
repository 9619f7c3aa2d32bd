// Compressed-space ALS (P/solver.py:39-190), fp64.
//
// One iteration = 6 launches, all stream-ordered and graph-capturable:
//   rotate   (warp/slice) T_k = (F_k cc) diag(w_k) H^T, polar Pi_k = Z_k P_k^T
//            (one-sided Jacobi), Theta_k = Pi_k^T F_k, mode-1 + gram(W) partials
//   solve_h  (1 CTA)      H = G1 pinv(W'W * V'V), column norms -> nh
//   mode2    (warp/slice) sum_k (w_k nh) (Theta_k^T H), gram(W nh) partials
//   solve_v  (1 CTA)      V = D (E * summed) pinv(...), norms, V'V, cc', pinv3
//   mode3    (warp/slice) G3 row, W_k = G3_k pinv3, metric e_k
//   finish   (1 warp)     e = sum of partials (fixed order), trace, stop rule
// Partials live in per-warp slots (each warp owns a slot and visits a fixed
// slice set), reduced in slot order: deterministic for a given device.
// Every kernel returns at once when the device stop flag is set, so the whole
// max_iters loop can be one CUDA graph with no host round trip
// (P/solver.py:180-184 evaluated on the device).
#include "dp2_common.cuh"
#include "dp2_internal.h"

namespace dp2 {

struct AlsBufs {
  double *theta, *cc, *nh, *HtH, *VtV, *pinv3, *G1, *WtW, *summed, *WtW2;
  double *p_g1, *p_wtw, *p_m2, *p_wtw2, *p_e, *scratch, *g3;
  int32_t* ctl;  // [0] stop flag
  int nwt;       // total warps (partial slots)
  int wpb;       // warps per block
};

__host__ __device__ inline int wpb_for(int R) { return R <= 16 ? 8 : (R <= 32 ? 4 : 1); }
__host__ __device__ inline int ldt_for(int R) { return R | 1; }
__host__ __device__ inline size_t warp_smem_doubles(int R) {
  const int ldt = ldt_for(R);
  return (size_t)2 * R * ldt + 3 * (size_t)R * R + 4 * R;
}

DP2_DEV double globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return (double)t;
}

// ------------------------------------------------------------ common loads
// Per-CTA shared: cc (R x R), H (R x R), E (R), aux (R x R), vec (R)
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
__host__ __device__ inline size_t cta_shared_doubles(int R) { return 3 * (size_t)R * R + 2 * R; }

// ------------------------------------------------------------ polar factor
// Pi = Z P^T of T (R x R) via one-sided Jacobi; exact-zero singular directions
// are completed to an orthonormal set (LAPACK returns some such completion).
// Ts, Vr: column-major (ldt); out: Pi row-major into ``pi``.
DP2_DEV void warp_polar(double* Ts, double* Vr, int ldt, int R, double* pi, double* nrm, int64_t* status,
                        int64_t k) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < R * ldt; e += 32) Vr[e] = ((e % ldt) == (e / ldt)) ? 1.0 : 0.0;
  __syncwarp();
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
  // Pi[a][d] = sum_i Z[a][i] P[d][i]   (Z = Ts columns, P = Vr columns)
  for (int e = lane; e < R * R; e += 32) {
    const int a = e / R, d = e % R;
    double s = 0.0;
    for (int i = 0; i < R; ++i) s = fma(Ts[i * ldt + a], Vr[i * ldt + d], s);
    pi[e] = s;
  }
  __syncwarp();
}

// ------------------------------------------------------------ small helpers
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

// cc = E * (D^T V) and VtV = V^T V with one warp per entry (no block barriers)
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

// ------------------------------------------------------------ prep / finish
// cc = E * (D^T V), VtV = V^T V, stop = 0, tstamp[0]
__global__ void als_prep_kernel(const double* D, const double* E, const double* V, int64_t J, int R,
                                AlsBufs b, int64_t* tstamp, int reset) {
  gram_dv_warps(D, E, V, J, R, b.cc, b.VtV, nullptr, nullptr);
  if (threadIdx.x == 0) {
    for (int r = 0; r < R; ++r) b.nh[r] = 1.0;
    if (reset) b.ctl[0] = 0;
    if (tstamp) tstamp[0] = (int64_t)globaltimer_ns();
  }
}

__global__ void als_finish_kernel(AlsBufs b, int it, double tol, double* trace, int64_t* tstamp,
                                  int32_t* iters) {
  if (b.ctl[0]) return;
  if (threadIdx.x != 0) return;
  double e = 0.0;
  for (int w = 0; w < b.nwt; ++w) e += b.p_e[w];
  trace[it] = e;
  if (tstamp) tstamp[it + 1] = (int64_t)globaltimer_ns();
  *iters = it + 1;
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
  int metric;     // mode3: also emit metric partials
  int write_w;    // mode3: W_k = G3_k pinv3 (else write G3 into Wout)
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

// accumulate an R x R block into this warp's global slot (first visit writes)
DP2_DEV void slot_add(double* slot, int e, double v, bool first) { slot[e] = first ? v : slot[e] + v; }

__global__ void als_rotate_kernel(SliceArgs a, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, ldt = ldt_for(R), lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CtaShared cs = carve_cta(sm, R);
  double* wbase = sm + cta_shared_doubles(R) + (size_t)wib * warp_smem_doubles(R);
  double* Ts = wbase;
  double* Vr = Ts + R * ldt;
  double* Fs = Vr + R * ldt;
  double* Th = Fs + R * R;
  double* Pi = Th + R * R;
  double* tmp = Pi + R * R;  // 4R
  load_cta_common(a, b, cs, true, false);
  const int gw = blockIdx.x * b.wpb + wib;
  bool first = true;
  for (int64_t k = gw; k < a.K; k += b.nwt) {
    const double* Fk = a.F + k * R * R;
    const double* wk = a.W + k * R;
    for (int e = lane; e < R * R; e += 32) Fs[e] = Fk[e];
    __syncwarp();
    // Th <- (F_k cc) * w_k   (reference: (core_block(k) @ core_cols) * w[k])
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, c = e % R;
      double s = 0.0;
      for (int q = 0; q < R; ++q) s = fma(Fs[i * R + q], cs.cc[q * R + c], s);
      Th[e] = s * wk[c];
    }
    __syncwarp();
    // T = Th H^T, stored column-major in Ts
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, d = e % R;
      double s = 0.0;
      for (int c = 0; c < R; ++c) s = fma(Th[i * R + c], cs.H[d * R + c], s);
      Ts[d * ldt + i] = s;
    }
    __syncwarp();
    warp_polar(Ts, Vr, ldt, R, Pi, tmp, a.status, k);
    // Theta = Pi^T F
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, c = e % R;
      double s = 0.0;
      for (int d = 0; d < R; ++d) s = fma(Pi[d * R + i], Fs[d * R + c], s);
      Th[e] = s;
      a.theta[k * R * R + e] = s;
      if (a.polar) a.polar[k * R * R + e] = Pi[e];
    }
    __syncwarp();
    if (a.mode1) {
      // g1[i][r] += w[k][r] * (Theta cc)[i][r];  wtw[i][r] += w[k][i] w[k][r]
      double* sg = b.p_g1 + (size_t)gw * R * R;
      double* sw = b.p_wtw + (size_t)gw * R * R;
      for (int e = lane; e < R * R; e += 32) {
        const int i = e / R, r = e % R;
        double s = 0.0;
        for (int q = 0; q < R; ++q) s = fma(Th[i * R + q], cs.cc[q * R + r], s);
        slot_add(sg, e, wk[r] * s, first);
        slot_add(sw, e, wk[i] * wk[r], first);
      }
    }
    first = false;
    __syncwarp();
  }
  if (a.mode1 && first) {  // warp had no slice: zero its slots
    for (int e = lane; e < R * R; e += 32) {
      b.p_g1[(size_t)gw * R * R + e] = 0.0;
      b.p_wtw[(size_t)gw * R * R + e] = 0.0;
    }
  }
}

// mode-1 partials from a given Theta stack (kernel-granular API)
__global__ void als_mode1_kernel(SliceArgs a, AlsBufs b) {
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CtaShared cs = carve_cta(sm, R);
  load_cta_common(a, b, cs, false, false);
  const int gw = blockIdx.x * b.wpb + wib;
  double* sg = b.p_g1 + (size_t)gw * R * R;
  double* sw = b.p_wtw + (size_t)gw * R * R;
  for (int e = lane; e < R * R; e += 32) { sg[e] = 0.0; sw[e] = 0.0; }
  for (int64_t k = gw; k < a.K; k += b.nwt) {
    const double* Th = a.theta + k * R * R;
    const double* wk = a.W + k * R;
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, r = e % R;
      double s = 0.0;
      for (int q = 0; q < R; ++q) s = fma(Th[i * R + q], cs.cc[q * R + r], s);
      sg[e] += wk[r] * s;
      sw[e] += wk[i] * wk[r];
    }
  }
}

__global__ void als_mode2_kernel(SliceArgs a, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CtaShared cs = carve_cta(sm, R);
  load_cta_common(a, b, cs, true, false);
  const int gw = blockIdx.x * b.wpb + wib;
  double* sm2 = b.p_m2 + (size_t)gw * R * R;
  double* sw2 = b.p_wtw2 + (size_t)gw * R * R;
  for (int e = lane; e < R * R; e += 32) { sm2[e] = 0.0; sw2[e] = 0.0; }
  for (int64_t k = gw; k < a.K; k += b.nwt) {
    const double* Th = a.theta + k * R * R;
    const double* wk = a.W + k * R;
    for (int e = lane; e < R * R; e += 32) {
      const int ai = e / R, r = e % R;
      double s = 0.0;  // (Theta^T H)[ai][r]
      for (int q = 0; q < R; ++q) s = fma(Th[q * R + ai], cs.H[q * R + r], s);
      const double wr = wk[r] * cs.vec[r], wa = wk[ai] * cs.vec[ai];
      sm2[e] += wr * s;
      sw2[e] += wa * wr;
    }
  }
}

template <int RT>
__global__ void als_mode3_kernel(SliceArgs a, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CtaShared cs = carve_cta(sm, R);
  load_cta_common(a, b, cs, true, a.write_w != 0);
  double* L = sm + cta_shared_doubles(R) + (size_t)wib * (2 * (size_t)R * R + 2 * R);  // R x 2R
  double* g3 = L + 2 * R * R;
  double* wn = g3 + R;
  const int gw = blockIdx.x * b.wpb + wib;
  double esum = 0.0;
  for (int64_t k = gw; k < a.K; k += b.nwt) {
    const double* Th = a.theta + k * R * R;
    // G3[r] = sum_i H[i][r] sum_j Theta[i][j] cc[j][r]
    for (int r = lane; r < R; r += 32) {
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
      a.Wout[k * R + c] = s;
    }
    __syncwarp();
    if (a.metric) {
      // L = [Theta * E | -(H * w_k)];  e_k = sum_j sum_i (L [D_j; V_j])_i^2
      const double* wk = a.write_w ? wn : a.W + k * R;
      for (int e = lane; e < 2 * R * R; e += 32) {
        const int i = e / (2 * R), c = e % (2 * R);
        L[e] = c < R ? Th[i * R + c] * cs.E[c] : -(cs.H[i * R + (c - R)] * wk[c - R]);
      }
      __syncwarp();
      for (int64_t j = lane; j < a.J; j += 32) {
        double dv[2 * RT];
#pragma unroll
        for (int c = 0; c < RT; ++c) {
          dv[c] = c < R ? a.D[j * R + c] : 0.0;
          dv[RT + c] = c < R ? a.V[j * R + c] : 0.0;
        }
        for (int i = 0; i < R; ++i) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < RT; ++c)
            if (c < R) s = fma(L[i * 2 * R + c], dv[c], s);
#pragma unroll
          for (int c = 0; c < RT; ++c)
            if (c < R) s = fma(L[i * 2 * R + R + c], dv[RT + c], s);
          esum = fma(s, s, esum);
        }
      }
      __syncwarp();
    }
  }
  if (a.metric) {
    esum = warp_sum(esum);
    if (lane == 0) b.p_e[gw] = esum;
  }
}

// ------------------------------------------------------------ solves (1 CTA)
// pinv of a symmetric R x R matrix (P/linalg.py:135-151 on a Hadamard of
// Grams): eigen-decomposition, |lambda| <= R * max|lambda| * 1e-12 dropped.
DP2_DEV void block_pinv_sym(double* A, double* U, double* out, int R, double* cs, int* flag, int64_t* status) {
  const int sw = jacobi_eig_block(A, R, U, R, R, cs, flag);
  if (sw > 40 && threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(status + ST_SWEEPCAP), 1ull);
  __shared__ double lmax;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < R; ++i) m = fmax(m, fabs(A[i * R + i]));
    lmax = m;
  }
  __syncthreads();
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

DP2_DEV void reduce_slots(const double* slots, int nslots, int n, double* out) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nslots; ++w) s += slots[(size_t)w * n + e];
    out[e] = s;
  }
}

struct SolveArgs {
  const double *D, *E;
  double *H, *V, *W;
  int64_t J;
  int R, normalize, nslots;
  int64_t* status;
  double* G2;  // J x R scratch
};

__global__ void als_solve_h_kernel(SolveArgs s, AlsBufs b) {
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
  __shared__ int flag;
  reduce_slots(b.p_g1, s.nslots, R * R, G1);
  reduce_slots(b.p_wtw, s.nslots, R * R, WtW);
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    Mh[e] = WtW[e] * b.VtV[e];
    b.G1[e] = G1[e];
    b.WtW[e] = WtW[e];
  }
  __syncthreads();
  block_pinv_sym(Mh, U, Pv, R, cs, &flag, s.status);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, c = e % R;
    double acc = 0.0;
    for (int q = 0; q < R; ++q) acc = fma(G1[i * R + q], Pv[q * R + c], acc);
    Hn[e] = acc;
  }
  __syncthreads();
  __shared__ double nrm[64];
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

__global__ void als_solve_v_kernel(SolveArgs s, AlsBufs b) {
  if (b.ctl[0]) return;
  extern __shared__ __align__(16) double sm[];
  const int R = s.R;
  const int64_t J = s.J;
  double* summed = sm;
  double* WtW2 = summed + R * R;
  double* Mv = WtW2 + R * R;
  double* U = Mv + R * R;
  double* Pv = U + R * R;
  double* es = Pv + R * R;  // R*R: E * summed
  double* cs = es + R * R;
  __shared__ int flag;
  __shared__ double nrm[64];
  reduce_slots(b.p_m2, s.nslots, R * R, summed);
  reduce_slots(b.p_wtw2, s.nslots, R * R, WtW2);
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    Mv[e] = WtW2[e] * b.HtH[e];
    es[e] = s.E[e / R] * summed[e];
    b.summed[e] = summed[e];
    b.WtW2[e] = WtW2[e];
  }
  __syncthreads();
  block_pinv_sym(Mv, U, Pv, R, cs, &flag, s.status);
  // G2 = D (E * summed);  V = G2 pinv
  for (int64_t e = threadIdx.x; e < J * R; e += blockDim.x) {
    const int64_t j = e / R;
    const int r = (int)(e % R);
    double acc = 0.0;
    for (int a = 0; a < R; ++a) acc = fma(s.D[j * R + a], es[a * R + r], acc);
    s.G2[e] = acc;
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < J * R; e += blockDim.x) {
    const int64_t j = e / R;
    const int r = (int)(e % R);
    double acc = 0.0;
    for (int a = 0; a < R; ++a) acc = fma(s.G2[j * R + a], Pv[a * R + r], acc);
    s.V[e] = acc;
  }
  __syncthreads();
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c = warp; c < R; c += nw) {
      double part = 0.0;
      for (int64_t j = lane; j < J; j += 32) part = fma(s.V[j * R + c], s.V[j * R + c], part);
      const double n = sqrt(warp_sum(part));
      if (lane == 0) nrm[c] = (s.normalize && !(n < 1e-300)) ? n : 1.0;
    }
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < J * R; e += blockDim.x) s.V[e] = s.V[e] / nrm[e % R];
  __syncthreads();
  gram_dv_warps(s.D, s.E, s.V, J, R, b.cc, b.VtV, Mv, b.HtH);
  __syncthreads();
  block_pinv_sym(Mv, U, b.pinv3, R, cs, &flag, s.status);
}

// ------------------------------------------------------------ host side
namespace {

struct AlsLayout {
  size_t theta, cc, nh, HtH, VtV, pinv3, G1, WtW, summed, WtW2, p_g1, p_wtw, p_m2, p_wtw2, p_e, G2, g3, ctl, total;
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

AlsLayout als_layout(int64_t K, int64_t J, int R) {
  AlsLayout L{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
  const size_t RR = (size_t)R * R * 8, nw = total_warps(K, R);
  L.theta = take(K * RR);
  L.cc = take(RR);
  L.nh = take(R * 8);
  L.HtH = take(RR);
  L.VtV = take(RR);
  L.pinv3 = take(RR);
  L.G1 = take(RR);
  L.WtW = take(RR);
  L.summed = take(RR);
  L.WtW2 = take(RR);
  L.p_g1 = take(nw * RR);
  L.p_wtw = take(nw * RR);
  L.p_m2 = take(nw * RR);
  L.p_wtw2 = take(nw * RR);
  L.p_e = take(nw * 8);
  L.G2 = take(J * R * 8);
  L.g3 = take(K * R * 8);
  L.ctl = take(64);
  L.total = off;
  return L;
}

AlsBufs make_bufs(char* ws, int64_t K, int64_t J, int R, size_t* g2_off) {
  const AlsLayout L = als_layout(K, J, R);
  AlsBufs b{};
  auto d = [&](size_t o) { return reinterpret_cast<double*>(ws + o); };
  b.theta = d(L.theta);
  b.cc = d(L.cc);
  b.nh = d(L.nh);
  b.HtH = d(L.HtH);
  b.VtV = d(L.VtV);
  b.pinv3 = d(L.pinv3);
  b.G1 = d(L.G1);
  b.WtW = d(L.WtW);
  b.summed = d(L.summed);
  b.WtW2 = d(L.WtW2);
  b.p_g1 = d(L.p_g1);
  b.p_wtw = d(L.p_wtw);
  b.p_m2 = d(L.p_m2);
  b.p_wtw2 = d(L.p_wtw2);
  b.p_e = d(L.p_e);
  b.scratch = d(L.G2);
  b.g3 = d(L.g3);
  b.ctl = reinterpret_cast<int32_t*>(ws + L.ctl);
  b.nwt = total_warps(K, R);
  b.wpb = wpb_for(R);
  if (g2_off) *g2_off = L.G2;
  return b;
}

size_t slice_smem(int R, int wpb, bool mode3) {
  const size_t per = mode3 ? (2 * (size_t)R * R + 2 * R) : warp_smem_doubles(R);
  return (cta_shared_doubles(R) + wpb * per) * 8;
}
size_t solve_smem(int R) { return (7 * (size_t)R * R + 3 * (R / 2 + 1) + 8) * 8; }

cudaError_t set_smem(const void* f, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int RT>
cudaError_t launch_mode3_t(const SliceArgs& a, const AlsBufs& b, cudaStream_t st) {
  const size_t sm = slice_smem(a.R, b.wpb, true);
  als_mode3_kernel<RT><<<b.nwt / b.wpb, 32 * b.wpb, sm, st>>>(a, b);
  return cudaGetLastError();
}
cudaError_t launch_mode3(const SliceArgs& a, const AlsBufs& b, cudaStream_t st) {
  if (a.R <= 16) return launch_mode3_t<16>(a, b, st);
  if (a.R <= 32) return launch_mode3_t<32>(a, b, st);
  return launch_mode3_t<64>(a, b, st);
}

cudaError_t launch_iteration(const SliceArgs& base, SolveArgs sv, const AlsBufs& b, int it, double tol,
                             double* trace, int64_t* tstamp, int32_t* iters, cudaStream_t st) {
  const int R = base.R, nb = b.nwt / b.wpb, nt = 32 * b.wpb;
  const size_t rs = slice_smem(R, b.wpb, false);
  SliceArgs a = base;
  a.mode1 = 1;
  als_rotate_kernel<<<nb, nt, rs, st>>>(a, b);
  als_solve_h_kernel<<<1, 256, solve_smem(R), st>>>(sv, b);
  als_mode2_kernel<<<nb, nt, rs, st>>>(a, b);
  als_solve_v_kernel<<<1, 512, solve_smem(R), st>>>(sv, b);
  a.metric = 1;
  a.write_w = 1;
  a.Wout = sv.W;
  cudaError_t e = launch_mode3(a, b, st);
  if (e != cudaSuccess) return e;
  als_finish_kernel<<<1, 32, 0, st>>>(b, it, tol, trace, tstamp, iters);
  return cudaGetLastError();
}

cudaError_t prepare(const SliceArgs& a, const AlsBufs& b, int R) {
  cudaError_t e = set_smem((const void*)als_rotate_kernel, slice_smem(R, b.wpb, false));
  if (e == cudaSuccess) e = set_smem((const void*)als_mode2_kernel, slice_smem(R, b.wpb, false));
  if (e == cudaSuccess) e = set_smem((const void*)als_mode1_kernel, slice_smem(R, b.wpb, false));
  if (e == cudaSuccess) e = set_smem((const void*)als_solve_h_kernel, solve_smem(R));
  if (e == cudaSuccess) e = set_smem((const void*)als_solve_v_kernel, solve_smem(R));
  const size_t m3 = slice_smem(R, b.wpb, true);
  if (e == cudaSuccess) e = set_smem((const void*)als_mode3_kernel<16>, m3);
  if (e == cudaSuccess) e = set_smem((const void*)als_mode3_kernel<32>, m3);
  if (e == cudaSuccess) e = set_smem((const void*)als_mode3_kernel<64>, m3);
  (void)a;
  return e;
}

}  // namespace

size_t als_bytes(int64_t K, int64_t J, int R) { return als_layout(K, J, R).total; }

cudaError_t als_run(const double* F, const double* D, const double* E, int64_t K, int64_t J, int R,
                    double* H, double* V, double* W, double* polar, int max_iters, double tol,
                    int normalize, double* trace, int64_t* tstamp, int32_t* iters, int use_graph,
                    char* ws, int64_t* status, cudaStream_t st) {
  size_t g2off = 0;
  AlsBufs b = make_bufs(ws, K, J, R, &g2off);
  SliceArgs a{};
  a.F = F;
  a.D = D;
  a.E = E;
  a.H = H;
  a.V = V;
  a.W = W;
  a.polar = polar;
  a.theta = b.theta;
  a.K = K;
  a.J = J;
  a.R = R;
  a.status = status;
  SolveArgs sv{};
  sv.D = D;
  sv.E = E;
  sv.H = H;
  sv.V = V;
  sv.W = W;
  sv.J = J;
  sv.R = R;
  sv.normalize = normalize;
  sv.nslots = b.nwt;
  sv.status = status;
  sv.G2 = b.scratch;
  cudaError_t e = prepare(a, b, R);
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
  AlsBufs b = make_bufs(ws, K, J, R, nullptr);
  SliceArgs a{};
  a.F = F; a.D = D; a.E = E; a.H = H; a.V = V; a.W = W;
  a.polar = polar; a.theta = const_cast<double*>(theta); a.K = K; a.J = J; a.R = R; a.status = status;
  cudaError_t e = prepare(a, b, R);
  if (e != cudaSuccess) return e;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  als_rotate_kernel<<<b.nwt / b.wpb, 32 * b.wpb, slice_smem(R, b.wpb, false), st>>>(a, b);
  return cudaGetLastError();
}

cudaError_t als_mttkrp(int mode, const double* theta, const double* D, const double* E, int64_t K,
                       int64_t J, int R, const double* H, const double* V, const double* W, double* out,
                       char* ws, cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R, nullptr);
  SliceArgs a{};
  a.D = D; a.E = E; a.H = H; a.V = V; a.W = W; a.theta = const_cast<double*>(theta); a.K = K; a.J = J; a.R = R;
  cudaError_t e = prepare(a, b, R);
  if (e != cudaSuccess) return e;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  const int nb = b.nwt / b.wpb, nt = 32 * b.wpb;
  const size_t rs = slice_smem(R, b.wpb, false);
  if (mode == 1) {
    als_mode1_kernel<<<nb, nt, rs, st>>>(a, b);
    reduce_parts_dev<<<1, 256, 0, st>>>(b.p_g1, b.nwt, (int64_t)R * R, out);
  } else if (mode == 2) {
    als_mode2_kernel<<<nb, nt, rs, st>>>(a, b);  // nh == 1 after prep
    reduce_parts_dev<<<1, 256, 0, st>>>(b.p_m2, b.nwt, (int64_t)R * R, b.summed);
    // out = D (E * summed)
    g2_kernel<<<(unsigned)((J * R + 255) / 256), 256, 0, st>>>(D, E, b.summed, J, R, out);
  } else {
    a.write_w = 0;
    a.metric = 0;
    a.Wout = out;
    e = launch_mode3(a, b, st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t als_update_factors(const double* theta, const double* D, const double* E, int64_t K,
                               int64_t J, int R, double* H, double* V, double* W, int normalize,
                               char* ws, int64_t* status, cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R, nullptr);
  SliceArgs a{};
  a.D = D; a.E = E; a.H = H; a.V = V; a.W = W; a.theta = const_cast<double*>(theta); a.K = K; a.J = J; a.R = R; a.status = status;
  SolveArgs sv{};
  sv.D = D; sv.E = E; sv.H = H; sv.V = V; sv.W = W; sv.J = J; sv.R = R; sv.normalize = normalize;
  sv.nslots = b.nwt; sv.status = status; sv.G2 = b.scratch;
  cudaError_t e = prepare(a, b, R);
  if (e != cudaSuccess) return e;
  const int nb = b.nwt / b.wpb, nt = 32 * b.wpb;
  const size_t rs = slice_smem(R, b.wpb, false);
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  als_mode1_kernel<<<nb, nt, rs, st>>>(a, b);
  als_solve_h_kernel<<<1, 256, solve_smem(R), st>>>(sv, b);
  als_mode2_kernel<<<nb, nt, rs, st>>>(a, b);
  als_solve_v_kernel<<<1, 512, solve_smem(R), st>>>(sv, b);
  a.write_w = 1;
  a.metric = 0;
  a.Wout = W;
  return launch_mode3(a, b, st);
}

cudaError_t als_metric(const double* theta, const double* D, const double* E, int64_t K, int64_t J,
                       int R, const double* H, const double* V, const double* W, double* out, char* ws,
                       cudaStream_t st) {
  AlsBufs b = make_bufs(ws, K, J, R, nullptr);
  SliceArgs a{};
  a.D = D; a.E = E; a.H = H; a.V = V; a.W = W; a.theta = const_cast<double*>(theta); a.K = K; a.J = J; a.R = R;
  a.metric = 1;
  a.write_w = 0;
  a.Wout = b.g3;
  cudaError_t e = prepare(a, b, R);
  if (e != cudaSuccess) return e;
  als_prep_kernel<<<1, 256, 0, st>>>(D, E, V, J, R, b, nullptr, 1);
  e = launch_mode3(a, b, st);
  if (e != cudaSuccess) return e;
  reduce_parts_dev<<<1, 32, 0, st>>>(b.p_e, b.nwt, 1, out);
  return cudaGetLastError();
}

}  // namespace dp2
