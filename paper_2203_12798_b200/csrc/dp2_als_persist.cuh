// Persistent ALS loop: kernel template and launcher (instantiated for R = 1..16,
// 20 and 24 in dp2_als_ps{a..f}.cu, dispatched from dp2_als.cu).
//
// The whole iteration loop of P/solver.py:152-184 in ONE cooperative launch:
// every CTA is resident, slices are owned by warps (warp w of the grid handles
// slices w, w + nwarps, ...), and an iteration is three slice phases separated
// by grid barriers, each followed by the R x R solve that the reference does
// between its sweeps -- computed REDUNDANTLY by every CTA from the ordered
// reduction of the per-CTA partial slots, so no CTA waits for a broadcast:
//
//   rotate  (warp/slice) T_k = (F_k cc) diag(w_k) H^T, polar Pi_k = Z_k P_k^T
//           (P/solver.py:54-60), Theta_k = Pi_k^T F_k, mode-1 + gram(W) partials
//   --- barrier ---  solve_h: H = G1 pinv(W'W * V'V), column norms (P/solver.py:88-97)
//   mode2   (warp/slice) sum_k (w_k nh) (Theta_k^T H), gram(W nh) partials
//   --- barrier ---  solve_v: V = D (E * summed) pinv(W'W * H'H), norms (:99-107)
//   mode3   (warp/slice) W_k = G3_k pinv(V'V * H'H) (:109-115) and the slice's
//           residual e_k = ||Theta_k E D^T - H S_k V^T||_F^2 (:117-124)
//   --- barrier ---  e = ordered sum, trace, device stop rule (:180-184)
//
// V is kept implicit: after the first V update V = D C exactly (C = R x R), so
// with G_D = D^T D (prep) every quantity the loop needs is R x R:
//   D^T V = G_D C,  V^T V = C^T G_D C,  ||V[:,c]||^2 = (C^T G_D C)[c][c],
//   e_k = tr(Delta_k G_D Delta_k^T),  Delta_k = Theta_k diag(E) - H S_k C^T,
// exact for any D (no orthonormality assumed) and J-independent; V itself is
// formed once, after the loop.  The polar factor is a one-sided Jacobi SVD
// held in registers (lane j owns column j), warm-started from the previous
// iteration's right singular vectors of the same slice.

#pragma once
#include "dp2_als_dev.cuh"
#include <cstdlib>

namespace dp2 {

constexpr int PS_CAP_PER_SM = 2;  // grid cap (partial slots are sized for it)

template <int R>
struct PsCfg {
  static constexpr int RR = R * R, LDT = R | 1;
  static constexpr int N = R + (R & 1);  // Jacobi columns (a zero column pads odd R)
  static constexpr int MAXW = 8;         // warps per CTA (upper bound; 255 registers)
  // per-warp shared layout (doubles)
  static constexpr int FS = 0, T = RR, US = 2 * RR, VS = 3 * RR, TH = 4 * RR, PI = 5 * RR, ACC1 = 6 * RR,
                       ACC2 = 7 * RR, TS = 8 * RR, VR = TS + R * LDT, TMP = VR + R * LDT, WTOT = TMP + 8 * R;
  // per-CTA shared layout (doubles)
  static constexpr int CC = 0, H = RR, VTV = 2 * RR, HTH = 3 * RR, C = 4 * RR, P3 = 5 * RR, GD = 6 * RR,
                       RED = 7 * RR /* 2 RR */, M = 9 * RR, U = 10 * RR, PV = 11 * RR, X = 12 * RR, Y = 13 * RR,
                       E = 14 * RR, NH = E + R, NRM = NH + R, CS = NRM + R, WE = CS + 3 * (R / 2 + 1) + 8,
                       CTOT = WE + 32;
  static constexpr size_t smem_bytes(int wpb) { return ((size_t)CTOT + (size_t)wpb * WTOT) * 8; }
};

struct PsArgs {
  const double *F, *D, *E;
  double *H, *V, *W, *polar;
  double *trace;
  int64_t* tstamp;
  int32_t* iters;
  int64_t K, J;
  int max_iters, normalize;
  double tol;
  double *slots, *eslots, *C, *GD;
  unsigned* bar;
  int64_t* status;
  double* gslots;    // per-group partial slots (<= 64 groups)
  unsigned* gcnt;    // per-group arrival counters (zeroed by the prep kernel)
  int64_t* stamps;  // optional (DP2_ALS_STAMPS=1): CTA 0's globaltimer at phase boundaries, 16 per iteration
};

#define PS_STAMP(slot)                                                                    \
  do {                                                                                    \
    if (p.stamps && blockIdx.x == 0 && threadIdx.x == 0 && it < 64)                       \
      p.stamps[it * 16 + (slot)] = (int64_t)globaltimer_ns();                              \
  } while (0)

DP2_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier for a co-resident (cooperative) grid: monotone arrival
// counter, reset to 0 by the prep kernel before the launch.
DP2_DEV void ps_grid_barrier(unsigned* bar, unsigned& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    while ((int)(ld_acquire_u32(bar) - target) < 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

// Ordered reduction of the grid's per-CTA slots (nblk x N) into out[N], done
// by every CTA: warp w sums a fixed contiguous block range for all entries
// (L2 loads, the slots were written by other SMs), then the warps' partials
// combine in warp order.  Deterministic for a given grid size.
template <int N>
DP2_DEV void ps_reduce_slots(const double* slots, int nblk, double* wscr, int wstride, double* out) {
  constexpr int NE = (N + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, WPB = blockDim.x >> 5;
  const int per = (nblk + WPB - 1) / WPB, b0 = warp * per, b1 = min(nblk, b0 + per);
  double v[NE];
#pragma unroll
  for (int u = 0; u < NE; ++u) v[u] = 0.0;
#pragma unroll 2
  for (int b = b0; b < b1; ++b)
#pragma unroll
    for (int u = 0; u < NE; ++u) {
      const int e = lane + 32 * u;
      if (e < N) v[u] += __ldcg(slots + (size_t)b * N + e);
    }
#pragma unroll
  for (int u = 0; u < NE; ++u) {
    const int e = lane + 32 * u;
    if (e < N) wscr[warp * wstride + e] = v[u];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < WPB; ++w) s += wscr[w * wstride + e];
    out[e] = s;
  }
  __syncthreads();
}

// Two-level ordered reduction, level 1: CTAs form groups of ~sqrt(nblk);
// after writing its slot each CTA arrives on its group's counter and the
// group's last arrival folds the group's slots (in CTA order) into the group
// slot before entering the grid barrier.  Level 2 (after the barrier) is then
// a reduction over <= ~sqrt(nblk) group slots instead of nblk CTA slots.
DP2_DEV int ps_group_size(int nblk) {
  int g = 1;
  while (g * g < nblk) ++g;
  return g;
}

template <int N>
DP2_DEV void ps_group_fold(const double* slots, double* gslots, unsigned* gcnt, double* wscr, int wstride) {
  __shared__ int last;
  const int nblk = gridDim.x, GS = ps_group_size(nblk), grp = blockIdx.x / GS;
  const int gsz = min(GS, nblk - grp * GS);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned old = atomicAdd(gcnt + grp, 1u);
    last = ((old + 1) % (unsigned)gsz) == 0;
    if (last) __threadfence();
  }
  __syncthreads();
  if (last) ps_reduce_slots<N>(slots + (size_t)grp * GS * N, gsz, wscr, wstride, gslots + (size_t)grp * N);
}

// C = op(A) op(B) for R x R row-major matrices, all threads of the CTA
template <int R, bool TA, bool TB>
DP2_DEV void cta_mm(const double* A, const double* B, double* C) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e % R;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) s = fma(TA ? A[q * R + i] : A[i * R + q], TB ? B[j * R + q] : B[q * R + j], s);
    C[e] = s;
  }
  __syncthreads();
}

// Polar factor Jacobi: jacobi_cols (dp2_common.cuh) with V accumulated and
// the loose stop (largest relative off-diagonal of the last sweep < 1e-4, so
// ~1e-8 remains: the polar factor enters the next ALS update, whose own
// rounding and the 1e-5 / 1e-6 parity bounds are far above that).
template <int R>
DP2_DEV int jacobi_reg(double (&a)[R], double (&v)[R]) {
  return jacobi_cols<R, true, true>(a, v);
}

template <int R>
__global__ void __launch_bounds__(PsCfg<R>::MAXW * 32, 1) als_persist_kernel(PsArgs p, AlsBufs b) {
  using Cf = PsCfg<R>;
  constexpr int RR = R * R, LDT = Cf::LDT;
  extern __shared__ __align__(16) double sm[];
  double* cs = sm;
  double* w = sm + Cf::CTOT + (size_t)(threadIdx.x >> 5) * Cf::WTOT;
  double* wscr = sm + Cf::CTOT + Cf::ACC1;  // per-warp 2RR scratch (acc1|acc2) for the slot reductions
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, WPB = blockDim.x >> 5;
  const int nblk = gridDim.x, ngrp = (nblk + ps_group_size(nblk) - 1) / ps_group_size(nblk);
  const int64_t gw = (int64_t)blockIdx.x * WPB + wib, nw = (int64_t)nblk * WPB;
  unsigned bar_target = 0;
  double* cc = cs + Cf::CC;
  double* Hs = cs + Cf::H;
  double* VtV = cs + Cf::VTV;
  double* HtH = cs + Cf::HTH;
  double* Cm = cs + Cf::C;
  double* P3 = cs + Cf::P3;
  double* GD = cs + Cf::GD;
  double* red = cs + Cf::RED;
  double* M = cs + Cf::M;
  double* U = cs + Cf::U;
  double* Pv = cs + Cf::PV;
  double* X = cs + Cf::X;
  double* Y = cs + Cf::Y;
  double* Es = cs + Cf::E;
  double* nh = cs + Cf::NH;
  double* nrm = cs + Cf::NRM;
  double* csc = cs + Cf::CS;
  double* we = cs + Cf::WE;
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    cc[e] = b.cc[e];
    Hs[e] = p.H[e];
    VtV[e] = b.VtV[e];
    GD[e] = p.GD[e];
  }
  for (int e = threadIdx.x; e < R; e += blockDim.x) {
    Es[e] = p.E[e];
    nh[e] = 1.0;
  }
  __syncthreads();
  __shared__ int vfast;  // the V solve's pinv was done during barrier 2
  if (threadIdx.x == 0) vfast = 0;
  double prev_e = 0.0;
  int it = 0;
  for (; it < p.max_iters; ++it) {
    PS_STAMP(0);
    // ---------------- rotate + mode-1 partials: G slices of this warp per Jacobi
    double* acc1 = w + Cf::ACC1;
    double* acc2 = w + Cf::ACC2;
    double* Th = w + Cf::TH;
    double* Pi = w + Cf::PI;
    for (int e = lane; e < RR; e += 32) { acc1[e] = 0.0; acc2[e] = 0.0; }
    for (int64_t k = gw; k < p.K; k += nw) {
      const long long dq0 = clock64();  // profiling (stamps only)
      double* Fs = w + Cf::FS;
      double* T = w + Cf::T;
      double* Us = w + Cf::US;
      double* Vs = w + Cf::VS;
      for (int e = lane; e < RR; e += 32) {
        Fs[e] = __ldg(p.F + k * RR + e);
        Vs[e] = it > 0 ? __ldcg(b.pprev + k * RR + e) : ((e / R == e % R) ? 1.0 : 0.0);
      }
      double wr[R];
#pragma unroll
      for (int r = 0; r < R; ++r) wr[r] = __ldcg(p.W + k * R + r);
      __syncwarp();
      wmm<R, false, false>(Fs, cc, Th);  // Th = F_k cc
      for (int e = lane; e < RR; e += 32) {
        double s = Th[e];
#pragma unroll
        for (int r = 0; r < R; ++r) s = (e % R == r) ? s * wr[r] : s;
        Th[e] = s;
      }
      __syncwarp();
      wmm<R, false, true>(Th, Hs, T);   // T = Th H^T
      wmm<R, false, false>(T, Vs, Us);  // A = T V_warm
      const long long dq1 = clock64();
      int sw32 = 0;
      // polar factor: one-sided Jacobi SVD of A in registers, mixed precision:
      // fp32 sweeps to ~1e-5, V re-orthonormalised in fp64 (one Newton-Schulz
      // step, V <- V (3I - V^T V) / 2), then fp64 sweeps from there (their
      // first sweep sees off-diagonals near fp32's floor, so the loose stop
      // ends it after one sweep with ~1e-12 left)
      {
        float af[R], vf[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          af[i] = lane < R ? (float)Us[i * R + lane] : 0.f;
          vf[i] = lane < R ? (float)Vs[i * R + lane] : 0.f;
        }
        sw32 = jacobi_cols_f32<R>(af, vf, 12);
        bool fin = true;
#pragma unroll
        for (int i = 0; i < R; ++i) fin &= isfinite(vf[i]);
        if (__all_sync(0xffffffffu, fin)) {  // else: keep V_warm
          __syncwarp();
          if (lane < R)
#pragma unroll
            for (int i = 0; i < R; ++i) Vs[i * R + lane] = (double)vf[i];
          __syncwarp();
          wmm<R, true, false>(Vs, Vs, Us);  // V^T V
          for (int e = lane; e < RR; e += 32) Us[e] = ((e / R == e % R) ? 1.5 : 0.0) - 0.5 * Us[e];
          __syncwarp();
          wmm<R, false, false>(Vs, Us, Pi);  // V (3I - V^T V) / 2
          for (int e = lane; e < RR; e += 32) Vs[e] = Pi[e];
          __syncwarp();
          wmm<R, false, false>(T, Vs, Us);  // A = T V
        }
      }
      double a[R], v[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        a[i] = lane < R ? Us[i * R + lane] : 0.0;
        v[i] = lane < R ? Vs[i * R + lane] : 0.0;
      }
      const int sw = jacobi_reg<R>(a, v);
      const long long dq2 = clock64();
      double s2 = 0.0;
#pragma unroll
      for (int i = 0; i < R; ++i) s2 = fma(a[i], a[i], s2);
      const double sig = sqrt(s2);
      const bool bad = lane < R && !(sig > 1e-300 && sig < 1e300);
      __syncwarp();
      if (__any_sync(0xffffffffu, bad) || sw > 40) {
        // singular T (or no convergence): one-sided Jacobi with orthonormal completion
        double* Ts = w + Cf::TS;
        double* Vr = w + Cf::VR;
        for (int e = lane; e < RR; e += 32) {
          const int i = e / R, c = e % R;
          Ts[c * LDT + i] = T[e];
          Vr[c * LDT + i] = (i == c) ? 1.0 : 0.0;
        }
        __syncwarp();
        warp_polar(Ts, Vr, LDT, R, Pi, w + Cf::TMP, p.status, k);
        for (int e = lane; e < RR; e += 32) Vs[e] = (e / R == e % R) ? 1.0 : 0.0;  // next warm start: cold
        __syncwarp();
      } else {
        if (lane < R) {
          const double inv = 1.0 / sig;
#pragma unroll
          for (int i = 0; i < R; ++i) {
            Us[i * R + lane] = a[i] * inv;
            Vs[i * R + lane] = v[i];
          }
        }
        __syncwarp();
        wmm<R, false, true>(Us, Vs, Pi);  // Pi = U V^T
      }
      for (int e = lane; e < RR; e += 32) {
        b.pprev[k * RR + e] = Vs[e];
        p.polar[k * RR + e] = Pi[e];
      }
      wmm<R, true, false>(Pi, Fs, Th);  // Theta = Pi^T F
      for (int e = lane; e < RR; e += 32) {
        b.theta[k * RR + e] = Th[e];
        const int i = e / R, r = e % R;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) s = fma(Th[i * R + q], cc[q * R + r], s);
        double wi = 0.0, wrr = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          wi = (q == i) ? wr[q] : wi;
          wrr = (q == r) ? wr[q] : wrr;
        }
        acc1[e] += wrr * s;
        acc2[e] += wi * wrr;
      }
      __syncwarp();
      if (p.stamps && lane == 0 && it < 64) {  // per-warp maxima: setup, Jacobi, epilogue cycles, sweeps, total
        unsigned long long* q = reinterpret_cast<unsigned long long*>(p.stamps + it * 16);
        const long long dq3 = clock64();
        atomicMax(q + 11, (unsigned long long)(dq1 - dq0));
        atomicMax(q + 12, (unsigned long long)(dq2 - dq1));
        atomicMax(q + 13, (unsigned long long)(dq3 - dq2));
        atomicMax(q + 14, (unsigned long long)(sw32 * 100 + sw));
        atomicMax(q + 15, (unsigned long long)(dq3 - dq0));
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * RR; e += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < WPB; ++q) s += sm[Cf::CTOT + (size_t)q * Cf::WTOT + Cf::ACC1 + e];
      p.slots[(size_t)blockIdx.x * 2 * RR + e] = s;
    }
    ps_group_fold<2 * RR>(p.slots, p.gslots, p.gcnt, wscr, Cf::WTOT);
    PS_STAMP(1);
    ps_grid_barrier(p.bar, bar_target);
    PS_STAMP(2);
    // ---------------- solve_h (every CTA)
    ps_reduce_slots<2 * RR>(p.gslots, ngrp, wscr, Cf::WTOT, red);  // red = [G1 | W'W]
    PS_STAMP(8);
    for (int e = threadIdx.x; e < RR; e += blockDim.x) M[e] = red[RR + e] * VtV[e];
    __syncthreads();
    block_pinv_sym<R>(M, U, Pv, R, csc, p.status);
    PS_STAMP(9);
    cta_mm<R, false, false>(red, Pv, X);  // Hn = G1 pinv
    for (int c = threadIdx.x; c < R; c += blockDim.x) {
      double n2 = 0.0;
      for (int i = 0; i < R; ++i) n2 = fma(X[i * R + c], X[i * R + c], n2);
      const double n = sqrt(n2);
      nrm[c] = (p.normalize && !(n < 1e-300)) ? n : 1.0;
      nh[c] = nrm[c];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
      Hs[e] = X[e] / nrm[e % R];
      if (blockIdx.x == 0) p.H[e] = Hs[e];
    }
    __syncthreads();
    cta_mm<R, true, false>(Hs, Hs, HtH);
    PS_STAMP(3);
    // ---------------- mode-2 partials
    for (int e = lane; e < RR; e += 32) { acc1[e] = 0.0; acc2[e] = 0.0; }
    for (int64_t k = gw; k < p.K; k += nw) {
      double* Th = w + Cf::TH;
      for (int e = lane; e < RR; e += 32) Th[e] = __ldcg(b.theta + k * RR + e);
      double wr[R];
#pragma unroll
      for (int r = 0; r < R; ++r) wr[r] = __ldcg(p.W + k * R + r) * nh[r];
      __syncwarp();
      for (int e = lane; e < RR; e += 32) {
        const int ai = e / R, r = e % R;
        double s = 0.0;  // (Theta^T H)[ai][r]
#pragma unroll
        for (int q = 0; q < R; ++q) s = fma(Th[q * R + ai], Hs[q * R + r], s);
        double wa = 0.0, wrr = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          wa = (q == ai) ? wr[q] : wa;
          wrr = (q == r) ? wr[q] : wrr;
        }
        acc1[e] += wrr * s;
        acc2[e] += wa * wrr;
      }
      __syncwarp();
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * RR; e += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < WPB; ++q) s += sm[Cf::CTOT + (size_t)q * Cf::WTOT + Cf::ACC1 + e];
      p.slots[(size_t)blockIdx.x * 2 * RR + e] = s;
    }
    ps_group_fold<2 * RR>(p.slots, p.gslots, p.gcnt, wscr, Cf::WTOT);
    PS_STAMP(4);
    // grid barrier 2, with the V solve's pinv computed while thread 0 waits:
    // its matrix (W''^T W'') o (H^T H) is known before the barrier -- W'' =
    // W diag(nh), and W^T W came with solve_h's reduction (red[RR..], intact
    // until this barrier's reduction).  Warp 1 (warp 0 with one warp) runs
    // the register Gauss-Jordan; if it declines, solve_v takes the usual path.
    __syncthreads();
    if (threadIdx.x == 0) {
      bar_target += gridDim.x;
      __threadfence();
      atomicAdd(p.bar, 1u);
    }
    if constexpr (R >= 2 && R <= 16) {
      if (wib == (WPB > 1 ? 1 : 0)) {
        for (int e = lane; e < RR; e += 32) M[e] = (red[RR + e] * nh[e / R]) * nh[e % R] * HtH[e];
        __syncwarp();
        const bool okk = warp_gj_inverse<R>(M, Pv);
        if (lane == 0) vfast = okk ? 1 : 0;
      }
    }
    if (threadIdx.x == 0) {
      while ((int)(ld_acquire_u32(p.bar) - bar_target) < 0) {
      }
      __threadfence();
    }
    __syncthreads();
    PS_STAMP(5);
    // ---------------- solve_v (every CTA), V = D C implicit
    ps_reduce_slots<2 * RR>(p.gslots, ngrp, wscr, Cf::WTOT, red);  // red = [summed | W''W'']
    PS_STAMP(10);
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
      if (!vfast) M[e] = red[RR + e] * HtH[e];
      Y[e] = Es[e / R] * red[e];  // E * summed
    }
    __syncthreads();
    if (!vfast) block_pinv_sym<R>(M, U, Pv, R, csc, p.status);
    cta_mm<R, false, false>(Y, Pv, X);   // EP = (E * summed) pinv
    cta_mm<R, false, false>(GD, X, Y);   // G_D EP
    for (int c = threadIdx.x; c < R; c += blockDim.x) {
      double n2 = 0.0;  // ||D EP[:,c]||^2 = (EP^T G_D EP)[c][c]
      for (int i = 0; i < R; ++i) n2 = fma(X[i * R + c], Y[i * R + c], n2);
      const double n = sqrt(fmax(n2, 0.0));
      nrm[c] = (p.normalize && !(n < 1e-300)) ? n : 1.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
      const double inv = 1.0 / nrm[e % R];
      Cm[e] = X[e] * inv;                 // C
      cc[e] = Es[e / R] * (Y[e] * inv);   // E * (D^T V) = E * (G_D C)
      if (blockIdx.x == 0) p.C[e] = Cm[e];
    }
    __syncthreads();
    cta_mm<R, false, false>(GD, Cm, Y);   // G_D C
    cta_mm<R, true, false>(Cm, Y, VtV);   // V^T V = C^T G_D C
    for (int e = threadIdx.x; e < RR; e += blockDim.x) M[e] = VtV[e] * HtH[e];
    __syncthreads();
    block_pinv_sym<R>(M, U, P3, R, csc, p.status);
    PS_STAMP(6);
    // ---------------- mode-3: W_k and the residual
    double eacc = 0.0;
    for (int64_t k = gw; k < p.K; k += nw) {
      double* Th = w + Cf::TH;
      double* Dl = w + Cf::T;   // Delta_k
      double* DG = w + Cf::US;  // Delta_k G_D
      for (int e = lane; e < RR; e += 32) Th[e] = __ldcg(b.theta + k * RR + e);
      __syncwarp();
      // G3[r] = sum_i H[i][r] sum_j Theta[i][j] cc[j][r]; lane r
      double g3 = 0.0;
      if (lane < R) {
        for (int i = 0; i < R; ++i) {
          double h = 0.0;
#pragma unroll
          for (int j = 0; j < R; ++j) h = fma(Th[i * R + j], cc[j * R + lane], h);
          g3 = fma(Hs[i * R + lane], h, g3);
        }
      }
      double wn[R];
#pragma unroll
      for (int r = 0; r < R; ++r) wn[r] = __shfl_sync(0xffffffffu, g3, r);
      // W_k[c] = sum_r G3[r] pinv3[r][c]; lane c (all lanes need all of W_k)
      double wc[R];
#pragma unroll
      for (int c = 0; c < R; ++c) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) s = fma(wn[r], P3[r * R + c], s);
        wc[c] = s;
      }
      if (lane < R) {
        double mine = 0.0;
#pragma unroll
        for (int c = 0; c < R; ++c) mine = (c == lane) ? wc[c] : mine;
        p.W[k * R + lane] = mine;
      }
      // Delta[i][j] = Theta[i][j] E[j] - sum_r H[i][r] W_k[r] C[j][r]
      for (int e = lane; e < RR; e += 32) {
        const int i = e / R, j = e % R;
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) s = fma(Hs[i * R + r] * wc[r], Cm[j * R + r], s);
        Dl[e] = Th[e] * Es[j] - s;
      }
      __syncwarp();
      wmm<R, false, false>(Dl, GD, DG);
      for (int e = lane; e < RR; e += 32) eacc = fma(Dl[e], DG[e], eacc);
      __syncwarp();
    }
    eacc = warp_sum(eacc);
    if (lane == 0) we[wib] = eacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < WPB; ++q) s += we[q];
      p.eslots[blockIdx.x] = s;
    }
    PS_STAMP(7);
    ps_grid_barrier(p.bar, bar_target);
    // ---------------- e, trace, stop rule (every CTA, identical decision)
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int q = lane; q < nblk; q += 32) s += __ldcg(p.eslots + q);
      s = warp_sum(s);
      if (lane == 0) we[WPB] = s;
    }
    __syncthreads();
    const double e = we[WPB];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.trace[it] = e;
      if (p.tstamp) p.tstamp[it + 1] = (int64_t)globaltimer_ns();
      *p.iters = it + 1;
    }
    const bool stop = it > 0 && (prev_e == 0.0 || fabs(prev_e - e) <= p.tol * prev_e);
    prev_e = e;
    __syncthreads();
    if (stop) break;
  }
  // V = D C, rows split over the grid
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < p.J * R;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / R;
    const int r = (int)(idx - j * R);
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) s = fma(p.D[j * R + q], Cm[q * R + r], s);
    p.V[idx] = s;
  }
}

// Grid shape: one slice per warp (the rotation is latency-bound per warp),
// the K warps spread over all SMs, at most MAXW warps and the smem budget per
// CTA; larger K loops each warp over several slices.
template <int R>
cudaError_t launch_persist_t(const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st) {
  using Cf = PsCfg<R>;
  const void* fn = (const void*)als_persist_kernel<R>;
  int maxw = Cf::MAXW;
  while (maxw > 1 && Cf::smem_bytes(maxw) > 220 * 1024) --maxw;
  const int64_t warps = p.K;
  int wpb = (int)((warps + sms - 1) / sms);
  if (const char* env = getenv("DP2_ALS_WPB")) wpb = atoi(env);
  wpb = wpb < 1 ? 1 : (wpb > maxw ? maxw : wpb);
  const size_t smem = Cf::smem_bytes(wpb);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, wpb * 32, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorCooperativeLaunchTooLarge;
  const int64_t cap = (int64_t)sms * (occ < PS_CAP_PER_SM ? occ : PS_CAP_PER_SM);
  int64_t grid = (warps + wpb - 1) / wpb;
  grid = grid < cap ? grid : cap;
  PsArgs pa = p;
  AlsBufs ba = b;
  void* args[] = {&pa, &ba};
  return cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(wpb * 32), args, smem, st);
}

// one per translation unit (R ranges 1-4, 5-8, 9-12, 13-16)
cudaError_t launch_persist_a(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st);
cudaError_t launch_persist_b(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st);
cudaError_t launch_persist_c(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st);
cudaError_t launch_persist_d(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st);
cudaError_t launch_persist_e(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st);
cudaError_t launch_persist_f(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st);


}  // namespace dp2
