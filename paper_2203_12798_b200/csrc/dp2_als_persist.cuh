// Persistent ALS loop (included by dp2_als.cu inside namespace dp2).
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

constexpr int PS_CAP_PER_SM = 2;  // grid cap (partial slots are sized for it)

template <int R>
struct PsCfg {
  static constexpr int RR = R * R, LDT = R | 1;
  static constexpr int WPB = R <= 12 ? 16 : 8;  // warps per CTA
  // per-warp shared layout (doubles)
  static constexpr int FS = 0, TH = RR, T = 2 * RR, US = 3 * RR, VS = 4 * RR, PI = 5 * RR, ACC1 = 6 * RR,
                       ACC2 = 7 * RR, TS = 8 * RR, VR = TS + R * LDT, TMP = VR + R * LDT, WTOT = TMP + 8 * R;
  // per-CTA shared layout (doubles)
  static constexpr int CC = 0, H = RR, VTV = 2 * RR, HTH = 3 * RR, C = 4 * RR, P3 = 5 * RR, GD = 6 * RR,
                       RED = 7 * RR /* 2 RR */, M = 9 * RR, U = 10 * RR, PV = 11 * RR, X = 12 * RR, Y = 13 * RR,
                       E = 14 * RR, NH = E + R, NRM = NH + R, CS = NRM + R, WE = CS + 3 * (R / 2 + 1) + 8,
                       CTOT = WE + 32;
  static constexpr size_t smem_bytes() { return ((size_t)CTOT + (size_t)WPB * WTOT) * 8; }
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
};

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
template <int N, int WPB>
DP2_DEV void ps_reduce_slots(const double* slots, int nblk, double* wscr, int wstride, double* out) {
  constexpr int NE = (N + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
#pragma unroll
    for (int w = 0; w < WPB; ++w) s += wscr[w * wstride + e];
    out[e] = s;
  }
  __syncthreads();
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

// One-sided Jacobi (Hestenes) on the columns held by lanes 0..R-1: a = column
// of A = T V, v = column of V.  Round-robin pairing (R-1 or R rounds per
// sweep); both lanes of a pair compute bitwise-identical (alpha, beta, gamma)
// -- fma(x, y, z) is symmetric in x, y -- so they apply the same rotation.
// Returns the sweeps used (cap + 1 when not converged).
template <int R>
DP2_DEV int jacobi_reg(double (&a)[R], double (&v)[R]) {
  constexpr int N = R + (R & 1);
  constexpr int CAP = 40;
  constexpr double TOL = 4.0 * R * 2.220446049250313e-16;
  const int lane = threadIdx.x & 31;
  for (int sw = 0; sw < CAP; ++sw) {
    bool rot = false;
    for (int r = 0; r < N - 1; ++r) {
      int p;
      if (lane >= N) p = lane;
      else if (lane == N - 1) p = r;
      else if (lane == r) p = N - 1;
      else p = (2 * r - lane + 2 * (N - 1)) % (N - 1);
      double pa[R], pv[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        pa[i] = __shfl_sync(0xffffffffu, a[i], p);
        pv[i] = __shfl_sync(0xffffffffu, v[i], p);
      }
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        al = fma(a[i], a[i], al);
        be = fma(pa[i], pa[i], be);
        ga = fma(a[i], pa[i], ga);
      }
      const bool lower = lane < p;
      const double alpha = lower ? al : be, beta = lower ? be : al;
      if (p != lane && fabs(ga) > TOL * sqrt(alpha * beta)) {
        const double zeta = (beta - alpha) / (2.0 * ga);
        const double az = fabs(zeta);
        const double t = az > 1e100 ? 0.5 / zeta : copysign(1.0, zeta) / (az + sqrt(fma(zeta, zeta, 1.0)));
        const double c = 1.0 / sqrt(fma(t, t, 1.0)), s = c * t;
        const double so = lower ? -s : s;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          a[i] = fma(c, a[i], so * pa[i]);
          v[i] = fma(c, v[i], so * pv[i]);
        }
        rot = true;
      }
    }
    if (!__any_sync(0xffffffffu, rot)) return sw + 1;
  }
  return CAP + 1;
}

// polar factor of T (row-major, per-warp smem) -> Pi; V of T's SVD -> Vs
// (warm start in: Vs holds the previous V or I).  Singular T (an exactly zero
// singular value) or a non-converged sweep falls back to warp_polar's
// orthonormal completion.
template <int R>
DP2_DEV void ps_polar(double* w, int64_t k, int64_t* status) {
  using Cf = PsCfg<R>;
  constexpr int RR = R * R, LDT = Cf::LDT;
  const int lane = threadIdx.x & 31;
  double* T = w + Cf::T;
  double* Us = w + Cf::US;
  double* Vs = w + Cf::VS;
  double* Pi = w + Cf::PI;
  wmm<R, false, false>(T, Vs, Us);  // A = T V_warm
  double a[R], v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    a[i] = lane < R ? Us[i * R + lane] : 0.0;
    v[i] = lane < R ? Vs[i * R + lane] : 0.0;
  }
  const int sw = jacobi_reg<R>(a, v);
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i) s2 = fma(a[i], a[i], s2);
  const double sig = sqrt(s2);
  const bool bad = lane < R && !(sig > 1e-300 && sig < 1e300);
  __syncwarp();
  if (__any_sync(0xffffffffu, bad) || sw > 40) {
    double* Ts = w + Cf::TS;
    double* Vr = w + Cf::VR;
    for (int e = lane; e < RR; e += 32) {
      const int i = e / R, c = e % R;
      Ts[c * LDT + i] = T[e];
      Vr[c * LDT + i] = (i == c) ? 1.0 : 0.0;
    }
    __syncwarp();
    warp_polar(Ts, Vr, LDT, R, Pi, w + Cf::TMP, status, k);
    for (int e = lane; e < RR; e += 32) Vs[e] = (e / R == e % R) ? 1.0 : 0.0;  // next warm start: cold
    __syncwarp();
    return;
  }
  const double inv = 1.0 / sig;
  if (lane < R) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      Us[i * R + lane] = a[i] * inv;
      Vs[i * R + lane] = v[i];
    }
  }
  __syncwarp();
  wmm<R, false, true>(Us, Vs, Pi);  // Pi = U V^T
}

template <int R>
__global__ void __launch_bounds__(PsCfg<R>::WPB * 32, 1) als_persist_kernel(PsArgs p, AlsBufs b) {
  using Cf = PsCfg<R>;
  constexpr int RR = R * R, WPB = Cf::WPB;
  extern __shared__ __align__(16) double sm[];
  double* cs = sm;
  double* w = sm + Cf::CTOT + (size_t)(threadIdx.x >> 5) * Cf::WTOT;
  double* wscr = sm + Cf::CTOT + Cf::ACC1;  // per-warp 2RR scratch (acc1|acc2) for the slot reductions
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nblk = gridDim.x;
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
  double prev_e = 0.0;
  int it = 0;
  for (; it < p.max_iters; ++it) {
    // ---------------- rotate + mode-1 partials
    double* acc1 = w + Cf::ACC1;
    double* acc2 = w + Cf::ACC2;
    for (int e = lane; e < RR; e += 32) { acc1[e] = 0.0; acc2[e] = 0.0; }
    for (int64_t k = gw; k < p.K; k += nw) {
      double* Fs = w + Cf::FS;
      double* Th = w + Cf::TH;
      double* T = w + Cf::T;
      double* Vs = w + Cf::VS;
      double* Pi = w + Cf::PI;
      const double* wk = p.W + k * R;
      for (int e = lane; e < RR; e += 32) {
        Fs[e] = __ldg(p.F + k * RR + e);
        Vs[e] = it > 0 ? __ldcg(b.pprev + k * RR + e) : ((e / R == e % R) ? 1.0 : 0.0);
      }
      double wr[R];
#pragma unroll
      for (int r = 0; r < R; ++r) wr[r] = __ldcg(wk + r);
      __syncwarp();
      wmm<R, false, false>(Fs, cc, Th);  // Th = F_k cc
      for (int e = lane; e < RR; e += 32) {
        double s = Th[e];
#pragma unroll
        for (int r = 0; r < R; ++r) s = (e % R == r) ? s * wr[r] : s;
        Th[e] = s;
      }
      __syncwarp();
      wmm<R, false, true>(Th, Hs, T);  // T = Th H^T
      ps_polar<R>(w, k, p.status);
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
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * RR; e += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < WPB; ++q) s += sm[Cf::CTOT + (size_t)q * Cf::WTOT + Cf::ACC1 + e];
      p.slots[(size_t)blockIdx.x * 2 * RR + e] = s;
    }
    ps_grid_barrier(p.bar, bar_target);
    // ---------------- solve_h (every CTA)
    ps_reduce_slots<2 * RR, WPB>(p.slots, nblk, wscr, Cf::WTOT, red);  // red = [G1 | W'W]
    for (int e = threadIdx.x; e < RR; e += blockDim.x) M[e] = red[RR + e] * VtV[e];
    __syncthreads();
    block_pinv_sym(M, U, Pv, R, csc, p.status);
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
    ps_grid_barrier(p.bar, bar_target);
    // ---------------- solve_v (every CTA), V = D C implicit
    ps_reduce_slots<2 * RR, WPB>(p.slots, nblk, wscr, Cf::WTOT, red);  // red = [summed | W''W'']
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
      M[e] = red[RR + e] * HtH[e];
      Y[e] = Es[e / R] * red[e];  // E * summed
    }
    __syncthreads();
    block_pinv_sym(M, U, Pv, R, csc, p.status);
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
    block_pinv_sym(M, U, P3, R, csc, p.status);
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
