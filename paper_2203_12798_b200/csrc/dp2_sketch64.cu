// Stage-1 streaming sketch pass on the fp64 tensor pipe (DMMA), warp-specialised.
//
// Same contract as the other streaming passes (dp2_stage1.cu run_sketch): for
// every piece p (segment x slice) of the store
//     out_part[p] (J x sp) = X_p^T (X_p B_k)          (P/linalg.py:124-126 fused)
// plus, on request, the Y = X_k B_k rows (y_out) and G_p = Y_p^T Y_p (g_part).
// X is fp64 (the reference's precision) or fp32 (exactly upcast; fp64
// products), B is fp64 (Omega_k or Q_Z,k).
//
// The pass is FP64-compute-bound on B200 (4 s flops per 8 (or 4) bytes of X
// against a measured 36.9 TF/s DMMA peak and 6.5 TB/s HBM), so the design
// goal is to keep the DMMA pipe issuing: every role runs its own loop over
// the CTA's tiles (8 rows) and hands off through mbarriers, never a block-wide
// barrier.
//
//   producer (1 warp)   TMA bulk copies: X rows of tile n into ring stage n % NS
//                       (padded row stride: conflict-free fragment loads), and
//                       per piece the slice's B image (fragment-major, one
//                       bulk copy per A warp share of J).
//   A warps (8)         Y_t (8 x SG) partial over their eighth of J:
//                       DMMA m8n8k4 with B fragments from the shared image
//                       (one accumulator set); partial -> ypart ring.
//   aux (3 warps)       each sums the 8 partials of a third of Y_t's fragments
//                       (rows past the piece zeroed), publishes them in
//                       B-fragment layout (yfin ring), flags non-finite values
//                       (status word 0 = lowest slice: a NaN / Inf anywhere in
//                       X_k reaches Y), writes Y rows.
//   B warps (16 / 8)    Z (J x SG) += X_t^T Y_t for their share of J (a
//                       sixteenth; an eighth when NT = 1), held in registers
//                       across the piece; flushed per piece.  They also
//                       accumulate the 8 x 8 tiles of G = Y^T Y (tile t on B
//                       warp t % NB: Y^T fragments are the B fragments).
// Roles fill whole warpgroups; setmaxnreg moves registers from the A and
// producer / aux groups to the B warps (struct Lay).
//
// Column groups of SG = 8 NT sketch columns run as separate CTAs (grid.y).
// J <= 512: up to 3 column blocks per CTA (B image <= 96 KB + a 3-stage X
// ring in 227 KB); 512 < J <= 1024: one column block per CTA.
#include "dp2_common.cuh"
#include "dp2_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace dp2 {
namespace s64 {

constexpr int TMAX = 16;        // rows per tile: TM = 8 (J > 256 per CTA), 16 (J <= 256)
constexpr int NA = 8;           // warps computing Y partials (split of J): two per SM sub-partition
constexpr int NY = 2;           // ypart / yfin ring depth
// warp w runs on SM sub-partition w % 4: two A warps and NB / 4 B warps per
// sub-partition keep the DMMA work per sub-partition equal.  A lone
// shared-memory-fed DMMA stream reaches only 76% of the pipe rate, two reach
// 95% (tools/dmma_lds_probe.cu), so the A product -- the critical path, which
// runs alone whenever the B warps wait for Y_t -- is spread over two warps per
// sub-partition.  Every role group fills whole warpgroups (4 warps; the last
// one is the producer and the aux warps) so that setmaxnreg can move registers
// from the other groups to the B warps (their Z accumulators).
constexpr int NAUX = 3;         // warps summing the partials into Y_t (a split of its fragments)
constexpr int NMISC = 4;        // producer + aux warps: one warpgroup
constexpr int REGS_A = 64, REGS_MISC = 56;
constexpr int NB_MAX = 16;
// NT sketch column blocks per CTA.  NT >= 2 (J <= 512): 16 B warps (Z rows
// split 16 ways, 24 accumulator doubles each at NT = 3), 28 warps launched at
// 72 registers, B warps raised to 80.  NT = 1 (one column block per CTA: J up
// to 1024): 8 B warps of up to 16 J-blocks (32 accumulator doubles), 20 warps
// launched at 96 registers -- measured on the c5 shard (J = 1000) 34.6 / 34.9
// ms per pass against 37.5 / 37.5 with 16 B warps; at c2 (NT = 3) 8 B warps of
// 48 accumulator doubles made no difference (3.80 / 3.89) and c3 (J = 256)
// slower (19.4 / 20.5 against 18.3 / 19.2).
template <int NT>
struct Lay {
  static constexpr int NB = NT == 1 ? 8 : 16;  // warps accumulating Z (split of J)
  static constexpr int WARP_A0 = 0, WARP_B0 = NA, WARP_PROD = NA + NB, WARP_AUX = NA + NB + 1;
  static constexpr int NWARPS = NMISC + NA + NB;
  static constexpr int NTHREADS = 32 * NWARPS;
  static constexpr int REGS_LAUNCH = 65536 / NTHREADS / 8 * 8;  // what __launch_bounds__(NTHREADS, 1) allows
  static constexpr int REGS_B = NT == 1 ? 128 : 80;
  static_assert(NA % 4 == 0 && NB % 4 == 0 && NMISC % 4 == 0 && 1 + NAUX <= NMISC && REGS_A <= REGS_LAUNCH &&
                    NB <= NB_MAX,
                "role groups fill whole warpgroups");
  static_assert(NA * REGS_A + NB * REGS_B + NMISC * REGS_MISC <= NWARPS * REGS_LAUNCH,
                "the B warps' increase comes from the other groups");
};
inline int nb_of(int NT) { return NT == 1 ? Lay<1>::NB : Lay<3>::NB; }
inline int nwarps_of(int NT) { return NMISC + NA + nb_of(NT); }

struct Params {
  const void* X;
  int64_t ldx;
  int J, JP, L, sp, ns;
  int rowbytes[2];          // bytes of each row copied by CTA 0 / 1 of the pair (its columns)
  const double* img;        // K x ng x (JP/4) x NT x 32 fragment-major B images
  const int32_t* piece_slice;
  const int64_t* piece_row0;
  const int32_t* piece_rows;
  const int32_t* seg_begin;
  double* out_part;         // npieces x J x sp
  double* y_out;            // total_rows x sp or null
  double* g_part;           // npieces x sp x sp or null (single column group)
  int64_t* status;
  uint32_t off_img, off_yp, off_yf, off_bar;
  unsigned long long* dbg;  // DP2_S64_DEBUG: per-warp wait cycles by barrier class, or null
};

DP2_DEV uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
DP2_DEV void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
DP2_DEV void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
DP2_DEV bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded wait: a protocol error traps instead of hanging the GPU
DP2_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t n = 1;; ++n) {
    if (mbar_try(bar, parity)) return;
    if ((n & 255u) == 0 && clock64() - t0 > 20000000000ll) __trap();
  }
}
DP2_DEV void warp_arrive(uint32_t bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
DP2_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
DP2_DEV void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// ---- cluster (CTA pair) primitives: the partner's shared memory (DSMEM)
DP2_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DP2_DEV uint32_t mapa(uint32_t local_addr, uint32_t rank) {  // same smem variable in CTA ``rank``
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
DP2_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
DP2_DEV bool mbar_try_cluster(uint32_t bar, uint32_t parity) {  // acquire at cluster scope
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
DP2_DEV void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  if (mbar_try_cluster(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t n = 1;; ++n) {
    if (mbar_try_cluster(bar, parity)) return;
    if ((n & 255u) == 0 && clock64() - t0 > 20000000000ll) __trap();
  }
}
DP2_DEV void st_cluster_v2(uint32_t cluster_addr, double a, double b) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(cluster_addr), "d"(a), "d"(b) : "memory");
}
// Exact fp32 -> fp64 widening.  F2F.F64.F32 runs at 16 lanes/clk/SM and
// competes with the DMMAs for the FP64 pipe, so with INT the exponent is
// re-biased with integer instructions instead (zero keeps its sign; denormals
// / Inf / NaN -- exponent 0 or 255 -- take the conversion instruction).
// Measured: c3 (J = 256, NT = 3: one conversion per 3 DMMAs) 18.3 / 19.1 ->
// 16.8 / 17.7 ms per pass; the c5 shard (NT = 1: one conversion per DMMA, ~9
// integer instructions each) 34.4 -> 56.3 ms, issue-bound -- so NT = 1 keeps
// the conversion instruction.
template <bool INT>
DP2_DEV double widen(double x) { return x; }
template <bool INT>
DP2_DEV double widen(float x) {
  if constexpr (!INT) return (double)x;
  const uint32_t u = __float_as_uint(x), a = u & 0x7fffffffu;
  uint32_t hi = ((a >> 3) + 0x38000000u) | (u & 0x80000000u);
  const uint32_t lo = u << 29;  // 0 for +-0
  if (a - 0x00800000u >= 0x7f000000u) {  // exponent 0 or 255
    if (a != 0u) return (double)x;
    hi = u;
  }
  return __hiloint2double((int)hi, (int)lo);
}

template <int N>
DP2_DEV void reg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
DP2_DEV void reg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
DP2_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// wait with cycle accounting into dacc[k] when DBG (DP2_S64_DEBUG=1)
#define S64_WAIT(barexpr, par, k)                        \
  do {                                                   \
    if (DBG) {                                           \
      const long long t0_ = clock64();                   \
      mbar_wait(barexpr, par);                           \
      dacc[k] += (unsigned long long)(clock64() - t0_);  \
    } else {                                             \
      mbar_wait(barexpr, par);                           \
    }                                                    \
  } while (0)
#define S64_WAIT_CL(barexpr, par, k)                     \
  do {                                                   \
    if (DBG) {                                           \
      const long long t0_ = clock64();                   \
      mbar_wait_cluster(barexpr, par);                   \
      dacc[k] += (unsigned long long)(clock64() - t0_);  \
    } else {                                             \
      mbar_wait_cluster(barexpr, par);                   \
    }                                                    \
  } while (0)
enum { D_XFULL = 0, D_XEMPTY, D_OFULL, D_OEMPTY, D_YPFULL, D_YPEMPTY, D_YFULL, D_YEMPTY, D_TOTAL, D_N = 10 };

// barrier slots
constexpr int MAXS = 12;  // X ring stages
enum { B_XFULL = 0, B_XEMPTY = MAXS, B_OFULL = 2 * MAXS, B_OEMPTY = 2 * MAXS + NA, B_YPFULL = 2 * MAXS + 2 * NA,
       B_YPEMPTY = B_YPFULL + NY, B_YFULL = B_YPEMPTY + NY, B_YEMPTY = B_YFULL + NY, B_COUNT = B_YEMPTY + NY };

// CL = 2: a CTA pair (thread-block cluster) shares each segment, CTA c
// handling columns [c JH, (c + 1) JH) of J (JH = JP / 2): half the B image and
// half-width X stages per CTA -- so about three times the ring depth -- with
// the four local Y partials of each tile exchanged through DSMEM (each CTA's
// aux sums all eight in the same global order, so both hold the identical
// Y_t for their B warps).
template <typename T, int NT, int CL, int TM, bool DBG>
__global__ void __launch_bounds__(Lay<NT>::NTHREADS, 1) sketch64_kernel(Params prm) {
  using LY = Lay<NT>;
  constexpr int NB = LY::NB, WARP_A0 = LY::WARP_A0, WARP_B0 = LY::WARP_B0, WARP_PROD = LY::WARP_PROD,
                WARP_AUX = LY::WARP_AUX, NWARPS = LY::NWARPS, NTHREADS = LY::NTHREADS, REGS_B = LY::REGS_B,
                REGS_LAUNCH = LY::REGS_LAUNCH;
  constexpr int SG = 8 * NT;
  constexpr int RB = TM / 8;            // DMMA row blocks per tile (A warps)
  constexpr int K2 = TM / 4;            // k-steps of 4 rows per tile (B warps, G)
  // one accumulator set: with two A warps and the B warps sharing the pipe a warp's NT (x RB) chains are
  // spaced beyond the DMMA latency, and a second set costs 2 NT adds per tile on the contended FP64 pipe
  constexpr int SETS = 1;
  // k-steps unrolled in the A loop (measured: 8 is ~1-2% faster than 4 at c3 / the c5 shard, 1.4% slower at c2)
  constexpr int UNR = (TM == 16 || NT == 1) ? 8 : 4;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = CL == 2 ? (int)cluster_rank() : 0;
  const int seg = blockIdx.x / CL, grp = blockIdx.y, ng = gridDim.y;
  const int J = prm.J, JP = prm.JP, L = prm.L, sp = prm.sp, NS = prm.ns;
  const int JH = JP / CL;            // columns of J owned by this CTA
  const int jofs = crank * JH;       // its first column
  const int col0 = grp * SG;
  T* xs = reinterpret_cast<T*>(smem);                                  // [NS][TM][L]
  double* img = reinterpret_cast<double*>(smem + prm.off_img);          // [JH/4][NT][32]
  double* ypart = reinterpret_cast<double*>(smem + prm.off_yp);         // [NY][CL NA][TM][SG]
  double* yfin = reinterpret_cast<double*>(smem + prm.off_yf);          // [NY][K2][NT][32]
  const uint32_t bar0 = su32(smem + prm.off_bar);
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };

  // zero the X ring (pad columns are never written; stale rows must be finite)
  for (int i = threadIdx.x; i < NS * TM * L; i += NTHREADS) xs[i] = T(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bar(B_XFULL + s), 1);
      mbar_init(bar(B_XEMPTY + s), NA + NB);
    }
    for (int a = 0; a < NA; ++a) {
      mbar_init(bar(B_OFULL + a), 1);
      mbar_init(bar(B_OEMPTY + a), 1);
    }
    for (int b = 0; b < NY; ++b) {
      mbar_init(bar(B_YPFULL + b), CL * NA);  // both CTAs' A warps
      mbar_init(bar(B_YPEMPTY + b), CL * NAUX);  // both CTAs' aux warps read this CTA's partials
      mbar_init(bar(B_YFULL + b), NAUX);
      mbar_init(bar(B_YEMPTY + b), NB);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if constexpr (CL == 2) cluster_sync();  // the partner's barriers exist before any remote arrival
  const uint32_t peer = crank ^ 1;

  const int pbeg = prm.seg_begin[seg], pend = prm.seg_begin[seg + 1];
  const int ksq = JH / (4 * NA);  // k-steps per A warp (its share of this CTA's columns)
  unsigned long long dacc[DBG ? D_N : 1] = {};
  const long long tstart = DBG ? clock64() : 0;

  // ------------------------------------------------------------ aux: Y_t, Y rows, non-finite
  // aux warp ax owns the fragments f = k2 NT + j with f % NAUX == ax
  auto aux_role = [&](const int ax) {
    constexpr int NF = (K2 * NT + NAUX - 1) / NAUX;
    int n = 0;
    for (int p = pbeg; p < pend; ++p) {
      const int ks = prm.piece_slice[p], rows = prm.piece_rows[p];
      const int64_t row0 = prm.piece_row0[p];
      int bad = 0;
      for (int t = 0; t * TM < rows; ++t, ++n) {
        const int b = n % NY;
        const int valid = min(TM, rows - t * TM);
        if constexpr (CL == 2) S64_WAIT_CL(bar(B_YPFULL + b), (n / NY) & 1, D_YPFULL);
        else S64_WAIT(bar(B_YPFULL + b), (n / NY) & 1, D_YPFULL);
        if (n >= NY) S64_WAIT(bar(B_YEMPTY + b), ((n / NY) - 1) & 1, D_YEMPTY);
        // element e of the B-fragment image: ks2 = e / (NT*32), j = (e / 32) % NT, lane' = e % 32
        //   -> Y[4 ks2 + (lane' & 3)][8 j + (lane' >> 2)]
        double* yf = yfin + (size_t)b * K2 * NT * 32;
        const double* ypb = ypart + (size_t)b * CL * NA * TM * SG;
        double fr[NF];
#pragma unroll
        for (int i = 0; i < NF; ++i) {
          const int f = ax + i * NAUX;
          if (f < K2 * NT) {
            const int k2 = f / NT, j = f - k2 * NT;
            const int row = 4 * k2 + (lane & 3), col = 8 * j + (lane >> 2);
            // slots in pair order (CTA 0's partials, then CTA 1's): same sum in both CTAs.  The adds
            // queue behind the DMMAs on the FP64 pipe (the aux warps' busy time), so none is spent on 0 + p
            double v = ypb[(size_t)row * SG + col];
#pragma unroll
            for (int aa = 1; aa < CL * NA; ++aa) v += ypb[((size_t)aa * TM + row) * SG + col];
            v = row < valid ? v : 0.0;
            bad |= !isfinite(v);
            fr[i] = v;
            yf[f * 32 + lane] = v;
          }
        }
        warp_arrive(bar(B_YFULL + b));
        warp_arrive(bar(B_YPEMPTY + b));
        if constexpr (CL == 2) {
          if (lane == 0) mbar_arrive_cluster(mapa(bar(B_YPEMPTY + b), peer));
        }
        if (prm.y_out != nullptr && crank == 0) {
#pragma unroll
          for (int i = 0; i < NF; ++i) {
            const int f = ax + i * NAUX;
            if (f < K2 * NT) {
              const int k2 = f / NT, j = f - k2 * NT;
              const int row = 4 * k2 + (lane & 3), col = col0 + 8 * j + (lane >> 2);
              if (row < valid && col < sp) prm.y_out[(row0 + (int64_t)t * TM + row) * sp + col] = fr[i];
            }
          }
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) status_min(prm.status, ST_NONFINITE, ks);
    }
  };
  // every role group first re-balances its registers (REGS_*)
  if (warp >= WARP_PROD) {
   reg_dec<REGS_MISC>();
   if (warp == WARP_PROD) {
    // ------------------------------------------------------------ producer
    const char* Xb = reinterpret_cast<const char*>(prm.X);
    const uint32_t qbytes = (uint32_t)ksq * NT * 32 * 8;
    int n = 0, rs = 0, rph = 0;  // tile count, ring stage and its phase
    for (int p = pbeg; p < pend; ++p) {
      const int ks = prm.piece_slice[p], rows = prm.piece_rows[p];
      const int64_t row0 = prm.piece_row0[p];
      const int pi = p - pbeg;
      // B image of this slice, share by share as each A warp frees it
      const double* src = prm.img + ((size_t)ks * ng + grp) * (size_t)(JP / 4) * NT * 32 +
                          (size_t)crank * (JH / 4) * NT * 32;
      if (lane < NA) {
        if (pi > 0) S64_WAIT(bar(B_OEMPTY + lane), (pi - 1) & 1, D_OEMPTY);
        mbar_expect_tx(bar(B_OFULL + lane), qbytes);
        bulk_load(su32(img) + (uint32_t)lane * qbytes, src + (size_t)lane * ksq * NT * 32, qbytes,
                  bar(B_OFULL + lane));
      }
      const int rowbytes = prm.rowbytes[crank];
      for (int t = 0; t * TM < rows; ++t, ++n) {
        const int s = rs;
        const int valid = min(TM, rows - t * TM);
        if (n >= NS) S64_WAIT(bar(B_XEMPTY + s), rph ^ 1, D_XEMPTY);
        if (++rs == NS) { rs = 0; rph ^= 1; }
        if (lane == 0) mbar_expect_tx(bar(B_XFULL + s), (uint32_t)(valid * rowbytes));
        __syncwarp();
        if (lane < valid && rowbytes > 0)
          bulk_load(su32(xs + ((size_t)s * TM + lane) * L),
                    Xb + ((size_t)(row0 + (int64_t)t * TM + lane) * prm.ldx + jofs) * sizeof(T), (uint32_t)rowbytes,
                    bar(B_XFULL + s));
      }
    }
   } else if (warp < WARP_AUX + NAUX) {
    aux_role(warp - WARP_AUX);
   }
  } else if (warp < WARP_A0 + NA) {
    if constexpr (REGS_A < REGS_LAUNCH) reg_dec<REGS_A>();
    // ------------------------------------------------------------ A warps: Y partials
    const int a = warp - WARP_A0;
    const int r = lane >> 2, q = lane & 3;
    int n = 0, rs = 0, rph = 0;
    for (int p = pbeg; p < pend; ++p) {
      const int rows = prm.piece_rows[p];
      const int pi = p - pbeg;
      S64_WAIT(bar(B_OFULL + a), pi & 1, D_OFULL);
      const double* im = img + (size_t)a * ksq * NT * 32 + lane;
      for (int t = 0; t * TM < rows; ++t, ++n) {
        const int s = rs, b = n % NY;
        S64_WAIT(bar(B_XFULL + s), rph, D_XFULL);
        if (++rs == NS) { rs = 0; rph ^= 1; }
        const T* xr = xs + ((size_t)s * TM + r) * L + a * (JH / NA) + q;
        double c[SETS][RB][NT][2];
#pragma unroll
        for (int u = 0; u < SETS; ++u)
#pragma unroll
          for (int rb = 0; rb < RB; ++rb)
#pragma unroll
            for (int j = 0; j < NT; ++j) c[u][rb][j][0] = c[u][rb][j][1] = 0.0;
#pragma unroll UNR
        for (int k = 0; k < ksq; k += SETS) {
#pragma unroll
          for (int u = 0; u < SETS; ++u) {
            double x[RB];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) x[rb] = widen<(NT > 1)>(xr[(size_t)8 * rb * L + 4 * (k + u)]);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              const double o = im[((k + u) * NT + j) * 32];
#pragma unroll
              for (int rb = 0; rb < RB; ++rb) dmma_8x8x4(c[u][rb][j][0], c[u][rb][j][1], x[rb], o);
            }
          }
        }
        // partial -> ypart[b][a] (C fragment: row r, cols 8j + 2q, +1)
        if (n >= NY) S64_WAIT(bar(B_YPEMPTY + b), ((n / NY) - 1) & 1, D_YPEMPTY);
        // slot crank NA + a of the pair-wide partial ring, written into both
        // CTAs' copies (the partner's through DSMEM)
        double* yp = ypart + (((size_t)b * CL * NA + crank * NA + a) * TM + r) * SG + 2 * q;
#pragma unroll
        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            double2 v;
            v.x = SETS == 2 ? c[0][rb][j][0] + c[SETS - 1][rb][j][0] : c[0][rb][j][0];
            v.y = SETS == 2 ? c[0][rb][j][1] + c[SETS - 1][rb][j][1] : c[0][rb][j][1];
            double* dst = yp + (size_t)8 * rb * SG + 8 * j;
            *reinterpret_cast<double2*>(dst) = v;
            if constexpr (CL == 2) st_cluster_v2(mapa(su32(dst), peer), v.x, v.y);
          }
        warp_arrive(bar(B_YPFULL + b));
        if constexpr (CL == 2) {  // the partner's aux sums this CTA's partials too
          if (lane == 0) mbar_arrive_cluster(mapa(bar(B_YPFULL + b), peer));
        }
        warp_arrive(bar(B_XEMPTY + s));
      }
      warp_arrive(bar(B_OEMPTY + a));
    }
  } else {
    reg_inc<REGS_B>();
    // ------------------------------------------------------------ B warps: Z += X_t^T Y_t
    const int bw = warp - WARP_B0;
    // J-blocks of 8 per B warp: <= 4 at J <= 512; J <= 1024 runs one sketch
    // column block per CTA (NT = 1) with up to 8
    constexpr int MBMAX = (NT == 1 ? 128 : 64) / NB;
    const int MB = JH / (8 * NB);
    const int jb0 = bw * MB;
    double z[MBMAX][NT][2];
#pragma unroll
    for (int i = 0; i < MBMAX; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) z[i][j][0] = z[i][j][1] = 0.0;
    // G = Y^T Y per piece (pass 2): 8 x 8 tile (gi, gj) owned by B warp
    // gi NT + gj -- Y^T fragments are the B fragments this warp loads anyway,
    // so the 2 NT^2 DMMAs per tile spread over the sub-partitions (the aux
    // warp alone made its sub-partition the slowest)
    constexpr int GT = (NT * NT + NB - 1) / NB;  // G tiles per B warp: tile bw + i NB
    const bool g_on = prm.g_part != nullptr && crank == 0;
    double g[GT][2];
#pragma unroll
    for (int i = 0; i < GT; ++i) g[i][0] = g[i][1] = 0.0;
    int n = 0, rs = 0, rph = 0;
    for (int p = pbeg; p < pend; ++p) {
      const int rows = prm.piece_rows[p];
      for (int t = 0; t * TM < rows; ++t, ++n) {
        const int s = rs, b = n % NY;
        S64_WAIT(bar(B_XFULL + s), rph, D_XFULL);
        if (++rs == NS) { rs = 0; rph ^= 1; }
        S64_WAIT(bar(B_YFULL + b), (n / NY) & 1, D_YFULL);
        const double* yf = yfin + (size_t)b * K2 * NT * 32 + lane;
        const T* xb = xs + ((size_t)s * TM + (lane & 3)) * L + 8 * jb0 + (lane >> 2);
#pragma unroll
        for (int k2 = 0; k2 < K2; ++k2) {
          double yv[NT];
#pragma unroll
          for (int j = 0; j < NT; ++j) yv[j] = yf[(k2 * NT + j) * 32];
          if (g_on) {
#pragma unroll
            for (int i = 0; i < GT; ++i) {
              const int gt = bw + i * NB;
              if (gt < NT * NT) {
                const int gi = gt / NT, gj = gt - gi * NT;
                double ya = 0.0, yb = 0.0;
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                  ya = j == gi ? yv[j] : ya;
                  yb = j == gj ? yv[j] : yb;
                }
                dmma_8x8x4(g[i][0], g[i][1], ya, yb);
              }
            }
          }
#pragma unroll
          for (int i = 0; i < MBMAX; ++i) {
            if (i < MB) {
              const double xv = widen<(NT > 1)>(xb[(size_t)4 * k2 * L + 8 * i]);
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma_8x8x4(z[i][j][0], z[i][j][1], xv, yv[j]);
            }
          }
        }
        warp_arrive(bar(B_YEMPTY + b));
        warp_arrive(bar(B_XEMPTY + s));
      }
      if (g_on) {  // G tile (gi, gj): rows 8 gi + (lane >> 2), cols 8 gj + 2 (lane & 3) (+1)
        double* gp = prm.g_part + (size_t)p * sp * sp;
#pragma unroll
        for (int i = 0; i < GT; ++i) {
          const int gt = bw + i * NB;
          if (gt < NT * NT) {
            const int gi = gt / NT, gj = gt - gi * NT;
            const int rr = 8 * gi + (lane >> 2), cc = 8 * gj + 2 * (lane & 3);
            if (rr < sp && cc < sp) {
              gp[(size_t)rr * sp + cc] = g[i][0];
              if (cc + 1 < sp) gp[(size_t)rr * sp + cc + 1] = g[i][1];
            }
          }
          g[i][0] = g[i][1] = 0.0;
        }
      }
      // piece complete: flush Z rows 8 (jb0 + i) + (lane >> 2), cols col0 + 8 j + 2 (lane & 3) (+1)
      double* out = prm.out_part + (size_t)p * J * sp;
#pragma unroll
      for (int i = 0; i < MBMAX; ++i) {
        if (i < MB) {
          const int m = jofs + 8 * (jb0 + i) + (lane >> 2);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int c = col0 + 8 * j + 2 * (lane & 3);
            if (m < J && c < sp) {
              if (c + 1 < sp) {
                double2 v;
                v.x = z[i][j][0];
                v.y = z[i][j][1];
                *reinterpret_cast<double2*>(out + (size_t)m * sp + c) = v;
              } else {
                out[(size_t)m * sp + c] = z[i][j][0];
              }
            }
            z[i][j][0] = z[i][j][1] = 0.0;
          }
        }
      }
    }
  }
  if constexpr (CL == 2) cluster_sync();  // the partner may still read this CTA's partials / barriers
  if (DBG && lane == 0) {
    dacc[D_TOTAL] = (unsigned long long)(clock64() - tstart);
    unsigned long long* d = prm.dbg + ((size_t)(blockIdx.y * gridDim.x + blockIdx.x) * NWARPS + warp) * D_N;
    for (int i = 0; i < D_N; ++i) d[i] = dacc[i];
  }
}

// Fragment-major B images: img[k][g][ks][j][l] = B[k][4 ks + (l & 3)][8 (NT g + j) + (l >> 2)]
// (0 outside J x sp).  One warp per (k, g, ks) unit: NT coalesced 256-byte
// stores, reads of 4 rows x 64 bytes per fragment.
template <int NT>
__global__ void __launch_bounds__(256) image_kernel(const double* __restrict__ B, int64_t K, int J, int JP, int sp,
                                                     int ng, double* __restrict__ img) {
  const int lane = threadIdx.x & 31;
  const int nks = JP / 4;
  const int64_t units = K * ng * nks;
  const int row_in = lane & 3, col_in = lane >> 2;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < units;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int ks = (int)(u % nks);
    const int64_t kg = u / nks;
    const int g = (int)(kg % ng);
    const int64_t k = kg / ng;
    const int row = 4 * ks + row_in;
    const double* src = B + ((size_t)k * J + (row < J ? row : 0)) * sp;
    double* dst = img + (size_t)u * NT * 32 + lane;
#pragma unroll
    for (int jj = 0; jj < NT; ++jj) {
      const int col = 8 * (NT * g + jj) + col_in;
      dst[jj * 32] = (row < J && col < sp) ? __ldg(src + col) : 0.0;
    }
  }
}

// CTA pairs split J when DP2_S64_PAIRS=1 and that costs at most ~15% column
// padding.  Off by default: measured at c2 fp64 the pair version (9 ring
// stages of half-width X, partials exchanged by DSMEM stores) ran 8.3 / 8.8 ms
// per pass against 4.2 / 4.4 ms for single CTAs -- with half of J per CTA the
// 8-row tile carries too little DMMA work per hand-off (A warps 48, B warps
// 12 per tile) to amortise the per-tile barrier and fragment-load overhead.
bool uses_pairs(int J) {
  static const bool on = getenv("DP2_S64_PAIRS") && atoi(getenv("DP2_S64_PAIRS")) != 0;
  const int JP2 = (J + 16 * NB_MAX - 1) / (16 * NB_MAX) * (16 * NB_MAX);
  return on && J >= 256 && J <= 512 && JP2 * 100 <= J * 115;
}

struct Plan {
  int NT, ng, JP, L, ns, CL, TM;
  size_t smem;
  uint32_t off_img, off_yp, off_yf, off_bar;
};

bool plan(int J, int sp, int elem, Plan* pl) {
  if (J < 1 || J > 1024 || sp < 8 || sp % 8) return false;
  const int nbt = sp / 8;
  // groups of <= 3 column blocks (last one zero padded); above J = 512 the
  // image of 3 blocks no longer fits next to the X ring: one block per CTA
  // group (X is then streamed once per block -- the pass stays DMMA-bound)
  const int NT = J > 512 ? 1 : (nbt <= 3 ? nbt : 3);
  const int ng = (nbt + NT - 1) / NT;
  const int CL = uses_pairs(J) ? 2 : 1;
  const int NB = nb_of(NT);
  const int JP = CL == 2 ? (J + 16 * NB - 1) / (16 * NB) * (16 * NB) : (J + 8 * NB - 1) / (8 * NB) * (8 * NB);
  const int JH = JP / CL;
  // tile height: keep ~96 DMMAs per A warp and ~24 per B warp per tile as J shrinks
  const int TM = JH > 256 ? 8 : 16;  // (32-row tiles at J <= 128 spill: the aux's Y_t fragments; 16-row tiles at
                                     // J = 1000 fp32, 2 ring stages: 35.6 ms per c5-shard pass against 33.8; 8-row tiles at J = 256:
                                     // 19.4 / 18.6 ms per c3 pass against 16.8 / 17.6)
  int L = JH + 4;  // elements: 8 B -> L % 16 == 4; 4 B -> L % 32 == 4
  if (elem == 8) {
    while (L % 16 != 4) ++L;
  } else {
    while (L % 32 != 4) ++L;
  }
  const int SG = 8 * NT;
  const size_t img = (size_t)(JH / 4) * NT * 32 * 8;
  const size_t yp = (size_t)NY * CL * NA * TM * SG * 8, yf = (size_t)NY * (TM / 4) * NT * 32 * 8;
  const size_t stage = (size_t)TM * L * elem;
  const size_t cap = 227 * 1024;
  int ns = MAXS;
  while (ns >= 2 && ns * stage + img + yp + yf + 8 * B_COUNT + 256 > cap) --ns;
  if (ns < 2) return false;
  pl->CL = CL;
  pl->TM = TM;
  pl->NT = NT;
  pl->ng = ng;
  pl->JP = JP;
  pl->L = L;
  pl->ns = ns;
  size_t off = ns * stage;
  off = (off + 127) & ~(size_t)127;
  pl->off_img = (uint32_t)off;
  off += img;
  pl->off_yp = (uint32_t)off;
  off += yp;
  pl->off_yf = (uint32_t)off;
  off += yf;
  pl->off_bar = (uint32_t)((off + 7) & ~(size_t)7);
  pl->smem = pl->off_bar + 8 * B_COUNT;
  return true;
}

// per-device image scratch (grown on demand, kept)
double* image_scratch(size_t bytes, cudaError_t* err) {
  static double* buf[64] = {};
  static size_t cap[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) {
    *err = cudaErrorInvalidDevice;
    return nullptr;
  }
  if (cap[dev] < bytes) {
    if (buf[dev]) cudaFree(buf[dev]);
    buf[dev] = nullptr;
    cap[dev] = 0;
    *err = cudaMalloc(&buf[dev], bytes);
    if (*err != cudaSuccess) return nullptr;
    cap[dev] = bytes;
  }
  *err = cudaSuccess;
  return buf[dev];
}

template <typename T, int NT, int CL, int TM>
cudaError_t launch_cl(const Params& prm, const Plan& pl, int nseg, cudaStream_t st) {
  auto kern = prm.dbg ? sketch64_kernel<T, NT, CL, TM, true> : sketch64_kernel<T, NT, CL, TM, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
  if (e != cudaSuccess) return e;
  if (CL == 1) {
    kern<<<dim3(nseg, pl.ng), Lay<NT>::NTHREADS, pl.smem, st>>>(prm);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CL * nseg, pl.ng);
  cfg.blockDim = dim3(Lay<NT>::NTHREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, prm);
}

template <typename T, int NT, int CL>
cudaError_t launch_tm(const Params& prm, const Plan& pl, int nseg, cudaStream_t st) {
  return pl.TM == 8 ? launch_cl<T, NT, CL, 8>(prm, pl, nseg, st) : launch_cl<T, NT, CL, 16>(prm, pl, nseg, st);
}

template <typename T, int NT>
cudaError_t launch(const Params& prm, const Plan& pl, int nseg, cudaStream_t st) {
  return pl.CL == 2 ? launch_tm<T, NT, 2>(prm, pl, nseg, st) : launch_tm<T, NT, 1>(prm, pl, nseg, st);
}

cudaError_t launch_any(int elem, int NT, const Params& prm, const Plan& pl, int nseg, cudaStream_t st) {
  if (elem == 8) {
    switch (NT) {
      case 1: return launch<double, 1>(prm, pl, nseg, st);
      case 2: return launch<double, 2>(prm, pl, nseg, st);
      default: return launch<double, 3>(prm, pl, nseg, st);
    }
  }
  switch (NT) {
    case 1: return launch<float, 1>(prm, pl, nseg, st);
    case 2: return launch<float, 2>(prm, pl, nseg, st);
    default: return launch<float, 3>(prm, pl, nseg, st);
  }
}

// DP2_S64_DEBUG: run with per-warp wait accounting and print the share of
// cycles each role spends waiting on each barrier class (debug aid; syncs)
cudaError_t launch_debug(int elem, int NT, Params prm, const Plan& pl, int nseg, cudaStream_t stream) {
  const int NB = nb_of(NT), NWARPS = nwarps_of(NT);
  const int WARP_A0 = 0, WARP_B0 = NA, WARP_PROD = NA + NB, WARP_AUX = NA + NB + 1;
  const size_t nd = (size_t)nseg * pl.CL * pl.ng * NWARPS * D_N;
  unsigned long long *dh = nullptr, *dd = nullptr;
  cudaError_t e = cudaHostAlloc(&dh, nd * 8, cudaHostAllocMapped);
  if (e != cudaSuccess) return e;
  memset(dh, 0, nd * 8);
  cudaHostGetDevicePointer(&dd, dh, 0);
  prm.dbg = dd;
  e = launch_any(elem, NT, prm, pl, nseg, stream);
  cudaStreamSynchronize(stream);
  const char* names[] = {"xfull", "xempty", "ofull", "oempty", "ypfull", "ypempty", "yfull", "yempty"};
  const char* roles[] = {"A", "B", "prod", "aux"};
  for (int role = 0; role < 4; ++role) {
    double acc[D_N] = {};
    int cnt = 0;
    for (size_t c = 0; c < (size_t)nseg * pl.CL * pl.ng; ++c)
      for (int w = 0; w < WARP_AUX + NAUX; ++w) {
        const int r = (w >= WARP_A0 && w < WARP_A0 + NA) ? 0 : (w >= WARP_B0 && w < WARP_B0 + NB) ? 1
                      : w == WARP_PROD ? 2 : 3;  // every aux warp
        if (r != role) continue;
        ++cnt;
        for (int i = 0; i < D_N; ++i) acc[i] += (double)dh[(c * NWARPS + w) * D_N + i];
      }
    fprintf(stderr, "[s64] %-4s total %.0f kcyc:", roles[role], acc[D_TOTAL] / (cnt ? cnt : 1) / 1e3);
    for (int i = 0; i < 8; ++i)
      if (acc[i] > 0) fprintf(stderr, " %s %.1f%%", names[i], 100.0 * acc[i] / acc[D_TOTAL]);
    fprintf(stderr, "\n");
  }
  cudaFreeHost(dh);
  return e;
}

}  // namespace s64

bool sketch64_pairs(int64_t J) { return s64::uses_pairs((int)J); }

bool sketch64_eligible(const dp2_store* st, int sp, bool xsq, bool gram) {
  if (xsq) return false;  // the per-piece sums of squares live in the older passes
  static const bool off = getenv("DP2_SKETCH64") && atoi(getenv("DP2_SKETCH64")) == 0;
  if (off) return false;
  const int elem = st->dtype == DP2_F64 ? 8 : 4;
  if ((st->J * elem) % 16 != 0 || (st->ldx * elem) % 16 != 0 || reinterpret_cast<uintptr_t>(st->X) % 16 != 0)
    return false;
  s64::Plan pl{};
  return s64::plan((int)st->J, sp, elem, &pl) && (!gram || pl.ng == 1);  // G needs one column group
}

cudaError_t run_sketch64(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                         int64_t* status, cudaStream_t stream, double* g_part) {
  const int elem = st->dtype == DP2_F64 ? 8 : 4;
  s64::Plan pl{};
  if (!s64::plan((int)st->J, sp, elem, &pl)) return cudaErrorInvalidValue;
  const int J = (int)st->J;
  const size_t img_elems = (size_t)st->K * pl.ng * (pl.JP / 4) * pl.NT * 32;
  cudaError_t e = cudaSuccess;
  double* img = s64::image_scratch(img_elems * 8, &e);
  if (!img) return e;
  {
    const int64_t warps = st->K * pl.ng * (pl.JP / 4);
    const unsigned blocks = (unsigned)std::min<int64_t>((warps + 7) / 8, 148 * 16);
    if (pl.NT == 1) s64::image_kernel<1><<<blocks, 256, 0, stream>>>(B, st->K, J, pl.JP, sp, pl.ng, img);
    else if (pl.NT == 2) s64::image_kernel<2><<<blocks, 256, 0, stream>>>(B, st->K, J, pl.JP, sp, pl.ng, img);
    else s64::image_kernel<3><<<blocks, 256, 0, stream>>>(B, st->K, J, pl.JP, sp, pl.ng, img);
  }
  s64::Params prm{};
  prm.X = st->X;
  prm.ldx = st->ldx;
  prm.J = J;
  prm.JP = pl.JP;
  prm.L = pl.L;
  prm.sp = sp;
  prm.ns = pl.ns;
  {  // each CTA of a pair copies its own columns of every row
    const int JH = pl.JP / pl.CL;
    for (int c = 0; c < 2; ++c) {
      const int cols = c < pl.CL ? std::max(0, std::min(JH, J - c * JH)) : 0;
      prm.rowbytes[c] = (cols * elem + 15) / 16 * 16;
    }
  }
  prm.img = img;
  prm.piece_slice = st->piece_slice;
  prm.piece_row0 = st->piece_row0;
  prm.piece_rows = st->piece_rows;
  prm.seg_begin = st->seg_begin;
  prm.out_part = out_part;
  prm.y_out = y_out;
  prm.g_part = (pl.ng == 1) ? g_part : nullptr;
  prm.status = status;
  prm.off_img = pl.off_img;
  prm.off_yp = pl.off_yp;
  prm.off_yf = pl.off_yf;
  prm.off_bar = pl.off_bar;
  const int nseg = st->nseg;
  static const bool dbg = getenv("DP2_S64_DEBUG") && atoi(getenv("DP2_S64_DEBUG")) != 0;
  if (dbg) return s64::launch_debug(elem, pl.NT, prm, pl, nseg, stream);
  return s64::launch_any(elem, pl.NT, prm, pl, nseg, stream);
}

}  // namespace dp2
