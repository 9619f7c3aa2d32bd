// Stage-1 streaming sketch pass for fp32 slice storage on the 5th-gen tensor
// cores (tcgen05.mma kind::tf32, accumulators in TMEM).
//
// Same contract as run_sketch_f32 (dp2_sketch32.cu) and the fp64 DMMA pass:
// per persistent segment, walk the pieces (segment x slice) tile by tile and
//   Y_t = X_t B            (P1: M = 64 rows, N = sp, K = J)
//   Z  += X_t^T Y_t        (P2: M = 128 columns of X, N = sp (padded to 16), K = 64 rows)
// writing one fp64 partial Z (J x sp) per piece, plus (pass 1) the per-piece
// sum of squares / non-finite flag and (pass 2) Y rows and G = Y^T Y.
// P/compress.py:64-103 (randomized_svd per slice) is what this computes the
// sketches of; the algebra is DESIGN.md §3.
//
// Data movement (one CTA per SM, 19 warps):
//   warp 13     TMA: lane 0 streams 64-row x 32-column boxes of X
//               (cp.async.bulk.tensor, SWIZZLE_128B) into a ring of 8 KB
//               chunk slots -- P1's K-major A operand, read by the tensor
//               core as is (tf32 = the top 19 bits of each fp32); lane 1
//               bulk-copies the slice's pre-tiled tf32 B image per piece.
//   warps 0-7   X^T producers: read each ring unit back, round to tf32
//               (cvt.rna) and tcgen05.st it into TMEM (lane = column of X,
//               TMEM column = row): P2's A operand X^T, which must be
//               K-major.  (tf32 MN-major shared-memory operands only exist in
//               the 128B-base-32B swizzle, which no K-major layout shares, so
//               one shared-memory copy cannot feed both products --
//               tools/umma_probe.cu measures this.)
//   warp 8      TMEM allocation + the elected thread issuing P1 and the
//               tcgen05.commit arrivals; warp 14 issues P2.
//   warps 9-12  epilogue: tcgen05.ld of Y (TMEM lanes = rows) -> rounded Y^T
//               into shared memory as P2's K-major B operand, the non-finite
//               flag, and the per-piece Z flush (TMEM lanes = columns of X).
//   warps 15-18 pass 2: Y rows out (coalesced through shared memory).
// TMEM: a ring of nxs X^T slots of 64 columns (nxs = 5 at J = 512: one unit
// more than a tile, so the X^T producers run ahead of P2 into the next tile),
// Z (32 columns per 128 columns of X), Y double-buffered (64 columns).  Ring
// slots are released right after P1, the X^T slots after P2, so HBM
// streaming overlaps both products.
//
// 512 < J <= 1024 (c5): X^T and Z of all J columns exceed TMEM, so a CTA
// pair (thread-block cluster of 2) shares each pair of segments: CTA r
// streams columns [r JH, (r + 1) JH) of every tile (JH = Jp / 2 <= 512) and
// loads its half of the B image; P1 yields a partial Y_t over those columns,
// the main epilogue group stores it into the peer's shared memory
// (st.shared::cluster, one remote mbarrier arrive per warp), and each CTA
// adds the two partials (fp32 addition commutes: both hold the same Y_t) to
// stage Y^T for its own P2, Z over its columns and the Z flush of its rows of
// the partial.  Rank 0 writes Y rows / G (pass 2); rank 1's per-piece sums of
// squares go to a scratch array that a small kernel adds.
//
// Precision: products in tf32 (10-bit mantissa, round-to-nearest on both
// operands), fp32 accumulation within a piece, fp64 partials across pieces --
// an opt-in speed mode (set_fp32_products("tf32")): within the 1e-3 fp32
// budget on c2, not on ~50-row slices (tests/test_gpu_scale_parity.py); the
// default fp32-storage path is the fp64 DMMA pass on upcast values.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cudaTypedefs.h>

#include "dp2_common.cuh"
#include "dp2_internal.h"

namespace dp2 {
namespace tcs {

constexpr int TM = 64;             // rows per tile
constexpr int CHUNK = TM * 128;    // bytes of one 32-column chunk (64 rows x 128 B)
constexpr int NXT = 256;           // X^T producers + statistics (warps 0-7)
constexpr int MMA_WARP = 8;
constexpr int EPI0 = 9 * 32;       // first epilogue thread (warps 9-12)
constexpr int NEPI = 128;
constexpr int TMA_WARP = 13;       // lane 0: X boxes into the ring; lane 1: B image per piece
constexpr int P2_WARP = 14;        // P2 issuer (P1 is issued by MMA_WARP)
constexpr int AUX0 = 15 * 32;      // first aux epilogue thread (warps 15-18): Y rows + G in pass 2
constexpr int NAUX = 128;
constexpr int NTHREADS = 19 * 32;
constexpr uint32_t TMEM_COLS = 512;

struct Params {
  const float* X;
  int64_t ldx;
  int J, Jp, sp, n2, nslot, nsup;
  const double* B;
  const float* btile;  // B pre-tiled per slice in the shared-memory image (tf32, K-major SW128)
  uint32_t bbytes;     // bytes of one slice's image
  const int32_t* piece_slice;
  const int64_t* piece_row0;
  const int32_t* piece_rows;
  const int32_t* seg_begin;
  double* out_part;
  double* y_out;
  double* xsq_part;
  double* g_part;
  int64_t* status;
  uint32_t off_b, off_y, off_yrow, off_bar;
  // J split across a CTA pair (J > 512): each CTA of the cluster streams JH
  // columns of every tile and the pair exchanges fp32 Y partials through
  // distributed shared memory (csize 1: one CTA per segment, JH = Jp)
  int csize, JH, nseg;
  int nxs, zcol, ycol;  // TMEM plan: X^T slots, Z and Y column bases
  uint32_t bstride;    // floats per slice image (Jp x sp)
  uint32_t off_pbuf;   // peer Y-partial buffers (2 x TM x sp fp32), csize 2
  double* xsq_hi;      // rank 1's per-piece sums of squares (added by the host), csize 2
  unsigned long long* dbg;  // per-CTA wait-time counters (DP2_TC_DEBUG), or null
  int y32;                  // y_out holds fp32 rows (the accumulator's own precision) instead of fp64
};

// ------------------------------------------------------------ PTX helpers
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
// bounded wait: a protocol error traps (kernel error) instead of hanging the GPU
DP2_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t n = 1;; ++n) {
    if (mbar_try(bar, parity)) return;
    if ((n & 255u) == 0 && clock64() - t0 > 20000000000ll) __trap();
  }
}
// cluster-scope variants (J split across a CTA pair)
DP2_DEV bool mbar_try_cl(uint32_t bar, uint32_t parity) {
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
DP2_DEV void mbar_wait_cl(uint32_t bar, uint32_t parity) {
  if (mbar_try_cl(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t n = 1;; ++n) {
    if (mbar_try_cl(bar, parity)) return;
    if ((n & 255u) == 0 && clock64() - t0 > 20000000000ll) __trap();
  }
}
DP2_DEV uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory location in CTA `rank` of the cluster
DP2_DEV uint32_t cl_map(uint32_t saddr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(saddr), "r"(rank));
  return d;
}
DP2_DEV void cl_arrive_remote(uint32_t cl_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_bar) : "memory");
}
DP2_DEV void cl_st_v4(uint32_t cl_addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(cl_addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
DP2_DEV void cl_st_f32(uint32_t cl_addr, float a) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(cl_addr), "f"(a) : "memory");
}
DP2_DEV void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
DP2_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// wait with optional accounting into dbg slot k of this CTA
#define TWAIT(barexpr, par, k)                                           \
  do {                                                                   \
    if (prm.dbg) {                                                       \
      const unsigned long long t0_ = gtime();                            \
      mbar_wait(barexpr, par);                                           \
      dacc[k] += gtime() - t0_;                                          \
    } else {                                                             \
      mbar_wait(barexpr, par);                                           \
    }                                                                    \
  } while (0)
// one arrival per warp (barrier counts in warps): __syncwarp orders the
// lanes' prior accesses before lane 0's release-arrive
DP2_DEV void warp_arrive(uint32_t bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
DP2_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
DP2_DEV void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DP2_DEV void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
DP2_DEV void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
DP2_DEV void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// tcgen05.ld/st are .sync.aligned: call sites that follow lane-divergent code
// (single-lane barrier waits, statistics) must reconverge first
DP2_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  __syncwarp();
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// round to tf32, nearest with ties away from zero: the same bits as
// cvt.rna.tf32.f32 for every finite fp32 value (all 4.28e9 finite patterns
// checked on the device, tools/tf32_round_check.cu) on the integer pipe
DP2_DEV float tf32r(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
DP2_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// shared-memory matrix descriptor, SWIZZLE_128B (sm_100 version 1)
DP2_DEV uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: f32 accumulate, tf32 A/B, majors, N, M
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// byte offset of element (row, col) inside a 128 B-row swizzled block (col < 32)
DP2_DEV uint32_t swz(int row, int col) {
  return (uint32_t)row * 128u + ((uint32_t)(((col >> 2) ^ row) & 7) << 4) + (uint32_t)(col & 3) * 4u;
}

// barrier slots (uint64 each) after off_bar
enum : int {
  BAR_BFULL = 0, BAR_BFREE, BAR_YSFULL = 3, BAR_ZFULL, BAR_ZFREE,
  BAR_YFULL = 16,   // [2] Y accumulator b holds tile t (P1 commit)
  BAR_YFREE = 18,   // [2] epilogue has read Y accumulator b
  BAR_YSTFREE = 20, // P2 has consumed the Y^T staging buffer
  BAR_PFULL = 21,   // [2] csize 2: the peer's Y partial of tile t landed in pbuf[t % 2]
  BAR_PFREE = 23,   // [2] csize 2: the peer has read the partial this CTA wrote into its pbuf[b]
  BAR_XT = 26,      // up to 8 x (full, free) for the TMEM X^T slots
  BAR_RING = 42     // nss x full, nss x empty
};

struct Unit {  // 64 rows x 128 columns of one tile
  int p, t, jb, rows;
  int64_t row0;
};

DP2_DEV void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  __syncwarp();
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// A operand from TMEM (K-major: lanes = M, columns = K)
DP2_DEV void tc_mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// elect.sync-predicated issue (whole warp executes; one lane issues)
DP2_DEV void tc_mma_ss_e(uint32_t d, uint32_t alo, uint32_t blo, uint32_t hi, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %4, p;\n\t}" ::"r"(d),
      "r"(alo), "r"(blo), "r"(hi), "r"(idesc), "r"(acc)
      : "memory");
}
DP2_DEV void tc_mma_ts_e(uint32_t d, uint32_t a_tmem, uint32_t blo, uint32_t hi, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], db, %4, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "r"(blo), "r"(hi), "r"(idesc), "r"(acc)
      : "memory");
}
DP2_DEV void tc_commit_e(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
DP2_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
DP2_DEV void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
DP2_DEV void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// TMEM columns: nxs X^T slots of 64 columns [0, 64 nxs) -- a ring over the
// units (tile, 128-column block), nxs > nsup so the X^T producers can run
// ahead of P2 into the next tile --, Z [zcol, +32 nsup), Y [ycol, +64)

__global__ void __launch_bounds__(NTHREADS, 1) sketch_tc_kernel(Params prm, const __grid_constant__ CUtensorMap xmap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  __shared__ double red[32];
  // csize 2: the CTA pair (cluster) c walks segments 2c and 2c + 1 (adjacent
  // row ranges: their pieces are consecutive), CTA rank r over the columns
  // [r JH, (r + 1) JH) of every tile
  const int csize = prm.csize;
  const uint32_t crank = csize > 1 ? cl_rank() : 0u;
  const int seg = csize > 1 ? (int)(blockIdx.x / 2) * 2 : (int)blockIdx.x;
  const int seg_end = csize > 1 ? min(seg + 2, prm.nseg) : seg + 1;
  const int pbeg = prm.seg_begin[seg], pend = prm.seg_begin[seg_end];
  if (pbeg >= pend) return;  // both CTAs of a pair return together
  const int j0 = (int)crank * prm.JH;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t base = (su32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - su32(smem_raw));
  const int J = prm.J, sp = prm.sp, n2 = prm.n2, nslot = prm.nslot, nsup = prm.nsup;
  const int nss = nslot / 4;  // superslots (4 chunks = one 128-column unit)
  const uint32_t ring = base, bsm = base + prm.off_b, ysm = base + prm.off_y;
  float* yrow = reinterpret_cast<float*>(gbase + prm.off_yrow);
  const uint32_t pbuf = base + prm.off_pbuf;
  const float* pbuf_f = reinterpret_cast<const float*>(gbase + prm.off_pbuf);
  const bool pass2 = prm.y_out != nullptr || prm.g_part != nullptr;  // Y rows and/or G wanted
  const bool auxon = pass2 && crank == 0;  // the pair's Y rows / G come from rank 0
  const uint32_t bars = base + prm.off_bar;
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };

  if (tid == 0) {
    mbar_init(bar(BAR_BFULL), 1);
    mbar_init(bar(BAR_BFREE), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(BAR_YFULL + b), 1);
      mbar_init(bar(BAR_YFREE + b), auxon ? NEPI + NAUX : NEPI);
      mbar_init(bar(BAR_PFULL + b), NEPI / 32);  // one per main epilogue warp of the peer
      mbar_init(bar(BAR_PFREE + b), (pass2 && crank == 1) ? (NEPI + NAUX) / 32 : NEPI / 32);  // the peer's readers
    }
    mbar_init(bar(BAR_YSTFREE), 1);
    mbar_init(bar(BAR_YSFULL), NEPI);
    mbar_init(bar(BAR_ZFULL), 1);
    mbar_init(bar(BAR_ZFREE), NEPI);
    for (int jb = 0; jb < prm.nxs; ++jb) {
      mbar_init(bar(BAR_XT + 2 * jb), NXT / 32);
      mbar_init(bar(BAR_XT + 2 * jb + 1), 1);
    }
    for (int s = 0; s < nss; ++s) {
      mbar_init(bar(BAR_RING + s), 1);  // TMA thread's arrive.expect_tx
      mbar_init(bar(BAR_RING + nss + s), 1 + NXT / 32);  // P1 commit + one per X^T warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Y^T rows >= sp stay zero (P2's N is sp rounded up to 16)
  {
    float* ys = reinterpret_cast<float*>(gbase + prm.off_y);
    for (int i = tid; i < 2 * n2 * 32; i += NTHREADS) ys[i] = 0.0f;
    fence_async_smem();
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (csize > 1) cl_sync();  // the peer's barriers are initialised before any remote arrive
  const uint32_t tmem = tmem_slot;
  const unsigned long long t_start = prm.dbg ? gtime() : 0ull;
  unsigned long long dacc[16] = {};  // wait-time accounting (DP2_TC_DEBUG)

  // unit iteration shared by both producer groups
  auto first_unit = [&](int p) {
    Unit u;
    u.p = p;
    u.t = 0;
    u.jb = 0;
    u.rows = min(TM, prm.piece_rows[p]);
    u.row0 = prm.piece_row0[p];
    return u;
  };
  auto next_unit = [&](Unit u) {
    if (++u.jb < nsup) return u;
    u.jb = 0;
    const int pr = prm.piece_rows[u.p];
    if ((u.t + 1) * TM < pr) {
      ++u.t;
      u.rows = min(TM, pr - u.t * TM);
      return u;
    }
    if (u.p + 1 >= pend) {
      u.p = pend;
      return u;
    }
    return first_unit(u.p + 1);
  };

  if (warp == TMA_WARP) {
    // ===================================================== TMA issuer
    // unit = 4 boxes of 64 rows x 32 columns (128 B inner, SWIZZLE_128B: the
    // UMMA K-major SW128 layout); rows past the piece or the store are other
    // slices' rows or TMA zero fill -- masked downstream (Y^T rows, X^T rows).
    if (lane == 1) {  // B image of each piece's slice, once P1 of the previous piece released it
      int pidx = 0;
      for (int p = pbeg; p < pend; ++p, ++pidx) {
        if (pidx > 0) TWAIT(bar(BAR_BFREE), (uint32_t)(pidx - 1) & 1u, 1);
        mbar_expect_tx(bar(BAR_BFULL), prm.bbytes);
        bulk_load(bsm, prm.btile + (size_t)prm.piece_slice[p] * prm.bstride + crank * (prm.bbytes / 4), prm.bbytes,
                  bar(BAR_BFULL));
      }
    }
    if (lane == 0) {
      Unit cur = first_unit(pbeg);
      int ss = 0;          // ring slot = ucount % nss, fill = ucount / nss (tracked incrementally)
      uint32_t fill = 0;
      while (cur.p < pend) {
        if (fill > 0) TWAIT(bar(BAR_RING + nss + ss), (fill - 1) & 1u, 0);
        mbar_expect_tx(bar(BAR_RING + ss), 4 * CHUNK);
        const int row = (int)(cur.row0 + (int64_t)cur.t * TM);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
          tma_load_2d(ring + (uint32_t)(ss * 4 + ch) * CHUNK, &xmap, j0 + cur.jb * 128 + ch * 32, row,
                      bar(BAR_RING + ss));
        if (++ss == nss) { ss = 0; ++fill; }
        cur = next_unit(cur);
      }
    }
    __syncwarp();
  } else if (tid < NXT) {
    // ===================================================== X^T producers
    // thread (q = warp % 4, h = warp / 4, lane) owns column 32 q + lane of
    // every unit, rows 32 h .. 32 h + 31: one 128 B swizzled ring row per
    // warp-wide LDS (conflict-free), rows past the piece zeroed, statistics,
    // rna rounding, one tcgen05.st.32x32b.x32 to TMEM lane 32 q + lane,
    // columns jb*64 + 32 h, once P2 of the previous tile consumed block jb.
    const int q = warp & 3, h = warp >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool stats = prm.xsq_part != nullptr;
    double sq = 0.0;
    int bad = 0;
    Unit cur = first_unit(pbeg);
    uint32_t rph = 0;  // ring slot ss = ucount % nss with parity rph = (ucount / nss) & 1
    int xs = 0;        // X^T slot = ucount % nxs, used for the xuse-th time
    uint32_t xuse = 0;
    int ss = 0;
    while (cur.p < pend) {
      if (tid == 0) TWAIT(bar(BAR_RING + ss), rph, 2);
      else mbar_wait(bar(BAR_RING + ss), rph);
      const unsigned char* srcb = gbase + (size_t)(ss * 4 + q) * CHUNK;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = *reinterpret_cast<const float*>(srcb + swz(h * 32 + i, lane));
      warp_arrive(bar(BAR_RING + nss + ss));  // the loads above are ordered before it
      const int rows_h = cur.rows - 32 * h;
      if (rows_h < 32)  // rows past the piece (other slices' rows / TMA zero fill)
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = i < rows_h ? v[i] : 0.0f;
      if (stats) {
        float s = 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) s = fmaf(v[i], v[i], s);
        if (!isfinite(s)) {  // Inf/NaN -- or an fp32 overflow of the squares: exact check
          double sd = 0.0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            bad |= !isfinite(v[i]);
            sd = fma((double)v[i], (double)v[i], sd);
          }
          sq += sd;
        } else {
          sq += (double)s;
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = tf32r(v[i]);
      if (xuse > 0) {
        if (tid == 0) TWAIT(bar(BAR_XT + 2 * xs + 1), (xuse - 1) & 1u, 3);
        else mbar_wait(bar(BAR_XT + 2 * xs + 1), (xuse - 1) & 1u);
      }
      tc_after();
      tmem_st32(tmem + lane_off + (uint32_t)(xs * 64 + 32 * h), v);
      tc_before();
      warp_arrive(bar(BAR_XT + 2 * xs));
      if (++xs == prm.nxs) { xs = 0; ++xuse; }
      if (++ss == nss) { ss = 0; rph ^= 1u; }
      const Unit nx = next_unit(cur);
      if (nx.p != cur.p && stats) {  // piece complete: sum of squares, non-finite flag
        const double tot = warp_sum(sq);
        const int anybad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
          red[warp] = tot;
          red[16 + warp] = anybad ? 1.0 : 0.0;
        }
        named_sync(1, NXT);
        if (tid == 0) {
          double t = 0.0;
          int b = 0;
          for (int w = 0; w < NXT / 32; ++w) {
            t += red[w];
            b |= red[16 + w] != 0.0;
          }
          (crank ? prm.xsq_hi : prm.xsq_part)[cur.p] = t;
          if (b) status_min(prm.status, ST_NONFINITE, prm.piece_slice[cur.p]);
        }
        named_sync(1, NXT);
        sq = 0.0;
        bad = 0;
      }
      cur = nx;
    }
  } else if (warp == MMA_WARP || warp == P2_WARP) {
    // ===================================================== MMA issuers (P1: MMA_WARP, P2: P2_WARP)
    // The whole warp runs the loop (warp-uniform descriptor arithmetic on the
    // uniform datapath: one add per MMA); elect.sync picks the issuing lane.
    // Descriptor words: lo = start>>4 | LBO(16 B)>>4 << 16, hi = SBO(1024)>>4 |
    // version 1 | SWIZZLE_128B; every operand address below is a compile-time
    // offset from a per-unit base.
    const uint32_t id1 = idesc_tf32(64, sp, 0, 0);   // X (smem, K-major) x B^T (K-major)
    const uint32_t id2 = idesc_tf32(128, n2, 0, 0);  // X^T (TMEM) x Y^T (K-major)
    const uint32_t dhi = (1024u >> 4) | (1u << 14) | (2u << 29);
    const uint32_t lbo = 1u << 16;
    const uint32_t ring_lo = (ring >> 4) | lbo, b_lo = (bsm >> 4) | lbo, y_lo = (ysm >> 4) | lbo;
    const uint32_t bch = (uint32_t)sp * 8;  // one 32-column chunk of B^T, in 16 B units
    uint32_t tcount = 0, rph = 0, xuse = 0;
    int ss = 0, pidx = 0, xs = 0;
    const uint32_t zcol = (uint32_t)prm.zcol, ycol = (uint32_t)prm.ycol;
#define MWAIT(barexpr, par, k)        \
  do {                                \
    if (lane == 0)                    \
      TWAIT(barexpr, par, k);         \
    else                              \
      mbar_wait(barexpr, par);        \
    __syncwarp();                     \
  } while (0)
    for (int p = pbeg; p < pend; ++p, ++pidx) {
      const int ntiles = (prm.piece_rows[p] + TM - 1) / TM;
      if (warp == MMA_WARP) {  // P1: Y(t) = X(t) B into accumulator t % 2
        MWAIT(bar(BAR_BFULL), (uint32_t)pidx & 1u, 4);
        tc_after();
        for (int t = 0; t < ntiles; ++t, ++tcount) {
          const uint32_t b = tcount & 1u;
          if (tcount >= 2) MWAIT(bar(BAR_YFREE + b), ((tcount >> 1) - 1) & 1u, 13);
          tc_after();
          for (int jb = 0; jb < nsup; ++jb) {
            MWAIT(bar(BAR_RING + ss), rph, 5);
            tc_after();
            const uint32_t a0 = ring_lo + (uint32_t)ss * (4 * CHUNK / 16);
            const uint32_t b0 = b_lo + (uint32_t)jb * 4 * bch;
            const unsigned long long tp1 = prm.dbg ? gtime() : 0ull;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                tc_mma_ss_e(tmem + ycol + 32 * b, a0 + ch * (CHUNK / 16) + kk * 2, b0 + ch * bch + kk * 2, dhi,
                            id1, (jb | ch | kk) != 0);
            tc_commit_e(bar(BAR_RING + nss + ss));
            if (prm.dbg && lane == 0) dacc[11] += gtime() - tp1;
            if (++ss == nss) { ss = 0; rph ^= 1u; }
          }
          if (t == ntiles - 1) tc_commit_e(bar(BAR_BFREE));
          tc_commit_e(bar(BAR_YFULL + b));
        }
      } else {  // P2: Z += X^T(t) Y(t)
        for (int t = 0; t < ntiles; ++t, ++tcount) {
          MWAIT(bar(BAR_YSFULL), tcount & 1u, 6);
          if (t == 0 && pidx > 0) MWAIT(bar(BAR_ZFREE), (uint32_t)(pidx - 1) & 1u, 7);
          tc_after();
          for (int jb = 0; jb < nsup; ++jb) {
            MWAIT(bar(BAR_XT + 2 * xs), xuse & 1u, 8);
            tc_after();
            const unsigned long long tp2 = prm.dbg ? gtime() : 0ull;
#pragma unroll
            for (int k = 0; k < TM / 8; ++k)
              tc_mma_ts_e(tmem + zcol + jb * 32, tmem + xs * 64 + k * 8, y_lo + (k >> 2) * (n2 * 8) + (k & 3) * 2,
                          dhi, id2, (t > 0 || k > 0) ? 1u : 0u);
            tc_commit_e(bar(BAR_XT + 2 * xs + 1));
            if (++xs == prm.nxs) { xs = 0; ++xuse; }
            if (prm.dbg && lane == 0) dacc[12] += gtime() - tp2;
          }
          tc_commit_e(bar(BAR_YSTFREE));
        }
        tc_commit_e(bar(BAR_ZFULL));
      }
    }
#undef MWAIT
  } else {
    // ===================================================== epilogue
    // main group (warps 9-12): Y -> rounded Y^T staging for P2, non-finite
    // flags (pass 1), the per-piece Z flush.  aux group (warps 15-18, pass 2
    // only): Y rows (coalesced through smem) and G = Y^T Y (fp64 DMMA), off
    // the staging -> P2 critical path.  Both read the Y accumulator.
    const bool aux = warp >= AUX0 / 32;
    const int q = warp & 3, et = aux ? tid - AUX0 : tid - EPI0;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    unsigned char* yb = gbase + prm.off_y;
    const bool do_g = prm.g_part != nullptr;
    const int ng = sp * sp;
    double gacc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    uint32_t tcount = 0;
    int pidx = 0;
    const int r = 16 * q + lane;  // M = 64 accumulator: row 16 q + l lives in TMEM lane 32 q + l (l < 16)
    for (int p = pbeg; p < pend && (!aux || auxon); ++p, ++pidx) {
      const int prows = prm.piece_rows[p];
      const int ntiles = (prows + TM - 1) / TM;
      for (int t = 0; t < ntiles; ++t, ++tcount) {
        const uint32_t b = tcount & 1u;
        if (et == 0 && !aux) TWAIT(bar(BAR_YFULL + b), (tcount >> 1) & 1u, 9);
        else mbar_wait(bar(BAR_YFULL + b), (tcount >> 1) & 1u);
        tc_after();
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + prm.ycol + 32 * b, v);
        tc_before();
        mbar_arrive(bar(BAR_YFREE + b));  // P1 may refill accumulator b once both groups read it
        if (csize > 1) {
          // J split: Y_t = own partial + the peer's (fp32 addition commutes, so
          // both CTAs form the same bits).  The main group sends its partial
          // into the peer's pbuf[b] once the peer has read tile t - 2 there.
          // pbuf[b] is column-major (TM rows per column): 16 lanes store / load
          // 64 contiguous bytes per column, conflict-free.  One remote arrive
          // per warp: __syncwarp orders the lanes' accesses before lane 0's
          // release at cluster scope.
          const uint32_t peer = crank ^ 1u;
          const uint32_t roff = b * (uint32_t)sp * TM + (uint32_t)r;
          if (!aux) {
            if (tcount >= 2) mbar_wait_cl(bar(BAR_PFREE + b), ((tcount >> 1) - 1) & 1u);
            if (lane < 16) {
              const uint32_t dst = cl_map(pbuf + roff * 4u, peer);
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (c < sp) cl_st_f32(dst + (uint32_t)(c * TM) * 4u, __uint_as_float(v[c]));
            }
            __syncwarp();
            if (lane == 0) cl_arrive_remote(cl_map(bar(BAR_PFULL + b), peer));
          }
          mbar_wait_cl(bar(BAR_PFULL + b), (tcount >> 1) & 1u);
          if (lane < 16)
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c < sp) v[c] = __float_as_uint(__uint_as_float(v[c]) + pbuf_f[roff + c * TM]);
          __syncwarp();
          if (lane == 0) cl_arrive_remote(cl_map(bar(BAR_PFREE + b), peer));
        }
        const int rows = min(TM, prows - t * TM);
        const bool valid = lane < 16 && r < rows;
        if (!aux) {
          if (tcount > 0) mbar_wait(bar(BAR_YSTFREE), (tcount - 1) & 1u);  // P2 of the previous tile done with Y^T
          if (lane < 16) {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              if (c >= sp) break;
              const float y = valid ? __uint_as_float(v[c]) : 0.0f;
              *reinterpret_cast<float*>(yb + (size_t)(r >> 5) * n2 * 128 + swz(c, r & 31)) = tf32r(y);
            }
          }
          fence_async_smem();
          tc_before();
          mbar_arrive(bar(BAR_YSFULL));
          if (!pass2 && valid) {  // Inf/NaN in X reach Y (B is dense Gaussian / Q_Z)
            bool nf = false;
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c < sp) nf |= !isfinite(__uint_as_float(v[c]));
            if (nf) status_min(prm.status, ST_NONFINITE, prm.piece_slice[p]);
          }
        } else {
          // Y rows through the shared row buffer: coalesced fp64 stores of the
          // tile's rows * sp contiguous values
          if (lane < 16)
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c < sp) yrow[r * (sp + 1) + c] = valid ? __uint_as_float(v[c]) : 0.0f;
          named_sync(4, NAUX);
          if (prm.y_out) {
            const int64_t o = (prm.piece_row0[p] + (int64_t)t * TM) * sp;
            float* yo32 = reinterpret_cast<float*>(prm.y_out) + o;
            double* yo = prm.y_out + o;
            for (int e = et; e < rows * sp; e += NAUX) {
              const int rr = e / sp, c = e - rr * sp;
              if (prm.y32) yo32[e] = yrow[rr * (sp + 1) + c];
              else yo[e] = (double)yrow[rr * (sp + 1) + c];
            }
          }
          if (do_g) {  // G += Y_t^T Y_t: fp64 DMMA m8n8k4 over 8x8 blocks of G
            const int nb = sp / 8, ew = et >> 5;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int blk = ew + 4 * s;
              if (blk < nb * nb) {
                const int bi = blk / nb, bj = blk - bi * nb;
                double c0 = gacc[2 * s], c1 = gacc[2 * s + 1];
#pragma unroll 4
                for (int kk = 0; kk < TM / 4; ++kk) {
                  const float* yr = yrow + (4 * kk + (lane & 3)) * (sp + 1);
                  dmma_8x8x4(c0, c1, (double)yr[8 * bi + (lane >> 2)], (double)yr[8 * bj + (lane >> 2)]);
                }
                gacc[2 * s] = c0;
                gacc[2 * s + 1] = c1;
              }
            }
          }
          named_sync(4, NAUX);  // yrow is rewritten for the next tile
        }
      }
      if (!aux) {  // piece complete: Z (TMEM lanes = columns of X) -> fp64 partial
        if (et == 0) TWAIT(bar(BAR_ZFULL), (uint32_t)pidx & 1u, 10);
        else mbar_wait(bar(BAR_ZFULL), (uint32_t)pidx & 1u);
        tc_after();
        double* out = prm.out_part + (size_t)p * J * sp;
        for (int jb = 0; jb < nsup; ++jb) {
          uint32_t z[32];
          tmem_ld32(tmem + lane_off + prm.zcol + jb * 32, z);
          const int j = j0 + jb * 128 + q * 32 + lane;
          if (j < J)
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c < sp) out[(size_t)j * sp + c] = (double)__uint_as_float(z[c]);
        }
        tc_before();
        mbar_arrive(bar(BAR_ZFREE));
      } else if (do_g) {
        const int nb = sp / 8, ew = et >> 5;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int blk = ew + 4 * s;
          if (blk < nb * nb) {
            const int bi = blk / nb, bj = blk - bi * nb;
            double* g = prm.g_part + (size_t)p * ng + (size_t)(8 * bi + (lane >> 2)) * sp + 8 * bj + 2 * (lane & 3);
            g[0] = gacc[2 * s];
            g[1] = gacc[2 * s + 1];
          }
          gacc[2 * s] = 0.0;
          gacc[2 * s + 1] = 0.0;
        }
      }
    }
  }
  if (prm.dbg) {
    // each slot is accounted by exactly one thread; the others add zeros
    if (tid == 0) dacc[15] = gtime() - t_start;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (dacc[k]) atomicAdd(prm.dbg + blockIdx.x * 16 + k, dacc[k]);
  }
  if (csize > 1) {  // no CTA leaves while its peer may still write its shared memory
    __syncwarp();
    cl_sync();
  }
  tc_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

// B (K x J x sp, fp64) -> per-slice images of the kernel's B shared memory:
// tf32 (rna), K-major SW128: 32-column chunk j/32, row c, swizzled granule
__global__ void __launch_bounds__(256) b_tile_kernel(const double* B, int64_t K, int J, int Jp, int sp, float* out) {
  // one block per slice (grid-stride over slices); thread = (row j, 4
  // consecutive columns c): 32-bit index math, 16-byte loads of B's row
  const int64_t per = (int64_t)Jp * sp;
  const int q4 = sp / 4;  // sp % 8 == 0
  for (int64_t k = blockIdx.x; k < K; k += gridDim.x) {
    const double* bk = B + k * (int64_t)J * sp;
    unsigned char* ok = reinterpret_cast<unsigned char*>(out + k * per);
    for (int e = threadIdx.x; e < Jp * q4; e += blockDim.x) {
      const int j = e / q4, c0 = (e - j * q4) * 4;
      double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
      if (j < J) {
        const double2 a = *reinterpret_cast<const double2*>(bk + (size_t)j * sp + c0);
        const double2 b = *reinterpret_cast<const double2*>(bk + (size_t)j * sp + c0 + 2);
        v = make_double4(a.x, a.y, b.x, b.y);
      }
      unsigned char* row = ok + (size_t)(j >> 5) * sp * 128;
      *reinterpret_cast<float*>(row + swz(c0, j & 31)) = tf32r((float)v.x);
      *reinterpret_cast<float*>(row + swz(c0 + 1, j & 31)) = tf32r((float)v.y);
      *reinterpret_cast<float*>(row + swz(c0 + 2, j & 31)) = tf32r((float)v.z);
      *reinterpret_cast<float*>(row + swz(c0 + 3, j & 31)) = tf32r((float)v.w);
    }
  }
}

// xsq[p] += hi[p]: the CTA pair's two column halves of each piece's sum of squares
__global__ void add_pieces_kernel(double* xsq, const double* hi, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) xsq[i] += hi[i];
}

}  // namespace tcs

namespace {
// 0: tf32 tensor cores when eligible (opt-in: single-pass tf32 products),
// 1: fp32 FFMA kernel, 2 (default): fp64 DMMA products on the exactly upcast
// values where the warp-specialised pass is eligible (J <= 512), else the FFMA
// kernel -- both at least the fp32 mode BASELINE.json states.
// DP2_SKETCH_ENGINE overrides the default at load time.
int initial_engine() {
  const char* e = getenv("DP2_SKETCH_ENGINE");
  return e && *e ? atoi(e) : 2;
}
int g_engine = initial_engine();
}

void set_sketch_engine(int e) { g_engine = e; }
int sketch_engine() { return g_engine; }

// shared-memory plan; 0 when the shape is not eligible for the tensor-core pass
// J <= 512: one CTA per segment over all columns; 512 < J <= 1024: a CTA
// pair (cluster of 2) per two segments, each CTA over JH = Jp / 2 columns
// (TMEM holds X^T and Z of at most 512 columns: 64 + 32 TMEM columns per
// 128 columns of X, plus the Y accumulators)
static size_t tc_plan(int J, int sp, tcs::Params* prm) {
  if (J < 1 || J > 1024 || sp < 8 || sp > 32 || sp % 8) return 0;
  const int csize = J > 512 ? 2 : 1;
  const int Jp = (J + 128 * csize - 1) / (128 * csize) * (128 * csize), JH = Jp / csize;
  const int n2 = (sp + 15) / 16 * 16;
  const size_t pb = csize > 1 ? (size_t)2 * tcs::TM * sp * 4 : 0;
  const size_t fixed = (size_t)sp * JH * 4 + (size_t)2 * n2 * 128 + (size_t)tcs::TM * (sp + 1) * 4 + pb + 16;
  const size_t cap = 227 * 1024 - 1024 - fixed;
  int nslot = (int)(cap / tcs::CHUNK) / 4 * 4;
  nslot = nslot > 24 ? 24 : nslot;
  if (nslot < 8) return 0;
  const int nss = nslot / 4;
  prm->J = J;
  prm->Jp = Jp;
  prm->JH = JH;
  prm->csize = csize;
  prm->sp = sp;
  prm->n2 = n2;
  prm->nslot = nslot;
  prm->nsup = JH / 128;
  // TMEM: Z 32 nsup + Y 64 columns, the rest (<= 8 slots) X^T
  prm->nxs = std::min(8, (512 - 32 * prm->nsup - 64) / 64);
  prm->zcol = 64 * prm->nxs;
  prm->ycol = prm->zcol + 32 * prm->nsup;
  prm->off_b = (uint32_t)nslot * tcs::CHUNK;
  prm->off_y = prm->off_b + (uint32_t)sp * JH * 4;
  prm->off_yrow = prm->off_y + 2u * n2 * 128;
  prm->off_pbuf = (prm->off_yrow + (uint32_t)tcs::TM * (sp + 1) * 4 + 15u) & ~15u;
  prm->off_bar = (prm->off_pbuf + (uint32_t)pb + 7u) & ~7u;
  return prm->off_bar + 8u * (tcs::BAR_RING + 2 * nss) + 1024;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

bool sketch_tc_eligible(const dp2_store* st, int sp) {
  tcs::Params prm{};
  return g_engine == 0 && st->dtype == DP2_F32 && st->ldx % 4 == 0 &&
         reinterpret_cast<uintptr_t>(st->X) % 16 == 0 && st->total_rows < (1ll << 31) &&
         tc_plan((int)st->J, sp, &prm) != 0 && encode_fn() != nullptr;
}

// per-device scratch (grown on demand, kept): the pre-tiled B images (slot
// 0) and rank 1's per-piece sums of squares of the CTA-pair pass (slot 1)
static float* btile_scratch(size_t bytes, cudaError_t* err, int slot = 0) {
  static float* bufs[2][64] = {};
  static size_t caps[2][64] = {};
  float** buf = bufs[slot];
  size_t* cap = caps[slot];
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

cudaError_t run_sketch_tc(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                          double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part, bool y32) {
  tcs::Params prm{};
  prm.y32 = y32 ? 1 : 0;
  const size_t smem = tc_plan((int)st->J, sp, &prm);
  if (smem == 0 || encode_fn() == nullptr) return cudaErrorInvalidValue;
  // B images: one bulk copy per piece replaces per-element conversion in the kernel
  prm.bbytes = (uint32_t)prm.JH * sp * 4;  // the part one CTA loads
  prm.bstride = (uint32_t)prm.Jp * sp;     // floats per slice image
  prm.nseg = st->nseg;
  cudaError_t be;
  float* bt = btile_scratch((size_t)st->K * prm.bstride * 4, &be);
  if (!bt) return be;
  if (prm.csize > 1 && xsq_part) {
    prm.xsq_hi = reinterpret_cast<double*>(btile_scratch((size_t)st->npieces * 8, &be, 1));
    if (!prm.xsq_hi) return be;
  }
  tcs::b_tile_kernel<<<(unsigned)(st->K < 2048 ? st->K : 2048), 256, 0, stream>>>(B, st->K, prm.J, prm.Jp, sp, bt);
  prm.btile = bt;
  // X as a 2-D tensor (J columns, total_rows rows, row pitch ldx*4 B); boxes
  // of 32 columns x 64 rows land in shared memory with the 128 B swizzle
  CUtensorMap xmap;
  const cuuint64_t dims[2] = {(cuuint64_t)st->J, (cuuint64_t)st->total_rows};
  const cuuint64_t strides[1] = {(cuuint64_t)st->ldx * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)tcs::TM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult cr = encode_fn()(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(st->X), dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    note_error("cuTensorMapEncodeTiled failed for the fp32 store");
    return cudaErrorInvalidValue;
  }
  prm.X = static_cast<const float*>(st->X);
  prm.ldx = st->ldx;
  prm.B = B;
  prm.piece_slice = st->piece_slice;
  prm.piece_row0 = st->piece_row0;
  prm.piece_rows = st->piece_rows;
  prm.seg_begin = st->seg_begin;
  prm.out_part = out_part;
  prm.y_out = y_out;
  prm.xsq_part = xsq_part;
  prm.g_part = g_part;
  prm.status = status;
  cudaError_t e = cudaFuncSetAttribute(tcs::sketch_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  static const bool debug = getenv("DP2_TC_DEBUG") != nullptr;
  if (debug) {
    cudaMalloc(&prm.dbg, (size_t)st->nseg * 16 * sizeof(unsigned long long));
    cudaMemsetAsync(prm.dbg, 0, (size_t)st->nseg * 16 * sizeof(unsigned long long), stream);
  }
  if (prm.csize == 1) {
    tcs::sketch_tc_kernel<<<st->nseg, tcs::NTHREADS, smem, stream>>>(prm, xmap);
    e = cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(2 * ((st->nseg + 1) / 2)));
    cfg.blockDim = dim3(tcs::NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (getenv("DP2_TC_DEBUG")) {
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, (void*)tcs::sketch_tc_kernel, &cfg);
      fprintf(stderr, "[dp2 tc] CTA pairs: %u launched, %d co-resident, smem %zu, JH %d, nslot %d\n",
              cfg.gridDim.x / 2, ncl, smem, prm.JH, prm.nslot);
    }
    e = cudaLaunchKernelEx(&cfg, tcs::sketch_tc_kernel, prm, xmap);
    if (e == cudaSuccess && xsq_part) {
      tcs::add_pieces_kernel<<<(unsigned)((st->npieces + 255) / 256), 256, 0, stream>>>(xsq_part, prm.xsq_hi,
                                                                                       st->npieces);
      e = cudaGetLastError();
    }
  }
  if (debug && e == cudaSuccess) {
    std::vector<unsigned long long> h((size_t)st->nseg * 16);
    cudaMemcpyAsync(h.data(), prm.dbg, h.size() * 8, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    const char* names[16] = {"tma.empty", "b.bfree", "xt.full", "xt.xtfree", "mma.bfull", "mma.full", "mma.ysfull",
                             "mma.zfree", "mma.xtfull", "epi.yfull", "epi.zfull", "mma.p1issue", "mma.p2issue", "mma.yfree", "", "total"};
    fprintf(stderr, "[dp2 tc] pass (%s) mean us per CTA:", y_out ? "2" : "1");
    for (int k = 0; k < 16; ++k) {
      if (!names[k][0]) continue;
      double m = 0;
      for (int c = 0; c < st->nseg; ++c) m += h[(size_t)c * 16 + k];
      fprintf(stderr, " %s=%.1f", names[k], m / st->nseg / 1e3);
    }
    fprintf(stderr, "\n");
    cudaFree(prm.dbg);
  }
  return e;
}

}  // namespace dp2
