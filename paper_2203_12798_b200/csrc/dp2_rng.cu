// Sketch matrices Omega_k on the device, bit-exact with the reference's
// Generator(PCG64(derived_seed(seed, k))).standard_normal((J, s_k))
// (P/linalg.py:122-123, 187-194).
//
//   SeedSequence([seed, k]) -> 1 uint64 (derived seed)   numpy SeedSequence hash
//   SeedSequence(derived)   -> 4 uint64 -> PCG64 state/inc (pcg setseq srandom)
//   PCG64 XSL-RR 128/64 stream -> 256-layer ziggurat (tables: dp2_ziggurat_tables.h)
//
// Warps walk segments of each slice's stream (32 draws in flight via
// jump-ahead, segments stitched exactly, see omega_emit_kernel).  The fast path (>99% of draws: one 64-bit
// output, one multiply) is exact IEEE arithmetic.  The rare
// tail branch (layer 0, about 2.6e-4 of draws) needs log1p, whose last bit
// differs between libm implementations, so every tail event is recorded
// (output index, the uniforms it consumed) and the host replays it with
// NumPy's own log1p and patches the value (paper_2203_12798_b200/rng.py).
// Wedge tests use explicit non-fused roundings (__dmul_rn/__dadd_rn) to
// match the reference's C evaluation order.
#include "dp2_common.cuh"
#include "dp2_internal.h"
#include "dp2_ziggurat_tables.h"

#include <algorithm>
#include <cstdlib>

namespace dp2 {

namespace {
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr uint64_t kPcgMulLo = 0x4385DF649FCCF645ull, kPcgMulHi = 0x2360ED051FC65DA4ull;
}  // namespace

__host__ __device__ inline int u64_words(uint64_t v, uint32_t* w) {
  if (v == 0) { w[0] = 0; return 1; }
  int n = 0;
  while (v) { w[n++] = (uint32_t)v; v >>= 32; }
  return n;
}

// numpy SeedSequence(entropy words).generate_state(2 * n64 uint32) as n64 uint64
__host__ __device__ inline void seed_sequence(const uint32_t* ent, int n_ent, int n64, uint64_t* out) {
  uint32_t pool[4];
  uint32_t hc = kInitA;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= kMultA;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    r ^= r >> 16;
    return r;
  };
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < n_ent; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t hb = kInitB;
  for (int i = 0; i < 2 * n64; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    if (i & 1) out[i / 2] |= (uint64_t)v << 32;
    else out[i / 2] = v;
  }
}

__host__ __device__ inline uint64_t derived_seed_u64(uint64_t seed, uint64_t index) {
  uint32_t ent[4];
  int n = u64_words(seed, ent);
  n += u64_words(index, ent + n);
  uint64_t out[1];
  seed_sequence(ent, n, 1, out);
  return out[0];
}

struct Pcg {
  uint64_t slo, shi, ilo, ihi;
  __device__ void step() {
    const uint64_t lo = slo * kPcgMulLo;
    uint64_t hi = __umul64hi(slo, kPcgMulLo) + slo * kPcgMulHi + shi * kPcgMulLo;
    const uint64_t nlo = lo + ilo;
    hi += ihi + (nlo < lo ? 1ull : 0ull);
    slo = nlo;
    shi = hi;
  }
  __device__ uint64_t next() {
    step();
    const uint64_t x = shi ^ slo;
    const unsigned rot = (unsigned)(shi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ double next_double() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
  // pcg64_set_seed / pcg_setseq_128_srandom_r on SeedSequence(seed).generate_state(4, uint64)
  __device__ void seed(uint64_t s) {
    uint32_t ent[2];
    const int n = u64_words(s, ent);
    uint64_t v[4];
    seed_sequence(ent, n, 4, v);
    // initstate = v0:v1 (hi:lo), initseq = v2:v3; inc = (initseq << 1) | 1
    ihi = (v[2] << 1) | (v[3] >> 63);
    ilo = (v[3] << 1) | 1ull;
    slo = 0;
    shi = 0;
    step();
    const uint64_t lo = slo + v[1];
    shi = shi + v[0] + (lo < slo ? 1ull : 0ull);
    slo = lo;
    step();
  }
};

struct TailRec {          // one layer-0 tail event, replayed on the host
  int64_t slice;          // local slice index
  int64_t index;          // output index within the slice (C order of J x s_k)
  int32_t attempts;       // accepted on this attempt (1..kTailAttempts)
  int32_t negative;       // output sign
  double u[8];            // (u1, u2) per attempt
};
constexpr int kTailAttempts = 4;

// 128-bit LCG arithmetic (mod 2^128) for PCG64 jump-ahead
struct U128 {
  uint64_t lo, hi;
};
__device__ inline U128 mul128(U128 a, U128 b) {
  return {a.lo * b.lo, __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo};
}
__device__ inline U128 add128(U128 a, U128 b) {
  const uint64_t lo = a.lo + b.lo;
  return {lo, a.hi + b.hi + (lo < a.lo ? 1ull : 0ull)};
}
__device__ inline uint64_t pcg_out(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// (A^p, S_p = sum_{i<p} A^i) of the PCG64 LCG (pcg_advance_lcg_128 with a
// unit increment): the state p steps after x is A^p x + S_p inc.
__device__ inline void lcg_coeffs(uint64_t p, U128& am, U128& as) {
  am = U128{1, 0};
  as = U128{0, 0};
  U128 cm{kPcgMulLo, kPcgMulHi}, cs{1, 0};
  while (p) {
    if (p & 1) {
      am = mul128(am, cm);
      as = add128(mul128(as, cm), cs);
    }
    cs = mul128(add128(cm, U128{1, 0}), cs);
    cm = mul128(cm, cm);
    p >>= 1;
  }
}
__device__ inline U128 lcg_jump(U128 x, U128 inc, uint64_t p) {
  U128 am, as;
  lcg_coeffs(p, am, as);
  return add128(mul128(am, x), mul128(as, inc));
}

struct ZigTabs {
  uint64_t ki[256];
  double wi[256], fi[256];
};
__device__ inline void load_zig(ZigTabs& T) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    T.ki[i] = kZigKi[i];
    T.wi[i] = __longlong_as_double((long long)kZigWiBits[i]);
    T.fi[i] = __longlong_as_double((long long)kZigFiBits[i]);
  }
  __syncthreads();
}

// Per-slice stream: inc and the state of draw 0 (Pcg::next steps, then outputs).
struct SliceStream {
  U128 b, inc;
};
// raw: PCG64(seed) itself (one stream, e.g. the stage-2 Omega); else
// PCG64(derived_seed(seed, gid)) (the per-slice streams, P/linalg.py:187-194)
__device__ inline SliceStream slice_stream(uint64_t seed, uint64_t gid, bool raw = false) {
  Pcg g;
  g.seed(raw ? seed : derived_seed_u64(seed, gid));
  const U128 inc{g.ilo, g.ihi};
  return SliceStream{add128(mul128(U128{g.slo, g.shi}, U128{kPcgMulLo, kPcgMulHi}), inc), inc};
}

// Sequential ziggurat attempt starting at draw p (one thread): advances p past
// the draws it consumes, returns the number of normals produced (0 or 1).
__device__ int zig_attempt_seq(const ZigTabs& T, const SliceStream& S, int64_t& p) {
  const U128 sp = lcg_jump(S.b, S.inc, (uint64_t)p);
  uint64_t r = pcg_out(sp);
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
  if (rabs < T.ki[idx]) {
    p += 1;
    return 1;
  }
  Pcg h;
  h.slo = sp.lo;
  h.shi = sp.hi;
  h.ilo = S.inc.lo;
  h.ihi = S.inc.hi;
  if (idx == 0) {
    int a = 0;
    for (;;) {
      const double u1 = h.next_double(), u2 = h.next_double();
      ++a;
      const double xx = __dmul_rn(-kZigInvR, log1p(-u1));
      const double yy = -log1p(-u2);
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) break;
    }
    p += 1 + 2 * a;
    return 1;
  }
  const double x = __dmul_rn((double)rabs, T.wi[idx]);
  const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(T.fi[idx - 1], -T.fi[idx]), h.next_double()), T.fi[idx]);
  p += 2;
  return lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x)) ? 1 : 0;
}

// Warp parse of one slice's stream from draw p0 (an attempt start) over the
// attempts starting before p_end, normals numbered from i0 (stops at total).
// Lane l holds the generator state of draw base + l (state_{p+l} = A^l
// state_p + inc S_l), so a batch of 32 consecutive draws is produced in
// parallel.  The ziggurat parse of the draw stream is sequential but almost
// always one draw per normal: every round, the lanes from the current
// attempt start up to the first draw that misses the fast rectangle are
// normals at once (ballot + prefix count); that wedge/tail draw is resolved
// by its lane with its own sequential generator, which then broadcasts its
// state so the warp re-bases behind the consumed draws.  Returns the normals
// produced (n_out) and the first attempt start >= p_end (p_out).  EMIT writes
// the normals (row-major J x s_k in an sp-wide row) and records tail events.
struct LaneJump {
  U128 Al, Cl, A32, C32;
};
template <bool EMIT>
__device__ void zig_parse(const ZigTabs& T, const SliceStream& S, const LaneJump& LJ, int lane, int64_t p0,
                          int64_t p_end, int64_t i0, int64_t total, double* o, int s, int sp, int64_t k,
                          TailRec* recs, int cap, int32_t* nrec, int32_t* redo, int64_t& n_out, int64_t& p_out) {
  const U128 A{kPcgMulLo, kPcgMulHi};
  if (p0 >= p_end) {
    n_out = 0;
    p_out = p0;
    return;
  }
  U128 st = add128(mul128(lcg_jump(S.b, S.inc, (uint64_t)p0), LJ.Al), LJ.Cl);
  int64_t base = p0, i = i0;
  int start = 0;
  p_out = p_end;
  // (row, column) of normal i, advanced incrementally (advance by d <= 33)
  int64_t row0 = EMIT ? i0 / s : 0;
  int col0 = EMIT ? (int)(i0 - row0 * s) : 0;
  // c / s by a 32-bit reciprocal: floor(c ceil(2^32/s) / 2^32) = floor(c/s)
  // exactly for c < 2^32 / s (here c < s + 64); s = 1 separately
  const uint32_t rcp_s = s > 1 ? (uint32_t)((0x100000000ull + (uint64_t)s - 1) / (uint64_t)s) : 0u;
  auto divs = [&](int c) { return s > 1 ? (int)__umulhi((uint32_t)c, rcp_s) : c; };
  auto advance = [&](int d) {
    if (!EMIT) return;
    col0 += d;
    const int q = divs(col0);
    col0 -= q * s;
    row0 += q;
  };
  auto at = [&](int off) -> double* {  // element of normal i + off (0 <= off < 32)
    const int c = col0 + off;
    const int q = divs(c);
    return o + (row0 + q) * sp + (c - q * s);
  };
  while (i < total) {
    const int64_t remp = p_end - base;
    const int lim = remp < 32 ? (int)remp : 32;
    uint64_t r = pcg_out(st);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, T.wi[idx]);
    if (sign) x = -x;
    const bool fast = rabs < T.ki[idx];
    unsigned slow = __ballot_sync(0xffffffffu, !fast) & (0xffffffffu << start);
    if (lim < 32) slow &= (1u << lim) - 1u;
    const int f = slow ? __ffs(slow) - 1 : lim;
    // lanes start .. f-1 are one-draw normals
    if (EMIT && lane >= start && lane < f) {
      if (i + (lane - start) < total) *at(lane - start) = x;
    }
    i += f - start;
    advance(f - start);
    if (f == lim) {
      if (lim < 32) break;  // reached p_end exactly
      st = add128(mul128(st, LJ.A32), LJ.C32);  // batch exhausted: every lane 32 draws on
      base += 32;
      start = 0;
      continue;
    }
    if (i >= total) break;
    // draw f misses the rectangle: its lane resolves the wedge / tail
    int produced = 0, consumed = 1;
    U128 last{0, 0};
    if (lane == f) {
      Pcg h;
      h.slo = st.lo;
      h.shi = st.hi;
      h.ilo = S.inc.lo;
      h.ihi = S.inc.hi;
      if (idx == 0) {
        TailRec rec;
        rec.slice = k;
        rec.index = i;
        rec.negative = (int)((rabs >> 8) & 1);
        int a = 0;
        double val = 0.0;
        for (;;) {
          const double u1 = h.next_double(), u2 = h.next_double();
          if (a < kTailAttempts) {
            rec.u[2 * a] = u1;
            rec.u[2 * a + 1] = u2;
          }
          ++a;
          const double xx = __dmul_rn(-kZigInvR, log1p(-u1));
          const double yy = -log1p(-u2);
          if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
            val = rec.negative ? -(kZigR + xx) : kZigR + xx;
            break;
          }
        }
        rec.attempts = a;
        consumed = 1 + 2 * a;
        if (EMIT) {
          if (a > kTailAttempts) {
            redo[k] = 1;
          } else {
            const int slot = atomicAdd(nrec, 1);
            if (slot < cap) recs[slot] = rec;
            else redo[k] = 1;
          }
          *at(0) = val;
        }
        produced = 1;
      } else {
        const double f0 = T.fi[idx - 1];
        const double f1 = T.fi[idx];
        const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(f0, -f1), h.next_double()), f1);
        consumed = 2;
        if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
          if (EMIT) *at(0) = x;
          produced = 1;
        }
      }
      last = U128{h.slo, h.shi};  // state of the last consumed draw
    }
    produced = __shfl_sync(0xffffffffu, produced, f);
    consumed = __shfl_sync(0xffffffffu, consumed, f);
    i += produced;
    advance(produced);
    const int nstart = f + consumed;
    if (base + nstart >= p_end) {
      p_out = base + nstart;
      break;
    }
    if (nstart < 32) {
      start = nstart;  // lanes still hold the draws behind the consumed ones
      continue;
    }
    // re-base: draw (base + nstart) = A * last + inc, then lane offsets
    last.lo = __shfl_sync(0xffffffffu, last.lo, f);
    last.hi = __shfl_sync(0xffffffffu, last.hi, f);
    st = add128(mul128(add128(mul128(last, A), S.inc), LJ.Al), LJ.Cl);
    base += nstart;
    start = 0;
  }
  n_out = i - i0;
}

// Segment length in draws: a normal takes ~1.013 draws on average (wedge
// uniforms, rejections, tails), so segments sized on 1.03 x the normal count
// leave the last one (which runs until the stream's normals are complete)
// without a long overhang; trailing segments past the end exit at once.
__device__ inline int64_t seg_len(int64_t total, int G) {
  return G == 1 ? total : (total * 103 + 100 * (int64_t)G - 1) / (100 * (int64_t)G);
}

__device__ inline LaneJump lane_jump(int lane, U128 inc) {
  LaneJump L;
  U128 sl, s32;
  lcg_coeffs((uint64_t)lane, L.Al, sl);
  lcg_coeffs(32, L.A32, s32);
  L.Cl = mul128(inc, sl);
  L.C32 = mul128(inc, s32);
  return L;
}

// Segment-parallel Omega: slice k's draw stream is cut into G segments of L_k
// = ceil(J s_k / G) draws.  omega_count_kernel parses segment g < G-1
// speculatively from its first draw gL (assuming it starts an attempt) and
// records (normals, first attempt start >= (g+1)L).  omega_emit_kernel
// recovers, for its segment, the true start and output offset by scanning
// the earlier segments' records: a segment whose true start t differs from hL
// (the previous attempt ran over the boundary, ~1% of segments) is repaired
// by stepping the true and the speculative parse one attempt at a time until
// they meet -- from there they coincide -- or the true one leaves the
// segment.  It then parses from its true start and writes.  The result is the
// sequential stream exactly.
__global__ void __launch_bounds__(128) omega_count_kernel(uint64_t seed, int64_t K, int J, const int32_t* s_k,
                                                          int G, const int64_t* slice_ids, int64_t* seg_n,
                                                          int64_t* seg_end, int raw) {
  __shared__ ZigTabs T;
  load_zig(T);
  const int lane = threadIdx.x & 31;
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= K * (G - 1)) return;
  const int64_t k = w / (G - 1);
  const int g = (int)(w - k * (G - 1));
  const int s = s_k[k];
  const int64_t total = (int64_t)J * s, L = seg_len(total, G);
  const SliceStream S = slice_stream(seed, slice_ids ? (uint64_t)slice_ids[k] : (uint64_t)k, raw != 0);
  const LaneJump LJ = lane_jump(lane, S.inc);
  int64_t n, e;
  zig_parse<false>(T, S, LJ, lane, g * L, (g + 1) * L, 0, INT64_MAX, nullptr, s, 0, k, nullptr, 0, nullptr,
                   nullptr, n, e);
  if (lane == 0) {
    seg_n[k * G + g] = n;
    seg_end[k * G + g] = e;
  }
}

__global__ void __launch_bounds__(128) omega_emit_kernel(uint64_t seed, int64_t K, int J, const int32_t* s_k,
                                                         int sp, int G, const int64_t* slice_ids,
                                                         const int64_t* seg_n, const int64_t* seg_end, double* out,
                                                         TailRec* recs, int cap, int32_t* nrec, int32_t* redo,
                                                         int raw) {
  __shared__ ZigTabs T;
  load_zig(T);
  const int lane = threadIdx.x & 31;
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= K * G) return;
  const int64_t k = w / G;
  const int g = (int)(w - k * G);
  const int s = s_k[k];
  const int64_t total = (int64_t)J * s, L = seg_len(total, G);
  double* o = out + (size_t)k * J * sp;
  if (s < sp) {  // zero padding columns: the slice's J x (sp - s) block, flat over its G warps
    const int pw = sp - s;
    for (int e = g * 32 + lane; e < J * pw; e += 32 * G) {
      const int j = e / pw;
      o[(int64_t)j * sp + s + (e - j * pw)] = 0.0;
    }
  }
  const SliceStream S = slice_stream(seed, slice_ids ? (uint64_t)slice_ids[k] : (uint64_t)k, raw != 0);
  // true start t and output offset O of segment g.  Warp-parallel: lane
  // sums the counts of segments h = lane, lane + 32, ... < g; a segment whose
  // predecessor ended past its first draw (misaligned) is repaired by its
  // lane, walking the true and the speculative attempts until they meet --
  // from there they coincide, so its end and every later start are
  // unchanged.  If a walk leaves the segment first (its end moves; never
  // observed), the starts are rebuilt by the sequential scan.
  int64_t part = 0;
  int lost = 0;
  for (int h = lane; h < g; h += 32) {
    int64_t n = seg_n[k * G + h];
    const int64_t t = h == 0 ? 0 : seg_end[k * G + h - 1];
    if (t != h * L) {
      const int64_t end_h = (h + 1) * L;
      int64_t pt = t, ps = h * L, ct = 0, cs = 0;
      for (;;) {
        if (pt >= end_h) {
          lost = 1;
          break;
        }
        if (pt == ps) {
          n = n - cs + ct;
          break;
        }
        if (ps < pt) cs += zig_attempt_seq(T, S, ps);
        else ct += zig_attempt_seq(T, S, pt);
      }
    }
    part += n;
  }
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  int64_t O = part, t = g == 0 ? 0 : seg_end[k * G + g - 1];
  if (__any_sync(0xffffffffu, lost)) {  // sequential scan (every lane alike)
    t = 0;
    O = 0;
    for (int h = 0; h < g; ++h) {
      const int64_t end_h = (h + 1) * L;
      int64_t n = seg_n[k * G + h], e = seg_end[k * G + h];
      if (t != h * L) {
        int64_t pt = t, ps = h * L, ct = 0, cs = 0;
        for (;;) {
          if (pt >= end_h) {
            n = ct;
            e = pt;
            break;
          }
          if (pt == ps) {
            n = n - cs + ct;
            break;
          }
          if (ps < pt) cs += zig_attempt_seq(T, S, ps);
          else ct += zig_attempt_seq(T, S, pt);
        }
      }
      O += n;
      t = e;
    }
  }
  if (O >= total) return;
  const LaneJump LJ = lane_jump(lane, S.inc);
  int64_t n, e;
  zig_parse<true>(T, S, LJ, lane, t, g == G - 1 ? INT64_MAX : (g + 1) * L, O, total, o, s, sp, k, recs, cap, nrec,
                  redo, n, e);
}

cudaError_t run_omega(uint64_t seed, int64_t K, int J, const int32_t* s_k, int sp, const int64_t* slice_ids,
                      double* out, void* recs, int cap, int32_t* nrec, int32_t* redo, cudaStream_t st,
                      int* launches, bool raw) {
  cudaMemsetAsync(nrec, 0, sizeof(int32_t), st);
  cudaMemsetAsync(redo, 0, sizeof(int32_t) * K, st);
  // segments per slice: about 48 warps per SM in flight, segments >= 512 draws
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Segments per stream: with >= 4 streams per SM one warp per stream keeps
  // the GPU busy (a count pass over all draws costs more than the latency it
  // hides); fewer streams (the stage-2 Omega is one) split into segments of
  // >= 512 draws, ~48 warps per SM.  DP2_OMEGA_SEGMENTS overrides.
  const char* env = getenv("DP2_OMEGA_SEGMENTS");
  const int64_t want = env ? std::max(1, atoi(env))
                           : (K >= (int64_t)sms * 4 ? 1 : ((int64_t)sms * 48 + K - 1) / K);
  const int64_t cap_len = std::max<int64_t>(1, (int64_t)J * sp / 512);
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>({want, cap_len, 1024}));
  int64_t* seg = nullptr;
  if (G > 1) {
    // grow-only per-device scratch (a stream-ordered pool allocation is
    // returned to the driver at every synchronisation and re-mapped next call)
    static int64_t* cache[64] = {};
    static size_t cache_bytes[64] = {};
    const size_t need = sizeof(int64_t) * 2 * K * G;
    if (dev < 64 && cache_bytes[dev] < need) {
      cudaStreamSynchronize(st);  // the old buffer may still be in use
      if (cache[dev]) cudaFree(cache[dev]);
      cache[dev] = nullptr;
      cache_bytes[dev] = 0;
      cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&cache[dev]), std::max<size_t>(need, 1 << 16));
      if (e != cudaSuccess) return e;
      cache_bytes[dev] = std::max<size_t>(need, 1 << 16);
    }
    if (dev >= 64) return cudaErrorInvalidDevice;
    seg = cache[dev];
    const int64_t wc = K * (G - 1);
    omega_count_kernel<<<(unsigned)((wc + 3) / 4), 128, 0, st>>>(seed, K, J, s_k, G, slice_ids, seg, seg + K * G,
                                                                 raw ? 1 : 0);
  }
  const int64_t we = K * G;
  omega_emit_kernel<<<(unsigned)((we + 3) / 4), 128, 0, st>>>(seed, K, J, s_k, sp, G, slice_ids, seg,
                                                              seg ? seg + K * G : nullptr, out,
                                                              static_cast<TailRec*>(recs), cap, nrec, redo,
                                                              raw ? 1 : 0);
  if (launches) *launches = G > 1 ? 2 : 1;
  return cudaGetLastError();
}

size_t tail_record_bytes() { return sizeof(TailRec); }
uint64_t derived_seed_host(uint64_t seed, uint64_t index) { return derived_seed_u64(seed, index); }

}  // namespace dp2
