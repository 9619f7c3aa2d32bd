// Sketch matrices Omega_k on the device, bit-exact with the reference's
// Generator(PCG64(derived_seed(seed, k))).standard_normal((J, s_k))
// (P/linalg.py:122-123, 187-194).
//
//   SeedSequence([seed, k]) -> 1 uint64 (derived seed)   numpy SeedSequence hash
//   SeedSequence(derived)   -> 4 uint64 -> PCG64 state/inc (pcg setseq srandom)
//   PCG64 XSL-RR 128/64 stream -> 256-layer ziggurat (tables: dp2_ziggurat_tables.h)
//
// One warp per slice walks that slice's stream (32 draws in flight via
// jump-ahead, see omega_kernel).  The fast path (>99% of draws: one 64-bit
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

// One warp per slice.  Lane l holds the generator state of draw base + l
// (state_{p+l} = A^l state_p + inc * (1 + A + ... + A^(l-1))), so a batch of
// 32 consecutive 64-bit draws is produced in parallel.  The ziggurat parse of
// the draw stream is inherently sequential but almost always one draw per
// normal: every round, the lanes from the current normal start up to the
// first draw that misses the fast rectangle emit their normals at once
// (ballot + prefix count); that one wedge/tail draw is resolved by its lane
// with its own sequential generator, which then broadcasts its state so the
// warp re-bases behind the consumed draws.  The output is the reference's
// stream exactly.
__global__ void __launch_bounds__(128) omega_kernel(uint64_t seed, int64_t K, int J, const int32_t* s_k, int sp,
                                                    const int64_t* slice_ids, double* out, TailRec* recs,
                                                    int cap, int32_t* nrec, int32_t* redo) {
  __shared__ uint64_t ki_s[256];
  __shared__ double wi_s[256], fi_s[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    ki_s[i] = kZigKi[i];
    wi_s[i] = __longlong_as_double((long long)kZigWiBits[i]);
    fi_s[i] = __longlong_as_double((long long)kZigFiBits[i]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= K) return;
  // jump constants: A^lane, S_lane = sum_{i<lane} A^i, and the same for 32
  const U128 A{kPcgMulLo, kPcgMulHi};
  U128 Al{1, 0}, Sl{0, 0}, P{1, 0}, S{0, 0};
  for (int i = 0; i < 32; ++i) {
    if (i == lane) {
      Al = P;
      Sl = S;
    }
    S = add128(S, P);
    P = mul128(P, A);
  }
  const U128 A32 = P, S32 = S;
  const uint64_t gid = slice_ids ? (uint64_t)slice_ids[k] : (uint64_t)k;
  Pcg g;
  g.seed(derived_seed_u64(seed, gid));
  const U128 inc{g.ilo, g.ihi};
  const U128 Cl = mul128(inc, Sl), C32 = mul128(inc, S32);
  // state of draw 0 (Pcg::next steps, then outputs)
  U128 b = add128(mul128(U128{g.slo, g.shi}, A), inc);
  U128 st = add128(mul128(b, Al), Cl);
  const int s = s_k[k];
  double* o = out + (size_t)k * J * sp;
  const int64_t total = (int64_t)J * s;
  for (int64_t e = lane; e < (int64_t)J * (sp - s); e += 32)  // zero padding columns
    o[(e / (sp - s)) * sp + s + e % (sp - s)] = 0.0;
  int64_t i = 0;  // normals emitted
  int start = 0;  // lane of the next normal start in this batch
  // (row, column) of normal i, advanced incrementally (no 64-bit division per
  // normal): advance by d <= 33 with s >= 1
  int64_t row0 = 0;
  int col0 = 0;
  auto advance = [&](int d) {
    col0 += d;
    while (col0 >= s) {
      col0 -= s;
      ++row0;
    }
  };
  auto at = [&](int off) -> double* {  // element of normal i + off (0 <= off < 32)
    int c = col0 + off;
    int64_t r = row0;
    while (c >= s) {
      c -= s;
      ++r;
    }
    return o + r * sp + c;
  };
  while (i < total) {
    uint64_t r = pcg_out(st);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, wi_s[idx]);
    if (sign) x = -x;
    const bool fast = rabs < ki_s[idx];
    const unsigned slow = __ballot_sync(0xffffffffu, !fast) & (0xffffffffu << start);
    const int f = slow ? __ffs(slow) - 1 : 32;
    // lanes start .. f-1 are one-draw normals
    if (lane >= start && lane < f) {
      const int64_t oi = i + (lane - start);
      if (oi < total) *at(lane - start) = x;
    }
    i += f - start;
    advance(f - start);
    if (f == 32) {  // batch exhausted: advance every lane by 32 draws
      st = add128(mul128(st, A32), C32);
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
      h.ilo = inc.lo;
      h.ihi = inc.hi;
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
        if (a > kTailAttempts) {
          redo[k] = 1;
        } else {
          const int slot = atomicAdd(nrec, 1);
          if (slot < cap) recs[slot] = rec;
          else redo[k] = 1;
        }
        *at(0) = val;
        produced = 1;
      } else {
        const double f0 = fi_s[idx - 1];
        const double f1 = fi_s[idx];
        const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(f0, -f1), h.next_double()), f1);
        consumed = 2;
        if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
          *at(0) = x;
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
    if (nstart < 32) {
      start = nstart;  // lanes still hold the draws behind the consumed ones
      continue;
    }
    // re-base: draw (base + nstart) = A * last + inc, then lane offsets
    last.lo = __shfl_sync(0xffffffffu, last.lo, f);
    last.hi = __shfl_sync(0xffffffffu, last.hi, f);
    b = add128(mul128(last, A), inc);
    st = add128(mul128(b, Al), Cl);
    start = 0;
  }
}

cudaError_t run_omega(uint64_t seed, int64_t K, int J, const int32_t* s_k, int sp, const int64_t* slice_ids,
                      double* out, void* recs, int cap, int32_t* nrec, int32_t* redo, cudaStream_t st) {
  cudaMemsetAsync(nrec, 0, sizeof(int32_t), st);
  cudaMemsetAsync(redo, 0, sizeof(int32_t) * K, st);
  omega_kernel<<<(unsigned)((K + 3) / 4), 128, 0, st>>>(seed, K, J, s_k, sp, slice_ids, out,
                                                        static_cast<TailRec*>(recs), cap, nrec, redo);
  return cudaGetLastError();
}

size_t tail_record_bytes() { return sizeof(TailRec); }
uint64_t derived_seed_host(uint64_t seed, uint64_t index) { return derived_seed_u64(seed, index); }

}  // namespace dp2
