// Sketch matrices Omega_k on the device, bit-exact with the reference's
// Generator(PCG64(derived_seed(seed, k))).standard_normal((J, s_k))
// (P/linalg.py:122-123, 187-194).
//
//   SeedSequence([seed, k]) -> 1 uint64 (derived seed)   numpy SeedSequence hash
//   SeedSequence(derived)   -> 4 uint64 -> PCG64 state/inc (pcg setseq srandom)
//   PCG64 XSL-RR 128/64 stream -> 256-layer ziggurat (tables: dp2_ziggurat_tables.h)
//
// One thread per slice walks that slice's stream.  The fast path (>99% of
// draws: one 64-bit output, one multiply) is exact IEEE arithmetic.  The rare
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

__global__ void __launch_bounds__(32) omega_kernel(uint64_t seed, int64_t K, int J, const int32_t* s_k, int sp,
                                                   const int64_t* slice_ids, double* out, TailRec* recs,
                                                   int cap, int32_t* nrec, int32_t* redo) {
  // lanes index the tables with different layers: shared memory, not the
  // (uniform-access) constant cache
  __shared__ uint64_t ki_s[256];
  __shared__ double wi_s[256], fi_s[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    ki_s[i] = kZigKi[i];
    wi_s[i] = __longlong_as_double((long long)kZigWiBits[i]);
    fi_s[i] = __longlong_as_double((long long)kZigFiBits[i]);
  }
  __syncthreads();
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const uint64_t gid = slice_ids ? (uint64_t)slice_ids[k] : (uint64_t)k;
  Pcg g;
  g.seed(derived_seed_u64(seed, gid));
  const int s = s_k[k];
  double* o = out + (size_t)k * J * sp;
  const int64_t total = (int64_t)J * s;
  int64_t i = 0;
  for (int j = 0; j < J; ++j) {
    for (int c = 0; c < s; ++c, ++i) {
      double val;
      for (;;) {
        uint64_t r = g.next();
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const int sign = (int)(r & 1);
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
        double x = __dmul_rn((double)rabs, wi_s[idx]);
        if (sign) x = -x;
        if (rabs < ki_s[idx]) { val = x; break; }
        if (idx == 0) {
          TailRec rec;
          rec.slice = k;
          rec.index = i;
          rec.negative = (int)((rabs >> 8) & 1);
          int a = 0;
          for (;;) {
            const double u1 = g.next_double(), u2 = g.next_double();
            if (a < kTailAttempts) { rec.u[2 * a] = u1; rec.u[2 * a + 1] = u2; }
            ++a;
            const double xx = __dmul_rn(-kZigInvR, log1p(-u1));
            const double yy = -log1p(-u2);
            if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
              val = rec.negative ? -(kZigR + xx) : kZigR + xx;
              break;
            }
          }
          rec.attempts = a;
          if (a > kTailAttempts) {
            redo[k] = 1;
          } else {
            const int slot = atomicAdd(nrec, 1);
            if (slot < cap) recs[slot] = rec;
            else redo[k] = 1;
          }
          break;
        }
        const double f0 = fi_s[idx - 1];
        const double f1 = fi_s[idx];
        const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(f0, -f1), g.next_double()), f1);
        if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) { val = x; break; }
      }
      o[(size_t)j * sp + c] = val;
    }
    for (int c = s; c < sp; ++c) o[(size_t)j * sp + c] = 0.0;
  }
  (void)total;
}

cudaError_t run_omega(uint64_t seed, int64_t K, int J, const int32_t* s_k, int sp, const int64_t* slice_ids,
                      double* out, void* recs, int cap, int32_t* nrec, int32_t* redo, cudaStream_t st) {
  cudaMemsetAsync(nrec, 0, sizeof(int32_t), st);
  cudaMemsetAsync(redo, 0, sizeof(int32_t) * K, st);
  omega_kernel<<<(unsigned)((K + 31) / 32), 32, 0, st>>>(seed, K, J, s_k, sp, slice_ids, out,
                                                          static_cast<TailRec*>(recs), cap, nrec, redo);
  return cudaGetLastError();
}

size_t tail_record_bytes() { return sizeof(TailRec); }
uint64_t derived_seed_host(uint64_t seed, uint64_t index) { return derived_seed_u64(seed, index); }

}  // namespace dp2
