// extern "C" entry points of libdpar2_b200.so (declared in include/dpar2_b200.h).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "dp2_internal.h"

#include <atomic>
#include <thread>

namespace {
thread_local std::string g_last_error;
thread_local std::string g_note;
std::atomic<int64_t> g_launches{0};
int ok(int64_t n) {
  g_launches += n;
  return DP2_OK;
}

int fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e) + (g_note.empty() ? "" : " [" + g_note + "]");
  g_note.clear();
  return DP2_ERR_CUDA;
}
int fail_arg(const char* msg) {
  g_last_error = msg;
  return DP2_ERR_ARG;
}
bool store_ok(const dp2_store* st) {
  if (!st || !st->X || st->J < 1 || st->K < 1 || st->ldx < st->J || st->nseg < 1) return false;
  const int elem = st->dtype == DP2_F64 ? 8 : 4;
  return (st->ldx * elem) % 16 == 0 && (st->dtype == DP2_F64 || st->dtype == DP2_F32);
}
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

namespace dp2 {
void note_error(const char* what) { g_note = what; }
}  // namespace dp2

extern "C" {

int dp2_abi_version(void) { return DP2_ABI_VERSION; }

const char* dp2_status_string(int s) {
  switch (s) {
    case DP2_OK: return "ok";
    case DP2_ERR_NONFINITE: return "non-finite input";
    case DP2_ERR_NOCONV: return "iteration did not converge";
    case DP2_ERR_SHAPE: return "shape / rank error";
    case DP2_ERR_CUDA: return "CUDA error";
    case DP2_ERR_ARG: return "invalid argument";
    default: return "unknown status";
  }
}

const char* dp2_last_error(void) { return g_last_error.c_str(); }

int64_t dp2_launch_count(int32_t reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

int dp2_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

int32_t dp2_stream_segments(int32_t dtype, int64_t J, int32_t sms) {
  if (sms < 1) return 1;
  // the DMMA pass as CTA pairs: one segment per pair
  const bool dmma = dtype == DP2_F64 || dp2::sketch_engine() == 2;
  if (dmma && dp2::sketch64_pairs(J)) return sms / 2 > 0 ? sms / 2 : 1;
  return (dtype == DP2_F64 || J <= 512 || (dmma && J <= 1024)) ? sms : 2 * sms;
}

int32_t dp2_set_sketch_engine(int32_t engine) {
  const int prev = dp2::sketch_engine();
  dp2::set_sketch_engine(engine);
  return prev;
}

int dp2_status_init(int64_t* status_dev, void* stream) {
  int64_t init[DP2_STATUS_WORDS] = {INT64_MAX, 0, INT64_MAX, INT64_MAX, 0, 0, 0, 0};
  cudaError_t e = cudaMemcpyAsync(status_dev, init, sizeof(init), cudaMemcpyHostToDevice, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  return e == cudaSuccess ? DP2_OK : fail(e, "dp2_status_init");
}

// ---------------------------------------------------------------- small uploads
// Copies read pinned (UVA-mapped) host memory directly from a kernel: no copy
// engine, so a few-KB upload on the compute stream never queues behind bulk
// slice uploads already submitted on another stream.
static __global__ void h2d_small_kernel(unsigned char* dst, const unsigned char* src, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((((uintptr_t)dst | (uintptr_t)src | n) & 7) == 0) {
    for (size_t w = i; w < n / 8; w += (size_t)gridDim.x * blockDim.x)
      reinterpret_cast<uint64_t*>(dst)[w] = reinterpret_cast<const volatile uint64_t*>(src)[w];
  } else {
    for (size_t b = i; b < n; b += (size_t)gridDim.x * blockDim.x) dst[b] = reinterpret_cast<const volatile unsigned char*>(src)[b];
  }
}

int dp2_copy_h2d_small(void* dst_dev, const void* src_pinned, size_t nbytes, void* stream) {
  if (nbytes == 0) return DP2_OK;
  if (!dst_dev || !src_pinned) return fail_arg("null pointer");
  const size_t words = (nbytes + 7) / 8;
  const unsigned blocks = (unsigned)std::min<size_t>(64, (words + 255) / 256);
  h2d_small_kernel<<<blocks, 256, 0, S(stream)>>>(static_cast<unsigned char*>(dst_dev),
                                                  static_cast<const unsigned char*>(src_pinned), nbytes);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ok(1) : fail(e, "dp2_copy_h2d_small");
}

// ---------------------------------------------------------------- planning
int dp2_greedy_partition(const int64_t* counts, int64_t K, int32_t workers, int64_t* order_out,
                         int32_t* owner_out, int64_t* loads_out) {
  if (K < 1) return fail_arg("need at least one slice");
  if (workers < 1) return fail_arg("need at least one worker");
  for (int64_t k = 0; k < K; ++k)
    if (counts[k] < 1) return fail_arg("row counts must be positive");
  std::vector<int64_t> order(K);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return counts[a] != counts[b] ? counts[a] > counts[b] : a < b;
  });
  std::vector<int64_t> loads(workers, 0);
  for (int64_t i = 0; i < K; ++i) {
    const int64_t k = order[i];
    int t = 0;
    for (int w = 1; w < workers; ++w)
      if (loads[w] < loads[t]) t = w;  // lowest index on ties
    owner_out[k] = t;
    loads[t] += counts[k];
    order_out[i] = k;
  }
  for (int w = 0; w < workers; ++w) loads_out[w] = loads[w];
  return DP2_OK;
}

int64_t dp2_piece_capacity(int64_t K, int32_t nseg) { return K + nseg; }

int dp2_plan_pieces(const int64_t* row_off, int64_t K, int32_t nseg, int32_t* piece_slice,
                    int64_t* piece_row0, int32_t* piece_rows, int32_t* seg_begin, int32_t* slice_piece,
                    int64_t* npieces_out) {
  if (K < 1 || nseg < 1) return fail_arg("bad plan arguments");
  const int64_t N = row_off[K];
  if (N < 1) return fail_arg("empty tensor");
  int64_t np = 0;
  int64_t k = 0;
  for (int32_t g = 0; g < nseg; ++g) {
    const int64_t a = N * g / nseg, b = N * (g + 1) / nseg;
    seg_begin[g] = (int32_t)np;
    int64_t r = a;
    while (r < b) {
      while (row_off[k + 1] <= r) ++k;
      const int64_t e = std::min<int64_t>(b, row_off[k + 1]);
      if (e - r > INT32_MAX) return fail_arg("piece too large");
      piece_slice[np] = (int32_t)k;
      piece_row0[np] = r;
      piece_rows[np] = (int32_t)(e - r);
      ++np;
      r = e;
    }
  }
  seg_begin[nseg] = (int32_t)np;
  // slice -> first piece (pieces are in global row order, hence slice order)
  int64_t p = 0;
  for (int64_t s = 0; s <= K; ++s) {
    while (p < np && piece_slice[p] < s) ++p;
    slice_piece[s] = (int32_t)p;
  }
  *npieces_out = np;
  return DP2_OK;
}

// ---------------------------------------------------------------- sketch matrices
uint64_t dp2_derived_seed(uint64_t seed, uint64_t index) { return dp2::derived_seed_host(seed, index); }

int dp2_omega_generate(uint64_t seed, int64_t K, int32_t J, const int32_t* s_dev, int32_t sp,
                       const int64_t* slice_ids_dev, double* out, dp2_tail_record* recs, int32_t cap,
                       int32_t* nrec_dev, int32_t* redo_dev, void* stream) {
  static_assert(sizeof(dp2_tail_record) == 88, "record layout");
  if (K < 1 || J < 1 || sp < 1 || cap < 0) return fail_arg("invalid omega shape");
  if (dp2::tail_record_bytes() != sizeof(dp2_tail_record)) return fail_arg("record layout mismatch");
  int launches = 0;
  cudaError_t e = dp2::run_omega(seed, K, J, s_dev, sp, slice_ids_dev, out, recs, cap, nrec_dev, redo_dev, S(stream),
                                 &launches);
  return e == cudaSuccess ? ok(launches) : fail(e, "dp2_omega_generate");
}

int dp2_omega_generate_stream(uint64_t seed, int64_t rows, int32_t width, const int32_t* width_dev, double* out,
                              dp2_tail_record* recs, int32_t cap, int32_t* nrec_dev, int32_t* redo_dev,
                              void* stream) {
  if (rows < 1 || width < 1 || rows * width > INT32_MAX || cap < 0 || !width_dev)
    return fail_arg("invalid omega stream shape");
  int launches = 0;
  cudaError_t e = dp2::run_omega(seed, 1, (int)rows, width_dev, width, nullptr, out, recs, cap, nrec_dev, redo_dev,
                                 S(stream), &launches, true);
  return e == cudaSuccess ? ok(launches) : fail(e, "dp2_omega_generate_stream");
}

int dp2_d2h_staged(void* dst_host, const void* src_dev, size_t nbytes, void* stream) {
  if ((!dst_host || !src_dev) && nbytes) return fail_arg("null buffer");
  cudaError_t e = dp2::d2h_staged(dst_host, src_dev, nbytes, S(stream));
  return e == cudaSuccess ? ok(0) : fail(e, "dp2_d2h_staged");
}

int dp2_omega_replay(const dp2_tail_record* recs, int64_t count, double* vals, int32_t* ok_out) {
  if (count < 0 || (count && (!recs || !vals || !ok_out))) return fail_arg("invalid replay arguments");
  constexpr double kR = 3.6541528853610087963519472518, kInvR = 0.27366123732975827203338247596;
  for (int64_t n = 0; n < count; ++n) {
    const dp2_tail_record& r = recs[n];
    int good = r.attempts >= 1 && r.attempts <= 4;
    double v = 0.0;
    for (int a = 0; good && a < r.attempts; ++a) {
      // P/linalg.py:122 -> numpy random_standard_normal, layer-0 tail branch
      const double xx = -kInvR * std::log1p(-r.u[2 * a]);
      const double yy = -std::log1p(-r.u[2 * a + 1]);
      const bool acc = (yy + yy) > (xx * xx);
      const bool last = a + 1 == r.attempts;
      if (acc != last) good = 0;
      if (last) v = r.negative ? -(kR + xx) : kR + xx;
    }
    vals[n] = v;
    ok_out[n] = good;
  }
  return DP2_OK;
}

// Replay + patch in one call (the exact-Omega path of rng.omega_device):
// records replayed on host threads, the accepted values scattered into
// out_dev[slice][index / w][index % w] (w = widths_host[slice], row stride sp)
// by a kernel reading a library-owned pinned buffer through UVA; slices whose
// acceptance decision differs get redo_host[slice] = 1.
static __global__ void omega_patch_kernel(const int64_t* idx, const double* val, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[((const volatile int64_t*)idx)[i]] = ((const volatile double*)val)[i];
}

namespace {
struct PatchBuf {
  int64_t* idx = nullptr;
  double* val = nullptr;
  int64_t cap = 0;
  cudaEvent_t done = nullptr;
};
PatchBuf g_patch[64];
std::mutex g_patch_mu;
}  // namespace

int dp2_omega_patch(const dp2_tail_record* recs, int64_t count, int64_t J, const int32_t* widths_host, int32_t sp,
                    double* out_dev, int32_t* redo_host, int32_t* patched_out, void* stream) {
  if (count < 0 || (count && (!recs || !widths_host || !out_dev || !redo_host))) return fail_arg("invalid patch arguments");
  if (patched_out) *patched_out = 0;
  if (count == 0) return DP2_OK;
  std::vector<double> vals((size_t)count);
  std::vector<int32_t> okv((size_t)count);
  const int hw = (int)std::thread::hardware_concurrency();
  // (thread start-up costs ~20 us each: only very large record counts use a team)
  const int nt = count < 32768 ? 1 : std::max(1, std::min(16, hw));
  std::vector<std::thread> team;
  std::vector<int> rc(nt, DP2_OK);
  const int64_t chunk = (count + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t a = t * chunk, b = std::min(count, a + chunk);
    if (a >= b) break;
    auto fn = [&, a, b, t] { rc[t] = dp2_omega_replay(recs + a, b - a, vals.data() + a, okv.data() + a); };
    if (nt == 1) fn(); else team.emplace_back(fn);
  }
  for (auto& th : team) th.join();
  for (int r : rc)
    if (r != DP2_OK) return r;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(cudaErrorInvalidDevice, "dp2_omega_patch");
  std::lock_guard<std::mutex> g(g_patch_mu);
  PatchBuf& pb = g_patch[dev];
  if (pb.done) cudaEventSynchronize(pb.done);  // the previous patch kernel is done reading the buffer
  if (pb.cap < count) {
    if (pb.idx) cudaFreeHost(pb.idx);
    if (pb.val) cudaFreeHost(pb.val);
    pb.idx = nullptr;
    pb.val = nullptr;
    pb.cap = 0;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&pb.idx), count * 8, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&pb.val), count * 8, cudaHostAllocDefault);
    if (e != cudaSuccess) return fail(e, "dp2_omega_patch");
    pb.cap = count;
    if (!pb.done && (e = cudaEventCreateWithFlags(&pb.done, cudaEventDisableTiming)) != cudaSuccess)
      return fail(e, "dp2_omega_patch");
  }
  int64_t n = 0;
  for (int64_t i = 0; i < count; ++i) {
    const dp2_tail_record& r = recs[i];
    if (!okv[i]) {
      redo_host[r.slice] = 1;
      continue;
    }
    const int64_t w = widths_host[r.slice];
    pb.idx[n] = r.slice * (J * sp) + (r.index / w) * sp + r.index % w;
    pb.val[n] = vals[i];
    ++n;
  }
  if (n) {
    omega_patch_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 64), 256, 0, S(stream)>>>(pb.idx, pb.val, n,
                                                                                                 out_dev);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventRecord(pb.done, S(stream));
    if (e != cudaSuccess) return fail(e, "dp2_omega_patch");
  }
  if (patched_out) *patched_out = (int32_t)n;
  return n ? ok(1) : DP2_OK;
}

// ---------------------------------------------------------------- host checks
// all-ones exponent <=> NaN/Inf; integer tests, so the inner loops vectorise
static bool rows_finite_f(const float* p, int64_t rows, int64_t ld, int64_t J) {
  for (int64_t r = 0; r < rows; ++r) {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(p + r * ld);
    uint32_t bad = 0;
    for (int64_t j = 0; j < J; ++j) bad |= ((row[j] & 0x7f800000u) == 0x7f800000u);
    if (bad) return false;
  }
  return true;
}
static bool rows_finite_d(const double* p, int64_t rows, int64_t ld, int64_t J) {
  for (int64_t r = 0; r < rows; ++r) {
    const uint64_t* row = reinterpret_cast<const uint64_t*>(p + r * ld);
    uint64_t bad = 0;
    for (int64_t j = 0; j < J; ++j) bad |= ((row[j] & 0x7ff0000000000000ull) == 0x7ff0000000000000ull);
    if (bad) return false;
  }
  return true;
}

int dp2_host_first_nonfinite(const void* const* ptrs, const int64_t* rows, const int64_t* ld, int64_t K, int64_t J,
                             int32_t dtype, int32_t threads, int64_t* first_bad) {
  if (K < 0 || J < 1 || !first_bad || (K && (!ptrs || !rows || !ld))) return fail_arg("invalid check arguments");
  if (dtype != DP2_F32 && dtype != DP2_F64) return fail_arg("dtype must be DP2_F32 or DP2_F64");
  std::atomic<int64_t> next{0}, bad{INT64_MAX};
  auto work = [&]() {
    for (int64_t k; (k = next.fetch_add(1)) < K;) {
      if (k > bad.load(std::memory_order_relaxed)) continue;
      const bool okk = dtype == DP2_F32 ? rows_finite_f(static_cast<const float*>(ptrs[k]), rows[k], ld[k], J)
                                        : rows_finite_d(static_cast<const double*>(ptrs[k]), rows[k], ld[k], J);
      if (!okk) {
        int64_t cur = bad.load();
        while (k < cur && !bad.compare_exchange_weak(cur, k)) {
        }
      }
    }
  };
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min<int>(nt, 64));
  if (K < 2 * nt) nt = std::max<int64_t>(1, K / 2);
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  *first_bad = bad.load();
  return DP2_OK;
}

int dp2_sketch_uses_tc(const dp2_store* st, int32_t sp) {
  if (!store_ok(st)) return 0;
  return dp2::sketch_tc_eligible(st, sp) ? 1 : 0;
}

// ---------------------------------------------------------------- device calls
int dp2_slice_stats(const dp2_store* st, double* sqnorm_dev, int64_t* status_dev, void* stream) {
  if (!store_ok(st)) return fail_arg("invalid store");
  cudaError_t e = dp2::run_slice_stats(st, sqnorm_dev, status_dev, S(stream));
  return e == cudaSuccess ? ok(3) : fail(e, "dp2_slice_stats");
}

int dp2_stream_pass(const dp2_store* st, const double* b_dev, int32_t sp, double* out_part, double* y_out,
                    double* g_part, double* xsq_part, int64_t* status_dev, void* stream) {
  if (!store_ok(st) || sp < 1 || !b_dev || !out_part) return fail_arg("invalid stream-pass arguments");
  if (g_part && sp > 32) return fail_arg("g_part needs sp <= 32");
  const int kind = dp2_sketch_kind(st, sp, xsq_part != nullptr, g_part != nullptr);
  cudaError_t e = dp2::run_sketch(st, b_dev, sp, out_part, y_out, xsq_part, status_dev, S(stream), g_part);
  return e == cudaSuccess ? ok(kind >= 2 ? 2 : 1) : fail(e, "dp2_stream_pass");
}

int32_t dp2_sketch_kind(const dp2_store* st, int32_t sp, int32_t xsq, int32_t gram) {
  if (!store_ok(st) || sp < 1) return -1;
  if (dp2::sketch_tc_eligible(st, sp)) return 2;
  const bool s64 = dp2::sketch64_eligible(st, sp, xsq != 0, gram != 0);
  if (st->dtype == DP2_F64) return s64 ? 3 : 0;
  return (dp2::sketch_engine() == 2 && s64) ? 3 : 1;
}

size_t dp2_stage1_workspace(const dp2_store* st, int32_t sp, int32_t rank) {
  return dp2::stage1_layout(st, sp, rank).total;
}

static int stage1_impl(const dp2_store* st, const double* omega_dev, const int32_t* s_dev, int32_t sp,
                       int32_t rank, double* A_out, double* M_out, int32_t* rank_out, void* ws, size_t ws_bytes,
                       int64_t* status_dev, float* timing_ms, void* stream, double* a_signs, int power_iters = 1) {
  if (!store_ok(st)) return fail_arg("invalid store");
  if (rank < 1 || rank > 64 || sp < rank || sp % 8 != 0 || (sp > 32 && sp % 32 != 0) || sp > 256)
    return fail_arg("invalid rank / sketch width");
  if (power_iters < 0 || power_iters > 64) return fail_arg("power_iters out of range");
  if (ws_bytes < dp2::stage1_layout(st, sp, rank).total) return fail_arg("workspace too small");
  cudaError_t e = dp2::run_stage1(st, omega_dev, s_dev, sp, rank, A_out, M_out, rank_out,
                                  static_cast<char*>(ws), status_dev, timing_ms, S(stream), a_signs, power_iters);
  // sp <= 32: 2 streaming passes + orth (Gram, Cholesky, substitution, CGS2
  // fallback) + gather, factor, A + candidates, signs, [apply signs],
  // complete; the tensor-core pass adds its two B-image kernels and
  // gram_y_piece_kernel.  sp > 32: 8 kernels [+ the sign fill].
  const int tc = dp2::sketch_tc_eligible(st, sp) ? 3 : 0;
  // the warp-specialised DMMA pass adds its B-image kernel per pass
  const int img = (dp2_sketch_kind(st, sp, 0, 0) == 3 ? 1 : 0) + (dp2_sketch_kind(st, sp, 0, sp <= 32) == 3 ? 1 : 0);
  const int n = (sp <= 32 ? (a_signs ? 11 : 12) + tc : (a_signs ? 9 : 8)) + img;
  return e == cudaSuccess ? ok(n) : fail(e, "dp2_stage1");
}

int dp2_stage1(const dp2_store* st, const double* omega_dev, const int32_t* s_dev, int32_t sp, int32_t rank,
               double* A_out, double* M_out, int32_t* rank_out, void* ws, size_t ws_bytes,
               int64_t* status_dev, float* timing_ms, void* stream) {
  return stage1_impl(st, omega_dev, s_dev, sp, rank, A_out, M_out, rank_out, ws, ws_bytes, status_dev, timing_ms,
                     stream, nullptr);
}

int dp2_stage1_signs(const dp2_store* st, const double* omega_dev, const int32_t* s_dev, int32_t sp, int32_t rank,
                     double* A_out, double* M_out, int32_t* rank_out, double* a_signs_out, void* ws,
                     size_t ws_bytes, int64_t* status_dev, float* timing_ms, void* stream) {
  if (!a_signs_out) return fail_arg("a_signs_out is null");
  return stage1_impl(st, omega_dev, s_dev, sp, rank, A_out, M_out, rank_out, ws, ws_bytes, status_dev, timing_ms,
                     stream, a_signs_out);
}

int dp2_stage1_power(const dp2_store* st, const double* omega_dev, const int32_t* s_dev, int32_t sp, int32_t rank,
                     int32_t power_iters, double* A_out, double* M_out, int32_t* rank_out, double* a_signs_out,
                     void* ws, size_t ws_bytes, int64_t* status_dev, float* timing_ms, void* stream) {
  return stage1_impl(st, omega_dev, s_dev, sp, rank, A_out, M_out, rank_out, ws, ws_bytes, status_dev, timing_ms,
                     stream, a_signs_out, power_iters);
}

size_t dp2_stage2_workspace(int64_t J, int64_t KR, int32_t s2, int32_t rank) {
  return dp2::stage2_bytes(J, KR, s2, rank);
}

int dp2_stage2_power(const double* M_dev, int64_t J, int64_t KR, const double* omega2_dev, int32_t s2,
                     int32_t rank, int32_t power_iters, double* D_out, double* E_out, double* F_out, void* ws,
                     size_t ws_bytes, int64_t* status_dev, void* stream) {
  if (rank < 1 || rank > 64 || s2 < rank || s2 > 150 || J < 1 || KR < 1) return fail_arg("invalid stage-2 shape");
  if (power_iters < 0 || power_iters > 64) return fail_arg("power_iters out of range");
  if (ws_bytes < dp2::stage2_bytes(J, KR, s2, rank)) return fail_arg("workspace too small");
  cudaError_t e = dp2::run_stage2(M_dev, J, KR, omega2_dev, s2, rank, D_out, E_out, F_out,
                                  static_cast<char*>(ws), status_dev, S(stream), power_iters);
  // our own DMMA GEMM kernels + ordered reductions + orth + final
  // launches: nn (2) per M-product, tn (1, +1 reduction when split), orth, gram (2), final, F
  const int tn = dp2::gemm_tn_splits(J, KR, s2) > 1 ? 2 : 1;
  return e == cudaSuccess ? ok(2 + power_iters * (tn + 2) + 1 + tn + 2 + 2) : fail(e, "dp2_stage2");
}

int dp2_stage2(const double* M_dev, int64_t J, int64_t KR, const double* omega2_dev, int32_t s2, int32_t rank,
               double* D_out, double* E_out, double* F_out, void* ws, size_t ws_bytes, int64_t* status_dev,
               void* stream) {
  return dp2_stage2_power(M_dev, J, KR, omega2_dev, s2, rank, 1, D_out, E_out, F_out, ws, ws_bytes, status_dev,
                          stream);
}

size_t dp2_als_workspace(int64_t K, int64_t J, int32_t R) { return dp2::als_bytes(K, J, R); }
size_t dp2_als_stamp_offset(int64_t K, int64_t J, int32_t R) { return dp2::als_stamp_offset(K, J, R); }

int dp2_als_run(const double* F, const double* D, const double* E, int64_t K, int64_t J, int32_t R, double* H,
                double* V, double* W, double* polar_out, int32_t max_iters, double tol, int32_t normalize,
                double* trace_out, int64_t* tstamp_out, int32_t* iters_out, int32_t use_graph, void* ws,
                size_t ws_bytes, int64_t* status_dev, void* stream) {
  if (max_iters < 1) return fail_arg("max_iters must be >= 1");
  if (R < 1 || R > 64 || K < 1 || J < 1) return fail_arg("invalid ALS shape");
  if (ws_bytes < dp2::als_bytes(K, J, R)) return fail_arg("workspace too small");
  int64_t launches = 0;
  cudaError_t e = dp2::als_run(F, D, E, K, J, R, H, V, W, polar_out, max_iters, tol, normalize, trace_out,
                               tstamp_out, iters_out, use_graph, static_cast<char*>(ws), status_dev, S(stream),
                               &launches);
  return e == cudaSuccess ? ok(launches) : fail(e, "dp2_als_run");
}

int dp2_als_phase(int32_t phase, const double* F, const double* D, const double* E, int64_t K, int64_t J,
                  int32_t R, double* H, double* V, double* W, double* polar, int32_t it, double tol,
                  int32_t normalize, double* trace_out, int64_t* tstamp_out, int32_t* iters_out,
                  const double* red_in, double* red_out, void* ws, size_t ws_bytes, int64_t* status_dev,
                  void* stream) {
  if (phase < 0 || phase > 6 || R < 1 || R > 64 || K < 1 || J < 1) return fail_arg("invalid ALS phase");
  if (ws_bytes < dp2::als_bytes(K, J, R)) return fail_arg("workspace too small");
  if ((phase == 2 || phase == 4 || phase == 6) && red_in == nullptr) return fail_arg("phase needs red_in");
  if ((phase == 1 || phase == 3 || phase == 5) && red_out == nullptr) return fail_arg("phase needs red_out");
  cudaError_t e = dp2::als_phase(phase, F, D, E, K, J, R, H, V, W, polar, it, tol, normalize, trace_out,
                                 tstamp_out, iters_out, red_in, red_out, static_cast<char*>(ws), status_dev,
                                 S(stream));
  static const int kLaunches[7] = {1, 3, 1, 3, 1, 3, 1};
  return e == cudaSuccess ? ok(kLaunches[phase]) : fail(e, "dp2_als_phase");
}

int dp2_update_rotations(const double* F, const double* D, const double* E, int64_t K, int64_t J, int32_t R,
                         const double* H, const double* V, const double* W, double* polar_out, double* theta_out,
                         void* ws, size_t ws_bytes, int64_t* status_dev, void* stream) {
  if (R < 1 || R > 64 || ws_bytes < dp2::als_bytes(K, J, R)) return fail_arg("invalid arguments");
  cudaError_t e = dp2::als_rotations(F, D, E, K, J, R, H, V, W, polar_out, theta_out, static_cast<char*>(ws),
                                     status_dev, S(stream));
  return e == cudaSuccess ? ok(2) : fail(e, "dp2_update_rotations");
}

int dp2_mttkrp(int32_t mode, const double* theta, const double* D, const double* E, int64_t K, int64_t J,
               int32_t R, const double* H, const double* V, const double* W, double* out, void* ws,
               size_t ws_bytes, void* stream) {
  if (mode < 1 || mode > 3 || R < 1 || R > 64 || ws_bytes < dp2::als_bytes(K, J, R))
    return fail_arg("invalid arguments");
  cudaError_t e = dp2::als_mttkrp(mode, theta, D, E, K, J, R, H, V, W, out, static_cast<char*>(ws), S(stream));
  return e == cudaSuccess ? ok(mode == 2 ? 4 : (mode == 1 ? 3 : 2)) : fail(e, "dp2_mttkrp");
}

int dp2_update_factors(const double* theta, const double* D, const double* E, int64_t K, int64_t J, int32_t R,
                       double* H, double* V, double* W, int32_t normalize, void* ws, size_t ws_bytes,
                       int64_t* status_dev, void* stream) {
  if (R < 1 || R > 64 || ws_bytes < dp2::als_bytes(K, J, R)) return fail_arg("invalid arguments");
  cudaError_t e = dp2::als_update_factors(theta, D, E, K, J, R, H, V, W, normalize, static_cast<char*>(ws),
                                          status_dev, S(stream));
  return e == cudaSuccess ? ok(6) : fail(e, "dp2_update_factors");
}

int dp2_convergence_metric(const double* theta, const double* D, const double* E, int64_t K, int64_t J,
                           int32_t R, const double* H, const double* V, const double* W, double* out, void* ws,
                           size_t ws_bytes, void* stream) {
  if (R < 1 || R > 64 || ws_bytes < dp2::als_bytes(K, J, R)) return fail_arg("invalid arguments");
  cudaError_t e = dp2::als_metric(theta, D, E, K, J, R, H, V, W, out, static_cast<char*>(ws), S(stream));
  return e == cudaSuccess ? ok(4) : fail(e, "dp2_convergence_metric");
}

int dp2_assemble_q(const dp2_store* st, const double* A, int32_t R, const double* polar, double* Q_out,
                   void* stream) {
  if (!store_ok(st) || R < 1 || R > 64) return fail_arg("invalid arguments");
  cudaError_t e = dp2::run_assemble_q(st, A, R, polar, Q_out, S(stream), nullptr);
  return e == cudaSuccess ? ok(1) : fail(e, "dp2_assemble_q");
}

int dp2_assemble_q_signed(const dp2_store* st, const double* A, int32_t R, const double* a_signs,
                          const double* polar, double* Q_out, void* stream) {
  if (!store_ok(st) || R < 1 || R > 64 || !a_signs) return fail_arg("invalid arguments");
  cudaError_t e = dp2::run_assemble_q(st, A, R, polar, Q_out, S(stream), a_signs);
  return e == cudaSuccess ? ok(1) : fail(e, "dp2_assemble_q_signed");
}

size_t dp2_fitness_workspace(const dp2_store* st) { return dp2::fitness_bytes(st); }

int dp2_fitness(const dp2_store* st, const double* Q, int32_t R, const double* H, const double* V,
                const double* W, double* out2_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!store_ok(st) || R < 1 || R > 64 || ws_bytes < dp2::fitness_bytes(st)) return fail_arg("invalid arguments");
  cudaError_t e = dp2::run_fitness(st, Q, R, H, V, W, out2_dev, static_cast<char*>(ws), S(stream));
  return e == cudaSuccess ? ok(2) : fail(e, "dp2_fitness");
}

int dp2_gemm_tn(const double* A, int64_t m, int64_t K, const double* B, int32_t n, double* out, void* stream) {
  if (!A || !B || !out || m < 1 || K < 1 || n < 1) return fail_arg("invalid arguments");
  cudaError_t e = dp2::run_gemm_tn(A, m, K, B, n, out, S(stream), nullptr);
  return e == cudaSuccess ? ok(1) : fail(e, "dp2_gemm_tn");
}

size_t dp2_zero_pass_workspace(int64_t K, int32_t R) { return dp2::zero_pass_bytes(K, R); }

int dp2_fitness_zero_pass(const double* MtV, int64_t K, int64_t J, int32_t R, const double* H, const double* V,
                          const double* W, const double* polar, const double* sqnorm, double* out2_dev, void* ws,
                          size_t ws_bytes, void* stream) {
  if (!MtV || !H || !V || !W || !polar || !sqnorm || !out2_dev || K < 1 || J < 1 || R < 1 || R > 64 ||
      ws_bytes < dp2::zero_pass_bytes(K, R))
    return fail_arg("invalid arguments");
  cudaError_t e = dp2::run_zero_pass_fitness(MtV, K, J, R, H, V, W, polar, sqnorm, out2_dev, static_cast<char*>(ws),
                                             S(stream));
  return e == cudaSuccess ? ok(3) : fail(e, "dp2_fitness_zero_pass");
}

}  // extern "C"
