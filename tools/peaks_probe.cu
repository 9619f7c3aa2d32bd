// Whole-GPU compute peaks for the roofline denominators SURVEY §8(d) asks for
// (MEASURED_PEAKS.json only has HBM and bf16): FP64 tensor (DMMA.8x8x4, the
// only fp64 MMA sm_100a has -- m16n8k16.f64 lowers to it), DFMA, FFMA and
// tcgen05.mma kind::tf32 (M=128 N=256 K=8, smem operands, one issuing thread
// per SM).  Every kernel runs on all SMs; time = CUDA events, best of 5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/peaks_probe tools/peaks_probe.cu
//   tools/bin/peaks_probe > profiles/r2_compute_peaks.json
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int CH = 8;  // independent accumulator chains per thread

__global__ void dmma_k(double* out, int n) {
  double c[CH][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = 0.0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename T>
__global__ void fma_k(T* out, int n) {
  T c[CH];
  const T a = T(1) + T(threadIdx.x) * T(1e-7), b = T(1e-7);
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j] = T(j);
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) c[j] = fma(c[j], a, b);
  }
  T s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j];
  if (s == T(12345.678)) out[threadIdx.x] = s;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void tf32_k(int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar;
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t hi = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO 1024, sm100 version, SWIZZLE_128B
    const uint32_t alo = (su32(base) >> 4) | (1u << 16), blo = (su32(base + 16384) >> 4) | (1u << 16);
    const uint32_t id = idesc_tf32(128, 256);
    __syncwarp();
    for (int i = 0; i < iters; ++i) {
      const uint32_t k = (uint32_t)(i & 3) * 2;
      asm volatile(
          "{\n\t.reg .pred e;\n\t.reg .b64 da, db;\n\tmov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
          "elect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %4, 1;\n\t}" ::"r"(tmem),
          "r"(alo + k), "r"(blo + k), "r"(hi), "r"(id)
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&mbar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&mbar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <typename F>
static float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;  // rep 0 = warm-up
  }
  return best;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* d;
  CK(cudaMalloc(&d, 1 << 20));
  const int n = 4096;
  // DMMA: 16 warps per SM (4 per SM sub-partition), CH chains each
  for (int wps : {8, 16, 32}) {
    const int blocks = sms * 2, threads = wps * 16;
    float ms = best_ms([&] { dmma_k<<<blocks, threads>>>((double*)d, n); });
    CK(cudaGetLastError());
    const double flops = 512.0 * CH * n * (double)blocks * threads / 32;
    printf("{\"probe\": \"dmma_m8n8k4_f64\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", wps, flops / ms / 1e9);
  }
  for (int tps : {512, 1024, 2048}) {
    const int blocks = sms * 2, threads = tps / 2;
    float ms = best_ms([&] { fma_k<double><<<blocks, threads>>>((double*)d, n); });
    CK(cudaGetLastError());
    const double flops = 2.0 * CH * n * (double)blocks * threads;
    printf("{\"probe\": \"dfma_f64\", \"threads_per_sm\": %d, \"tflops\": %.2f}\n", tps, flops / ms / 1e9);
  }
  for (int tps : {512, 1024, 2048}) {
    const int blocks = sms * 2, threads = tps / 2;
    float ms = best_ms([&] { fma_k<float><<<blocks, threads>>>((float*)d, n * 4); });
    CK(cudaGetLastError());
    const double flops = 2.0 * CH * n * 4 * (double)blocks * threads;
    printf("{\"probe\": \"ffma_f32\", \"threads_per_sm\": %d, \"tflops\": %.2f}\n", tps, flops / ms / 1e9);
  }
  {
    const int smem = 48 * 1024 + 1024, iters = 20000;
    CK(cudaFuncSetAttribute(tf32_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float ms = best_ms([&] { tf32_k<<<sms, 128, smem>>>(iters); });
    CK(cudaGetLastError());
    const double flops = 2.0 * 128 * 256 * 8 * (double)iters * sms;
    printf("{\"probe\": \"tcgen05_tf32_m128n256k8_ss\", \"ctas\": %d, \"tflops\": %.2f}\n", sms, flops / ms / 1e9);
  }
  printf("{\"sms\": %d, \"clock_khz_attr\": %d}\n", sms, clk);
  return 0;
}
