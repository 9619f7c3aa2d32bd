// mbarrier hand-off latency between warps of one CTA (try_wait spin loops).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
}
template <bool ALL_LANES>
__global__ void pingpong(int n, long long* out) {
  __shared__ __align__(8) uint64_t x, y;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&x)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&y)));
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (w == 0) {
      if (lane == 0) arrive(&x);
      if (ALL_LANES || lane == 0) wait(&y, i & 1);
      __syncwarp();
    } else if (w == 1) {
      if (ALL_LANES || lane == 0) wait(&x, i & 1);
      __syncwarp();
      if (lane == 0) arrive(&y);
    }
  }
  if (threadIdx.x == 0) out[0] = clock64() - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  for (int v = 0; v < 2; ++v) {
    const int n = 10000;
    if (v) pingpong<true><<<1, 64>>>(n, d); else pingpong<false><<<1, 64>>>(n, d);
    cudaDeviceSynchronize();
    if (v) pingpong<true><<<1, 64>>>(n, d); else pingpong<false><<<1, 64>>>(n, d);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.0f cycles per round trip (2 hand-offs)\n", v ? "all 32 lanes wait" : "lane 0 waits", (double)h / n);
  }
  return 0;
}
