// Throughput probe: cycles per tcgen05.mma kind::tf32 for the skinny shapes
// of the stage-1 sketch (back-to-back, one issuing thread, same operands).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_rate tools/umma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int MODE>  // 0: SS, 1: TS (A from TMEM)
__global__ void rate(int M, int N, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar;
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t hi = (1024u >> 4) | (1u << 14) | (2u << 29);
    const uint32_t alo = (su32(base) >> 4) | (1u << 16), blo = (su32(base + 32768) >> 4) | (1u << 16);
    const uint32_t id = idesc_tf32(M, N, 0, 0);
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t k = (uint32_t)(i & 3) * 2;
      if (MODE == 0) {
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b64 da, db;\n\tmov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
            "elect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %4, 1;\n\t}" ::"r"(
                tmem + 256),
            "r"(alo + k), "r"(blo + k), "r"(hi), "r"(id)
            : "memory");
      } else {
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b64 db;\n\tmov.b64 db, {%2, %3};\n\t"
            "elect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], db, %4, 1;\n\t}" ::"r"(
                tmem + 256),
            "r"(tmem + (uint32_t)(i & 7) * 8), "r"(blo + k), "r"(hi), "r"(id)
            : "memory");
      }
    }
    const long long t1 = clock64();
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&mbar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&mbar)));
    const long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  struct C { int mode, M, N; } cs[] = {{0, 64, 24},  {0, 128, 24}, {0, 128, 32}, {1, 128, 32},
                                       {1, 128, 24}, {0, 64, 256}, {0, 128, 256}, {1, 128, 256}, {0, 64, 8}};
  const int iters = 4096;
  for (auto c : cs) {
    for (int rep = 0; rep < 2; ++rep) {
      if (c.mode == 0) rate<0><<<1, 128, 70000>>>(c.M, c.N, iters, d);
      else rate<1><<<1, 128, 70000>>>(c.M, c.N, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
    }
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s M=%3d N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma, floor %.1f\n", c.mode ? "TS" : "SS", c.M, c.N,
           (double)h[0] / iters, (double)h[1] / iters, (c.M > 128 ? c.M : 128) * c.N / 256.0);
  }
  return 0;
}
