// Layout probe for tcgen05.mma kind::tf32 operand descriptors (one CTA, one
// M=128 x N=32 x K=8 MMA per case): which shared-memory layouts does the
// hardware accept for MN-major / K-major A?  Prints the max abs error of D
// against a host reference for each case.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe tools/umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// A element (m, k) byte offset for each case; B is K-major SW128 (known good)
__device__ uint32_t a_off(int cs, int m, int k) {
  switch (cs) {
    case 0:  // MN-major SWIZZLE_128B (16 B granule ^ k%8), 128 B rows of m, MN blocks of 32 at 1024
      return (m / 32) * 1024 + k * 128 + ((((m % 32) / 4) ^ (k % 8)) << 4) + (m % 4) * 4;
    case 1:  // MN-major SWIZZLE_128B_BASE32B (32 B granule ^ k%4), 4-row atoms (512 B), MN blocks at 1024
      return (m / 32) * 1024 + (k / 4) * 512 + (k % 4) * 128 + ((((m % 32) / 8) ^ (k % 4)) << 5) + (m % 8) * 4;
    case 2:  // MN-major INTERLEAVE: core = 8 k-rows x 16 B (4 m), m-cores contiguous
      return (m / 4) * 128 + (k % 8) * 16 + (m % 4) * 4;
    case 3:  // K-major INTERLEAVE: core = 8 m-rows x 16 B (4 k); m-cores at 256, k-cores at 128
      return (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4;
    case 4:  // MN-major INTERLEAVE, same bytes as 2, LBO/SBO swapped in the descriptor
      return (m / 4) * 128 + (k % 8) * 16 + (m % 4) * 4;
    case 5:  // MN-major BASE32B, same bytes as 1, LBO/SBO swapped in the descriptor
      return (m / 32) * 1024 + (k / 4) * 512 + (k % 4) * 128 + ((((m % 32) / 8) ^ (k % 4)) << 5) + (m % 8) * 4;
    case 6:  // K-major SWIZZLE_128B_BASE32B: 128 B rows of k, 32 B granule ^ m%4 (SBO 512)
    case 7:  // same bytes, SBO 1024
      return m * 128 + ((((k % 32) / 8) ^ (m % 4)) << 5) + (k % 8) * 4;
    case 8:  // K-major BASE32B, the K=8 slice at k = 8..15 of the row (descriptor start + 32 B)
      return m * 128 + ((((k + 8) / 8) ^ (m % 4)) << 5) + (k % 8) * 4;
    default:
      return 0;
  }
}

__global__ void probe(int cs, const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar;
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  unsigned char* As = base;          // 16 KB
  unsigned char* Bs = base + 16384;  // 4 KB
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 5 * 1024; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.f;
  __syncthreads();
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int m = e / 8, k = e % 8;
    *reinterpret_cast<float*>(As + a_off(cs, m, k)) = A[m * 8 + k];
  }
  for (int e = tid; e < 32 * 8; e += blockDim.x) {
    const int n = e / 8, k = e % 8;
    *reinterpret_cast<float*>(Bs + n * 128 + ((((k / 4) ^ (n % 8)) & 7) << 4) + (k % 4) * 4) = B[k * 32 + n];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    uint64_t ad;
    int amn = 1;
    switch (cs) {
      case 0: ad = sdesc(su32(As), 1024, 1024, 2); break;
      case 1: ad = sdesc(su32(As), 1024, 512, 1); break;
      case 2: ad = sdesc(su32(As), 4096, 128, 0); break;  // LBO: k-core stride (unused, K=8), SBO: m-core stride
      case 3: ad = sdesc(su32(As), 128, 256, 0); amn = 0; break;  // LBO: k-core stride, SBO: m-core stride
      case 4: ad = sdesc(su32(As), 128, 4096, 0); break;  // swapped
      case 5: ad = sdesc(su32(As), 512, 1024, 1); break;  // swapped
      case 6: ad = sdesc(su32(As), 16, 512, 1); amn = 0; break;
      case 7: ad = sdesc(su32(As), 16, 1024, 1); amn = 0; break;
      default: ad = sdesc(su32(As) + 32, 16, 512, 1); amn = 0; break;
    }
    const uint64_t bd = sdesc(su32(Bs), 16, 1024, 2);
    const uint32_t id = idesc_tf32(128, 32, amn, 0);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(id), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&mbar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int c = 0; c < 32; ++c) D[(warp * 32 + (tid & 31)) * 32 + c] = __uint_as_float(v[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  std::vector<float> A(128 * 8), B(8 * 32), D(128 * 32);
  for (int i = 0; i < 128 * 8; ++i) A[i] = (float)((i * 37) % 17 - 8) / 4.0f;  // exact in tf32
  for (int i = 0; i < 8 * 32; ++i) B[i] = (float)((i * 11) % 13 - 6) / 2.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const char* names[] = {"MN-major SW128", "MN-major SW128_BASE32B", "MN-major INTERLEAVE (LBO=k,SBO=m)",
                         "K-major INTERLEAVE", "MN-major INTERLEAVE (LBO=m,SBO=k)",
                         "MN-major BASE32B (LBO=512,SBO=1024)", "K-major BASE32B (SBO=512)",
                         "K-major BASE32B (SBO=1024)", "K-major BASE32B k=8..15 (+32 B)"};
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int cs = 0; cs < 9; ++cs) {
    if (only >= 0 && cs != only) continue;
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, 32768>>>(cs, dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("case %d %s: CUDA error %s\n", cs, names[cs], cudaGetErrorString(e));
      return 1;  // context is dead after an error
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, mag = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 32; ++n) {
        double r = 0;
        for (int k = 0; k < 8; ++k) r += (double)A[m * 8 + k] * B[k * 32 + n];
        err = fmax(err, fabs(r - D[m * 32 + n]));
        mag = fmax(mag, fabs(r));
      }
    printf("case %d %-36s max|err| %.3e (max|D| %.1f)\n", cs, names[cs], err, mag);
  }
  return 0;
}
