// Feasibility probe for an int8 (Ozaki-split) tcgen05 product and for L2
// re-reads of a streamed tile:
//   1. tcgen05.mma kind::i8, M=128, K=32, N in {32, 64, 128, 224, 256},
//      K-major SWIZZLE_128B A/B from shared memory, s32 accumulate: exactness
//      against a host reference (s8 x s8, u8 x u8, s8 x u8) and the issue rate
//      on every SM (back-to-back MMAs into one accumulator).
//   2. streaming read of a large buffer by 148 CTAs, each tile read twice with
//      a lag of one tile (second read should hit L2) vs read once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o i8_probe tools/i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::i8: D s32 (2), A/B 0 = u8, 1 = s8
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int as, int bs) {
  return (2u << 4) | ((uint32_t)as << 7) | ((uint32_t)bs << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
// K-major SW128: row r (of M or N), byte k (< 128)
__device__ __forceinline__ uint32_t swz8(int r, int k) {
  return (uint32_t)r * 128u + ((uint32_t)(((k >> 4) ^ r) & 7) << 4) + (uint32_t)(k & 15);
}

__global__ void mma_probe(int N, int as, int bs, const int8_t* A, const int8_t* B, int* D, int reps,
                          long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar;
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  unsigned char* As = base;              // 128 x 128 B (K = 128 bytes: 4 MMAs of K=32)
  unsigned char* Bs = base + 128 * 128;  // 256 x 128 B
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 128; e += blockDim.x) As[swz8(e / 128, e % 128)] = (unsigned char)A[e];
  for (int e = tid; e < 256 * 128; e += blockDim.x) Bs[swz8(e / 128, e % 128)] = (unsigned char)B[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N, as, bs);
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int kk = 0; kk < 4; ++kk) {
        // K-major SW128: the K=32 slice kk starts 32 B into the 128 B row (row 0's granule)
        const uint64_t ad = sdesc(su32(As) + kk * 32, 16, 1024);
        const uint64_t bd = sdesc(su32(Bs) + kk * 32, 16, 1024);
        const uint32_t acc = (r | kk) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
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
  if (tid == 0) {
    t1 = clock64();
    if (blockIdx.x == 0) cycles[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (blockIdx.x == 0) {
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int c = 0; c < 32; ++c) D[(warp * 32 + (tid & 31)) * 256 + c0 + c] = (int)v[c];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// 148 CTAs, each streams its contiguous share in tiles of `tile` bytes; with
// twice=1 every tile t is read again after tile t+1 (lag of one tile)
__global__ void l2_probe(const double2* __restrict__ X, size_t per_cta, size_t tile, int twice, double* sink) {
  const double2* base = X + (size_t)blockIdx.x * (per_cta / 16);
  const size_t nt = per_cta / tile, tv = tile / 16;
  double acc = 0;
  for (size_t t = 0; t < nt; ++t) {
    const double2* p = base + t * tv;
    for (size_t i = threadIdx.x; i < tv; i += blockDim.x) {
      double2 v = __ldg(p + i);
      acc += v.x + v.y;
    }
    if (twice && t > 0) {
      const double2* q = base + (t - 1) * tv;
      for (size_t i = threadIdx.x; i < tv; i += blockDim.x) {
        double2 v = __ldg(q + i);
        acc += v.x - v.y;
      }
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  const int nsm = prop.multiProcessorCount;
  std::vector<int8_t> A(128 * 128), B(256 * 128);
  srand(1);
  for (auto& a : A) a = (int8_t)(rand() & 255);
  for (auto& b : B) b = (int8_t)(rand() & 255);
  int8_t *dA, *dB;
  int* dD;
  long long* dc;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * 256 * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  const int smem = 128 * 128 + 256 * 128 + 2048;
  cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<int> D(128 * 256);
  const int sg[3][2] = {{1, 1}, {0, 0}, {1, 0}};
  for (int c = 0; c < 3; ++c) {
    const int as = sg[c][0], bs = sg[c][1], N = 224;
    mma_probe<<<1, 128, smem>>>(N, as, bs, dA, dB, dD, 1, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mma error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long long bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        long long r = 0;
        for (int k = 0; k < 128; ++k) {
          const int a = as ? (int)A[m * 128 + k] : (int)(uint8_t)A[m * 128 + k];
          const int b = bs ? (int)B[n * 128 + k] : (int)(uint8_t)B[n * 128 + k];
          r += a * b;
        }
        if (r != D[m * 256 + n]) ++bad;
      }
    printf("exactness a_signed=%d b_signed=%d N=%d: %lld mismatches of %d\n", as, bs, N, bad, 128 * N);
  }
  const int Ns[] = {32, 64, 128, 224, 256};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int N : Ns) {
    const int reps = 4096;
    mma_probe<<<nsm, 128, smem>>>(N, 1, 0, dA, dB, dD, 64, dc);
    cudaEventRecord(e0);
    mma_probe<<<nsm, 128, smem>>>(N, 1, 0, dA, dB, dD, reps, dc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    const double macs = (double)nsm * reps * 4 * 128.0 * N * 32;
    printf("i8 M=128 N=%3d K=32: %.1f TOPS (event), %.1f MAC/clk/SM (clock64 %lld cycles, %.1f clk/MMA)\n", N,
           2 * macs / (ms * 1e-3) / 1e12, (double)reps * 4 * 128 * N * 32 / cyc, cyc, (double)cyc / (reps * 4));
  }
  // L2 re-read probe
  const size_t total = 9ull << 30;
  double2* X;
  double* sink;
  if (cudaMalloc(&X, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&sink, 8);
  cudaMemset(X, 0, total);
  const size_t per = (total / nsm) & ~((size_t)(1 << 20) - 1);
  const size_t tiles[] = {64 << 10, 128 << 10, 256 << 10, 512 << 10};
  for (size_t tile : tiles) {
    const size_t pc = per / tile * tile;
    float ms[2];
    for (int tw = 0; tw < 2; ++tw) {
      l2_probe<<<nsm, 1024>>>(X, pc, tile, tw, sink);
      cudaEventRecord(e0);
      l2_probe<<<nsm, 1024>>>(X, pc, tile, tw, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms[tw], e0, e1);
    }
    printf("tile %4zu KB (footprint ~%zu MB): once %.3f ms (%.0f GB/s), twice %.3f ms (ratio %.3f)\n", tile >> 10,
           2 * tile * nsm >> 20, ms[0], (double)pc * nsm / (ms[0] * 1e6), ms[1], ms[1] / ms[0]);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(e));
  return 0;
}
