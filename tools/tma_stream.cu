// TMA streaming probe: achievable HBM read bandwidth of 2-D tensor-map boxes
// (the stage-1 sketch's access pattern) with a per-CTA mbarrier ring and no
// consumers.  Rows x J fp32 matrix; each CTA streams a contiguous row range.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_stream tools/tma_stream.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int BOXR, int NSLOT, int COLSPLIT>
__global__ void __launch_bounds__(32, 1) stream(const __grid_constant__ CUtensorMap map, int rows, int J, int* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[NSLOT];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  constexpr int SLOT = BOXR * 128 * 4;  // 4 boxes of 32 columns per slot (= 128 columns)
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NSLOT; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // this CTA's row range (and, with COLSPLIT, its column half)
  const int nblk = gridDim.x / COLSPLIT, b = blockIdx.x / COLSPLIT, half = blockIdx.x % COLSPLIT;
  const int r0 = (int)((long long)rows * b / nblk), r1 = (int)((long long)rows * (b + 1) / nblk);
  const int c0 = half * (J / COLSPLIT), c1 = c0 + J / COLSPLIT;
  uint32_t n = 0;
  for (int r = r0; r < r1; r += BOXR)
    for (int c = c0; c < c1; c += 128, ++n) {
      const int s = n % NSLOT;
      if (n >= NSLOT) {  // wait for the previous fill of this slot, then reuse it
        uint32_t ok = 0, par = ((n / NSLOT) - 1) & 1;
        while (!ok)
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
              : "=r"(ok)
              : "r"(su32(&full[s])), "r"(par));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(SLOT));
      for (int ch = 0; ch < 4; ++ch)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(base + s * SLOT + ch * BOXR * 128)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(c + ch * 32), "r"(r), "r"(su32(&full[s]))
            : "memory");
    }
  for (uint32_t k = (n > NSLOT ? n - NSLOT : 0); k < n; ++k) {  // drain
    const int s = k % NSLOT;
    uint32_t ok = 0, par = (k / NSLOT) & 1;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&full[s])), "r"(par));
  }
  if (sink) sink[blockIdx.x] = base[0];
}

int main() {
  const int J = 512;
  const long long rows = 2300000;
  float* X;
  cudaMalloc(&X, rows * J * 4);
  cudaMemset(X, 0, rows * J * 4);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, int boxr, int nslot, int split, const char* name) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)J, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)J * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)boxr};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = boxr * 512 * nslot + 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) kern<<<sms, 32, smem>>>(map, (int)rows, J, nullptr);
    cudaEventRecord(a);
    for (int rep = 0; rep < 5; ++rep) kern<<<sms, 32, smem>>>(map, (int)rows, J, nullptr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-34s %.3f ms  %.0f GB/s  (%s)\n", name, ms, rows * J * 4.0 / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(stream<64, 5, 1>, 64, 5, 1, "box 32x64, 5 slots (160 KB)");
  run(stream<64, 5, 2>, 64, 5, 2, "box 32x64, 5 slots, column halves");
  run(stream<64, 3, 1>, 64, 3, 1, "box 32x64, 3 slots");
  run(stream<64, 6, 1>, 64, 6, 1, "box 32x64, 6 slots");
  run(stream<128, 3, 1>, 128, 3, 1, "box 32x128, 3 slots (192 KB)");
  run(stream<32, 10, 1>, 32, 10, 1, "box 32x32, 10 slots");
  return 0;
}
