// Check: integer round-to-nearest-away at the tf32 boundary ((u + 0x1000) &
// 0xFFFFE000) == cvt.rna.tf32.f32 for every finite fp32 bit pattern class
// (all exponents x mantissa patterns incl. ties), on the device.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/tf32_round_check tools/tf32_round_check.cu
#include <cstdio>
#include <cstdint>
__global__ void check(unsigned long long* bad, unsigned long long* n) {
  const uint32_t e = blockIdx.x;             // exponent 0..254 (finite)
  for (uint32_t m = threadIdx.x; m < (1u << 23); m += blockDim.x * 64) {
    for (int sub = 0; sub < 64; ++sub) {
      const uint32_t mm = (m + sub * blockDim.x) & 0x7FFFFFu;
      for (uint32_t s = 0; s < 2; ++s) {
        const uint32_t u = (s << 31) | (e << 23) | mm;
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(__uint_as_float(u)));
        const uint32_t q = (u + 0x1000u) & 0xFFFFE000u;
        if (q != r) atomicAdd(bad, 1ull);
        atomicAdd(n, 1ull);
      }
    }
  }
}
int main() {
  unsigned long long *bad, *n;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&n, 8); *bad = 0; *n = 0;
  check<<<255, 256>>>(bad, n);
  cudaDeviceSynchronize();
  printf("checked %llu patterns, mismatches %llu (%s)\n", *n, *bad, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
