// Microbenchmark: issue rate of the Philox-4x32-10 chains alone (no FP64),
// and with the FP64 kinematics, to locate the issue-efficiency limit of k_spec.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__constant__ uint32_t K0[10], K1[10];
__device__ __forceinline__ void philox(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ K0[r], n2 = hi0 ^ c3 ^ K1[r];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
}
template <int NP, bool FP64>
__global__ void __launch_bounds__(256, 2) k(double* out, uint32_t iters) {
  const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * NP;
  double acc[NP];
  uint32_t xacc = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) acc[k] = 0.0;
  for (uint32_t t = 0; t < iters; ++t) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      uint32_t a0 = t, a1 = i0 + k, a2 = 0, a3 = 0;
      uint32_t b0 = t, b1 = i0 + k, b2 = 0, b3 = 1;
      philox(a0, a1, a2, a3);
      philox(b0, b1, b2, b3);
      if (FP64) {
        const double r1 = __dmul_rn(__ull2double_rn((uint64_t(a0) << 21) | (a1 >> 11)), 0x1.0p-53);
        const double r2 = __dmul_rn(__ull2double_rn((uint64_t(b0) << 21) | (b1 >> 11)), 0x1.0p-53);
        double v = __dadd_rn(__dadd_rn(acc[k], __dmul_rn(2.0, __dmul_rn(r1, 0.5))), __dmul_rn(2.0, __dmul_rn(r2, 0.25)));
        v = v < -50.0 ? -50.0 : (50.0 < v ? 50.0 : v);
        acc[k] = v;
      } else {
        xacc ^= a0 ^ a1 ^ b0 ^ b1;
      }
    }
  }
  double s = xacc;
#pragma unroll
  for (int k = 0; k < NP; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NP, bool FP64>
void run(const char* name, double* out) {
  int per_sm = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k<NP, FP64>, 256, 0);
  const int grid = per_sm * nsm;
  const uint32_t iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<NP, FP64><<<grid, 256>>>(out, 10);
  cudaEventRecord(a);
  k<NP, FP64><<<grid, 256>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double philox_calls = 2.0 * NP * iters * grid * 256.0;
  printf("%-22s grid=%d x 256 (per_sm %d): %.3f ms, %.3e particle-draw-pairs/s\n", name, grid, per_sm, ms,
         philox_calls / 2 / (ms * 1e-3));
}
int main() {
  uint32_t k0[10], k1[10], a = 1, b = 0;
  for (int r = 0; r < 10; ++r) { k0[r] = a; k1[r] = b; a += 0x9E3779B9u; b += 0xBB67AE85u; }
  cudaMemcpyToSymbol(K0, k0, sizeof k0); cudaMemcpyToSymbol(K1, k1, sizeof k1);
  double* out; cudaMalloc(&out, 148 * 8 * 256 * 8 * 8);
  run<1, false>("philox NP=1", out);
  run<4, false>("philox NP=4", out);
  run<1, true>("philox+fp64 NP=1", out);
  run<4, true>("philox+fp64 NP=4", out);
  return 0;
}
