// Microbenchmark: per-SMSP throughput of the integer ops Philox-4x32-10 is
// made of on sm_100a (IMAD.WIDE.U32, IMAD.HI.U32, IMAD, LOP3), to size the
// fma-pipe roof of the register-resident pass kernels.
// Each thread runs C independent chains; the grid fills every SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP, int C>
__global__ void __launch_bounds__(256) k(uint32_t* out, uint32_t iters, uint32_t m) {
  uint32_t x[C], y[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { x[c] = threadIdx.x * 7u + c; y[c] = blockIdx.x + c * 3u; }
  for (uint32_t t = 0; t < iters; ++t) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (OP == 0) {  // IMAD.WIDE.U32 + LOP3 (one Philox half-round)
        const uint64_t p = static_cast<uint64_t>(x[c]) * m;
        x[c] = static_cast<uint32_t>(p >> 32) ^ y[c] ^ t;
        y[c] = static_cast<uint32_t>(p);
      } else if (OP == 1) {  // IMAD.HI.U32 + LOP3
        x[c] = __umulhi(x[c], m) ^ y[c];
        y[c] += t;
      } else if (OP == 2) {  // IMAD (lo) only
        x[c] = x[c] * m + y[c];
      } else {  // LOP3 only
        x[c] = x[c] ^ y[c] ^ t;
        y[c] = (y[c] & x[c]) | m;
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s ^= x[c] ^ y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP, int C>
void run(const char* name, uint32_t* out, int nsm, double ops_per_chain_step) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k<OP, C>, 256, 0);
  const int grid = per_sm * nsm;
  const uint32_t iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<OP, C><<<grid, 256>>>(out, 10, 0xD2511F53u);
  cudaEventRecord(a);
  k<OP, C><<<grid, 256>>>(out, iters, 0xD2511F53u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double warp_steps = double(iters) * C * grid * 256 / 32;  // chain steps, per warp
  const double smsp_cycles = ms * 1e-3 * clk_khz * 1e3 * nsm * 4;
  printf("%-26s C=%d grid=%d: %.3f ms  %.3f warp-chain-steps/cycle/SMSP (%.2f cycles each)\n", name, C, grid, ms,
         warp_steps / smsp_cycles, smsp_cycles / warp_steps);
  (void)ops_per_chain_step;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  cudaMalloc(&out, 148 * 8 * 256 * 4 * 8);
  run<0, 4>("imad.wide+lop3", out, nsm, 2);
  run<0, 8>("imad.wide+lop3", out, nsm, 2);
  run<1, 8>("imad.hi+lop3(+iadd)", out, nsm, 3);
  run<2, 8>("imad", out, nsm, 1);
  run<3, 8>("lop3 x2", out, nsm, 2);
  return 0;
}
