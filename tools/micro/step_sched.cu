// Microbenchmark: instruction-scheduling variants of k_spec's d = 1 iteration
// body (NP = 4 cubic particles per thread, the reference's two Philox draws per
// particle, vel/pos step with clamps, cubic fitness, pbest compare), to test
// whether mixing the IMAD.WIDE-bound Philox with the FP64/select work inside a
// warp raises fma-heavy pipe utilisation. Compile like the library
// (-fmad=false). Run: ./step_sched
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2205_01313_b200/csrc/cupso_device.cuh"
using namespace cupso;


__device__ __forceinline__ void fence_block(uint32_t t) {
  // a block boundary ptxas cannot schedule across (never taken)
  if (t == 0xfffffff0u) asm volatile("trap;");
}

template <int V, int NP = 4>
__global__ void __launch_bounds__(256, 2) k(KParams P, double* out, uint32_t iters, double g) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t g0 = NP * u;
  double x[NP], v[NP], pb[NP], pbf[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    x[k] = 0.001 * (g0 + k);
    v[k] = 0.0;
    pb[k] = x[k];
    pbf[k] = 1e300;
  }
  uint32_t hits = 0;
  // V2 / V3: iteration t+1's draws computed during iteration t (all warps / odd warps only)
  const bool ahead = V == 2 || (V == 3 && ((threadIdx.x >> 5) & 1));
  double n1[NP], n2[NP];
  if (V >= 2) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      n1[k] = uniform53(P, 0, g0 + k, 0, 0);
      n2[k] = uniform53(P, 0, g0 + k, 0, 1);
    }
  }
  for (uint32_t t = 0; t < iters; ++t) {
    double f[NP];
    if constexpr (V >= 2) {
      if (ahead) {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const double r1 = n1[k], r2 = n2[k];
          n1[k] = uniform53(P, t + 1, g0 + k, 0, 0);
          n2[k] = uniform53(P, t + 1, g0 + k, 0, 1);
          v[k] = vel_step53(P, v[k], x[k], pb[k], g, r1, r2);
          x[k] = pos_step(P, x[k], v[k]);
          Fit<kCubic> a;
          a.add_first(x[k]);
          f[k] = a.value();
        }
      } else {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const double r1 = uniform53(P, t, g0 + k, 0, 0), r2 = uniform53(P, t, g0 + k, 0, 1);
          v[k] = vel_step53(P, v[k], x[k], pb[k], g, r1, r2);
          x[k] = pos_step(P, x[k], v[k]);
          Fit<kCubic> a;
          a.add_first(x[k]);
          f[k] = a.value();
        }
      }
    } else if constexpr (V == 0) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double r1 = uniform53(P, t, g0 + k, 0, 0), r2 = uniform53(P, t, g0 + k, 0, 1);
        v[k] = vel_step53(P, v[k], x[k], pb[k], g, r1, r2);
        x[k] = pos_step(P, x[k], v[k]);
        Fit<kCubic> a;
        a.add_first(x[k]);
        f[k] = a.value();
      }
    } else {
      // V1: two halves; the second half's Philox shares a block with the first half's kinematics
      double r1[NP], r2[NP];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        r1[k] = uniform53(P, t, g0 + k, 0, 0);
        r2[k] = uniform53(P, t, g0 + k, 0, 1);
      }
      fence_block(t);
#pragma unroll
      for (int k = 2; k < 4; ++k) {
        r1[k] = uniform53(P, t, g0 + k, 0, 0);
        r2[k] = uniform53(P, t, g0 + k, 0, 1);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        v[k] = vel_step53(P, v[k], x[k], pb[k], g, r1[k], r2[k]);
        x[k] = pos_step(P, x[k], v[k]);
        Fit<kCubic> a;
        a.add_first(x[k]);
        f[k] = a.value();
      }
      fence_block(t + 1);
#pragma unroll
      for (int k = 2; k < 4; ++k) {
        v[k] = vel_step53(P, v[k], x[k], pb[k], g, r1[k], r2[k]);
        x[k] = pos_step(P, x[k], v[k]);
        Fit<kCubic> a;
        a.add_first(x[k]);
        f[k] = a.value();
      }
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < NP; ++k) any |= f[k] > pbf[k];
    if (any) {
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (f[k] > pbf[k]) {
          pbf[k] = f[k];
          pb[k] = x[k];
          ++hits;
        }
    }
  }
  double s = hits;
#pragma unroll
  for (int k = 0; k < NP; ++k) s += x[k] + v[k] + pb[k];
  out[u] = s;
}

template <int V, int NP = 4>
void run(const char* name, const KParams& P, double* out, int nsm, int per_sm = 2) {
  const int grid = per_sm * nsm;
  const uint32_t iters = 4000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<V, NP><<<grid, 256>>>(P, out, 10, 0.5);
  cudaEventRecord(a);
  k<V, NP><<<grid, 256>>>(P, out, iters, 0.5);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %.3f ms  %.3e particle-updates/s\n", name, ms, double(grid) * 256 * NP * iters / (ms * 1e-3));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  KParams P{};
  P.w = 1.0; P.c1 = 2.0; P.c2 = 2.0;
  P.min_pos = -10; P.max_pos = 10; P.min_v = -10; P.max_v = 10;
  P.c1s = 2.0 * 0x1.0p-53; P.c2s = 2.0 * 0x1.0p-53; P.scaled_ok = 1;
  uint32_t a = 1, b = 0;
  for (int r = 0; r < 10; ++r) { P.k0[r] = a; P.k1[r] = b; a += 0x9E3779B9u; b += 0xBB67AE85u; }
  double* out;
  cudaMalloc(&out, 148 * 2 * 256 * 8 * 4);
  for (int rep = 0; rep < 2; ++rep) {
    run<0>("V0 straight (k_spec body)", P, out, nsm);
    run<1>("V1 halves, mixed blocks", P, out, nsm);
    // the tail round's shapes: per-particle rate of NP = 2 at full occupancy,
    // and of NP = 4 with half / a quarter of the warps
    run<0, 2>("V0 NP=2, 16 warps/SM", P, out, nsm);
    run<0, 4>("V0 NP=4, 8 warps/SM", P, out, nsm, 1);
    run<0, 1>("V0 NP=1, 16 warps/SM", P, out, nsm);
    run<2>("V2 draw-ahead, all warps", P, out, nsm);
    run<3>("V3 draw-ahead, odd warps", P, out, nsm);
  }
  return 0;
}
