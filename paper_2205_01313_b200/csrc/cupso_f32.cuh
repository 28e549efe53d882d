// cupso_f32.cuh -- the FP32 engine "cuda-sync-f32".
//
// The reference is FP64 throughout (swarm.hpp:31-35); this engine
// is the north star's FP32 shape of the same synchronous algorithm, checked
// statistically rather than bitwise:
//   * state as FP32 SoA rows, 4 adjacent particles per thread moved with one
//     float4 (LDG.128 / STG.128) per row;
//   * one Philox-4x32-10 call per (iteration pair, particle, axis): words 0/1
//     give (r1, r2) on the even iteration, words 2/3 on the odd one (the FP64
//     engines draw two calls per iteration, slots 0/1, using two words each);
//   * kinematics with FMA and FMNMX clamps, fitness in FP32;
//   * the gbest aggregation is the paper's atomic scheme on a packed 64-bit
//     key: (order-preserving FP32 fitness << 32) | ~particle, so one u64
//     atomicMax is "fitness descending, ties to the lower index" (beats(),
//     engine.hpp:38-41) -- warp shuffle max, one SMEM atomicMax per warp into
//     the block's slot, one global atomicMax per block;
//   * the speculative register-resident passes of k_spec (cupso_spec.cuh),
//     same SpecCtl schedule and spec_decide.
// The handle keeps the FP64 state authoritative for every other entry point:
// it is converted to FP32 when a cuda-sync-f32 step starts and back when any
// FP64 consumer (another engine, download, device pointers) needs it.
#pragma once

#include "cupso_spec.cuh"

namespace cupso {

struct KState32 {
  float* pos;
  float* vel;
  float* pb;
  float* pbf;
};

// Run parameters in FP32 (rounded from the FP64 pso_params on the host).
struct KParams32 {
  float w, c1, c2, min_pos, max_pos, min_v, max_v;
};

// cos(2 pi v) for the FP32 rastrigin term: a = 2v and its nearest integer k
// are exact, so r = a - k in [-0.5, 0.5] is the exact reduced argument and
// cos(2 pi v) = (-1)^k cos(pi r); cos(pi r) is a degree-5 polynomial in r^2
// (Chebyshev fit, max error 1.2e-7 ~ 1 ulp at 1, the class of cospif) --
// branch-free and about half of cospif's instructions.
__device__ __forceinline__ float cos2pi_f32(float v) {
  const float a = 2.f * v;
  const float k = rintf(a);
  const float r = __fsub_rn(a, k);
  const float z = __fmul_rn(r, r);
  float c = __fmaf_rn(z, -0.02439611405134201f, 0.2349332571029663f);
  c = __fmaf_rn(z, c, -1.3352099657058716f);
  c = __fmaf_rn(z, c, 4.058708667755127f);
  c = __fmaf_rn(z, c, -4.934802055358887f);
  c = __fmaf_rn(z, c, 1.f);
  const uint32_t odd = __float_as_uint(__fadd_rn(k, 0x1.8p23f)) & 1u;  // parity of k (|k| < 2^22)
  return __uint_as_float(__float_as_uint(c) ^ (odd << 31));
}

template <int F>
struct Fit32;
template <>
struct Fit32<kCubic> {
  float acc = 0.f;
  __device__ __forceinline__ void add(float v, uint32_t) {
    acc += __fmaf_rn(__fmaf_rn(v - 0.8f, v, -1000.f), v, 8000.f);
  }
  __device__ __forceinline__ float value() const { return acc; }
  __device__ __forceinline__ void merge_xor(int off, int w) { acc += __shfl_xor_sync(0xffffffffu, acc, off, w); }
};
template <>
struct Fit32<kSphere> {
  float acc = 0.f;
  __device__ __forceinline__ void add(float v, uint32_t) { acc = __fmaf_rn(v, v, acc); }
  __device__ __forceinline__ float value() const { return -acc; }
  __device__ __forceinline__ void merge_xor(int off, int w) { acc += __shfl_xor_sync(0xffffffffu, acc, off, w); }
};
template <>
struct Fit32<kRosenbrock> {
  float acc = 0.f, prev = 0.f;
  __device__ __forceinline__ void add(float v, uint32_t axis) {
    if (axis > 0) {
      const float a = __fmaf_rn(-prev, prev, v);
      const float b = 1.f - prev;
      acc += __fmaf_rn(100.f * a, a, b * b);
    }
    prev = v;
  }
  __device__ __forceinline__ float value() const { return -acc; }
  __device__ __forceinline__ void merge_xor(int off, int w) { acc += __shfl_xor_sync(0xffffffffu, acc, off, w); }
};
template <>
struct Fit32<kGriewank> {
  float sum = 0.f, prod = 1.f;
  __device__ __forceinline__ void add(float v, uint32_t axis) {
    sum = __fmaf_rn(v * v, 1.f / 4000.f, sum);
    prod *= cosf(v * rsqrtf(static_cast<float>(axis + 1)));
  }
  __device__ __forceinline__ float value() const { return -((1.f + sum) - prod); }
  __device__ __forceinline__ void merge_xor(int off, int w) {
    sum += __shfl_xor_sync(0xffffffffu, sum, off, w);
    prod *= __shfl_xor_sync(0xffffffffu, prod, off, w);
  }
};
template <>
struct Fit32<kRastrigin> {
  float acc = 0.f;
  __device__ __forceinline__ void add(float v, uint32_t) {
    acc += __fmaf_rn(v, v, __fmaf_rn(-10.f, cos2pi_f32(v), 10.f));
  }
  __device__ __forceinline__ float value() const { return -acc; }
  __device__ __forceinline__ void merge_xor(int off, int w) { acc += __shfl_xor_sync(0xffffffffu, acc, off, w); }
};

// Packed (fitness, particle) key: u64 max == beats() order.
__device__ __forceinline__ unsigned long long key32(float f, uint32_t i) {
  const uint32_t b = __float_as_uint(f);
  const uint32_t o = (b >> 31) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(o) << 32) | static_cast<unsigned long long>(~i);
}
__device__ __forceinline__ float key_fit(unsigned long long k) {
  const uint32_t o = static_cast<uint32_t>(k >> 32);
  return __uint_as_float((o >> 31) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ uint32_t key_idx(unsigned long long k) { return ~static_cast<uint32_t>(k); }

template <int NP>
__device__ __forceinline__ void ldv32(const float* p, float (&o)[NP]) {
  if constexpr (NP == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    o[0] = t.x;
    o[1] = t.y;
    o[2] = t.z;
    o[3] = t.w;
  } else if constexpr (NP == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    o[0] = t.x;
    o[1] = t.y;
  } else {
    o[0] = *p;
  }
}
template <int NP>
__device__ __forceinline__ void stv32(float* p, const float (&o)[NP]) {
  if constexpr (NP == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  } else if constexpr (NP == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(o[0], o[1]);
  } else {
    *p = o[0];
  }
}

// The FP32 stream: one Philox call per particle-axis and PAIR of iterations,
// counter {t/2, particle, axis, 0}; even iterations take words 0/1 as (r1, r2),
// odd ones words 2/3 -- all four words used, a quarter of the FP64 engines'
// draw cost. 24-bit uniforms in [0, 1).
__device__ __forceinline__ float u24(uint32_t w) { return __uint2float_rz(w >> 8) * 0x1.0p-24f; }
__device__ __forceinline__ void philox_pair(const KParams& P, uint32_t t, uint32_t i, uint32_t axis, uint32_t& w0,
                                            uint32_t& w1, uint32_t& w2, uint32_t& w3) {
  w0 = t >> 1;
  w1 = i;
  w2 = axis;
  w3 = 0;
  philox10(w0, w1, w2, w3, P);
}
__device__ __forceinline__ void uniform2_f32(const KParams& P, uint32_t t, uint32_t i, uint32_t axis, float& r1,
                                             float& r2) {
  uint32_t w0, w1, w2, w3;
  philox_pair(P, t, i, axis, w0, w1, w2, w3);
  r1 = u24((t & 1u) ? w2 : w0);
  r2 = u24((t & 1u) ? w3 : w1);
}

// The key slot of the pass lives right after SpecCtl in the control buffer.
struct SpecCtl32 {
  SpecCtl ctl;
  unsigned long long key;  // best (fit, particle) admitted at the pass's last iteration
};

// Pass tail shared by the FP32 pass kernels.
__device__ __forceinline__ void spec32_finish(const KParams& P, const KState32& So, const KCtl& C, SpecCtl32* sc32,
                                              unsigned long long& s_key, unsigned long long& s_adm, int& s_last,
                                              uint32_t t_end, uint32_t kmax, unsigned char* rec_out, uint32_t tl,
                                              unsigned long long bkey, uint32_t adm) {
  SpecCtl* sc = &sc32->ctl;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const size_t ld = P.ld;
  // ---- aggregation: warp shuffle max of the packed key, one SMEM atomicMax
  // per warp, one global atomicMax per block (the paper's atomic scheme)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, bkey, off);
    bkey = o > bkey ? o : bkey;
  }
  const uint32_t wadm = __reduce_add_sync(0xffffffffu, adm);
  if (lane == 0) {
    if (bkey) atomicMax(&s_key, bkey);
    if (wadm) atomicAdd(&s_adm, static_cast<unsigned long long>(wadm));
  }
  __syncthreads();
  if (tid == 0) {
    if (s_key) atomicMax(&sc32->key, s_key);
    if (s_adm) atomicAdd(&C.admitted[tl], s_adm);
    __threadfence();
    s_last = last_block_done(C);
  }
  __syncthreads();
  if (!s_last) return;
  // ---- last block: the pass record, then the shared decision (spec_decide)
  __threadfence();
  const unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(&sc32->key);
  SpecRec* rec = reinterpret_cast<SpecRec*>(rec_out);
  double* rpos = reinterpret_cast<double*>(rec_out + sizeof(SpecRec));
  const uint32_t wi = key ? key_idx(key) : kNoParticle;
  for (uint32_t a = tid; a < P.d; a += blockDim.x)
    rpos[a] = key ? static_cast<double>(__ldcg(&So.pos[static_cast<size_t>(a) * ld + (wi - P.base)])) : 0.0;
  if (tid == 0) {
    rec->tmin = ld_volatile_u32(&sc->tmin);
    rec->admitted = static_cast<uint32_t>(__ldcg(&C.admitted[tl]));
    rec->fit = key ? static_cast<double>(key_fit(key)) : -INFINITY;
    rec->particle = wi;
    rec->pad = 0;
    C.admitted[tl] = 0;
    sc32->key = 0;
    __threadfence();
  }
  __syncthreads();
  spec_decide(P, C, sc, rec_out, 1, t_end, kmax);
}

// One thread unit of a k_spec32 pass (NP adjacent particles from li); false
// when the pass already failed at t0. As spec_unit of the FP64 kernels.
template <int F, int D, int NP>
__device__ __forceinline__ bool spec32_unit(const KParams& P, const KParams32& Q, const KState32& Si,
                                            const KState32& So, SpecCtl* sc, uint32_t li, uint32_t t0, uint32_t K,
                                            bool inplace, float snap_fit, const float (&gp)[D], uint32_t& tstop,
                                            unsigned long long& bkey, uint32_t& adm) {
  const uint32_t tl = t0 + K - 1;
  const size_t ld = P.ld;
  tstop = min(tstop, ld_relaxed_gpu(&sc->tmin));
  uint32_t te = min(t0 + K, tstop);
  if (te <= t0) return false;
  const uint32_t g0 = P.base + li;
  float x[D][NP], v[D][NP], pb[D][NP], pbf[NP];
  bool ok[NP];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const size_t at = static_cast<size_t>(a) * ld + li;
    ldv32<NP>(Si.pos + at, x[a]);
    ldv32<NP>(Si.vel + at, v[a]);
    ldv32<NP>(Si.pb + at, pb[a]);
  }
  ldv32<NP>(Si.pbf + li, pbf);
#pragma unroll
  for (int k = 0; k < NP; ++k) ok[k] = k == 0 || li + k < P.n;
  uint32_t t = t0;
  bool bad = false, dirty = false;
  uint32_t odd_w[D][NP][2];  // words 2/3 of the pair's call, for its odd iteration
  for (; t < te; ++t) {
    Fit32<F> acc[NP];
    // warp-uniform: a fresh call on even iterations (and on a unit's first)
    const bool fresh = !(t & 1u) || t == t0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        float r1, r2;
        if (fresh) {
          uint32_t w0, w1;
          philox_pair(P, t, g0 + k, a, w0, w1, odd_w[a][k][0], odd_w[a][k][1]);
          r1 = u24((t & 1u) ? odd_w[a][k][0] : w0);
          r2 = u24((t & 1u) ? odd_w[a][k][1] : w1);
        } else {
          r1 = u24(odd_w[a][k][0]);
          r2 = u24(odd_w[a][k][1]);
        }
        const float xv = x[a][k];
        float nv = __fmaf_rn(Q.c2 * r2, gp[a] - xv, __fmaf_rn(Q.c1 * r1, pb[a][k] - xv, Q.w * v[a][k]));
        nv = fminf(fmaxf(nv, Q.min_v), Q.max_v);
        const float nx = fminf(fmaxf(xv + nv, Q.min_pos), Q.max_pos);
        v[a][k] = nv;
        x[a][k] = nx;
        acc[k].add(nx, a);
      }
    }
    float fv[NP];
    bool any = false;  // fast path: the snapshot is >= every pbest (see k_spec)
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      fv[k] = acc[k].value();
      any |= ok[k] && fv[k] > pbf[k];
    }
    if (any) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const float f = fv[k];
        if (!ok[k]) continue;
        if (f > pbf[k]) {
          dirty = true;
          pbf[k] = f;
#pragma unroll
          for (int a = 0; a < D; ++a) pb[a][k] = x[a][k];
        }
        if (f > snap_fit) {
          if (t < tl) {
            bad = true;
          } else {
            ++adm;
            const unsigned long long kk = key32(f, g0 + k);
            bkey = kk > bkey ? kk : bkey;
          }
        }
      }
      if (bad) {
        atomicMin(&sc->tmin, t);
        tstop = t;
        break;
      }
    }
    if (((t - t0) & 15u) == 15u) {
      tstop = min(tstop, ld_relaxed_gpu(&sc->tmin));
      te = min(te, tstop);
    }
  }
  if (!bad && t == t0 + K) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const size_t at = static_cast<size_t>(a) * ld + li;
      stv32<NP>(So.pos + at, x[a]);
      stv32<NP>(So.vel + at, v[a]);
    }
    if (!inplace || dirty) {
#pragma unroll
      for (int a = 0; a < D; ++a) stv32<NP>(So.pb + static_cast<size_t>(a) * ld + li, pb[a]);
      stv32<NP>(So.pbf + li, pbf);
    }
  }
  return true;
}

template <int F, int D, int NP, int MINB>
__global__ void __launch_bounds__(kSyncThreads, MINB) k_spec32(KParams P, KParams32 Q, KState32 S0, KState32 S1,
                                                              KCtl C, SpecCtl32* sc32, uint32_t t_end, uint32_t kmax,
                                                              unsigned char* rec_out) {
  __shared__ float s_gpos[D];
  __shared__ unsigned long long s_key;
  __shared__ unsigned long long s_adm;
  __shared__ uint32_t s_ctl[4];
  __shared__ int s_last;
  SpecCtl* sc = &sc32->ctl;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    s_ctl[0] = ld_volatile_u32(&sc->t0);
    s_ctl[1] = ld_volatile_u32(&sc->K);
    s_ctl[2] = ld_volatile_u32(&sc->parity);
    s_ctl[3] = ld_volatile_u32(&sc->kspec);
    s_key = 0;
    s_adm = 0;
  }
  if (tid < D) s_gpos[tid] = static_cast<float>(C.snap_pos[tid]);
  __syncthreads();
  const uint32_t t0 = s_ctl[0], K = s_ctl[1], par = s_ctl[2];
  if (t0 >= t_end) return;
  const bool inplace = K == 1;
  const KState32 Si = par ? S1 : S0;
  const KState32 So = inplace ? Si : (par ? S0 : S1);
  // the FP32 engine filters against the FP32 value of the snapshot fitness
  const float snap_fit = static_cast<float>(C.snap->fit);
  const uint32_t tl = t0 + K - 1;
  float gp[D];
#pragma unroll
  for (int a = 0; a < D; ++a) gp[a] = s_gpos[a];
  unsigned long long bkey = 0;
  uint32_t adm = 0;
  uint32_t tstop = ld_relaxed_gpu(&sc->tmin);
  // full rounds of NP-particle units, then -- when the last round would be at
  // most half full -- one round of NP/2-particle units (as k_spec)
  const uint32_t nthr = gridDim.x * blockDim.x, gt = blockIdx.x * blockDim.x + tid;
  uint32_t n_main = P.n;
  if constexpr (NP >= 2) {
    const uint32_t rem = P.n % (NP * nthr);
    if (rem && rem <= (NP / 2) * nthr) n_main = P.n - rem;
  }
  const uint32_t units = (n_main + NP - 1) / NP;
  bool live = true;
  for (uint32_t u = gt; u < units; u += nthr) {
    if (!(live = spec32_unit<F, D, NP>(P, Q, Si, So, sc, NP * u, t0, K, inplace, snap_fit, gp, tstop, bkey, adm)))
      break;
  }
  if constexpr (NP >= 2) {
    const uint32_t li = n_main + (NP / 2) * gt;
    if (live && li < P.n)
      spec32_unit<F, D, NP / 2>(P, Q, Si, So, sc, li, t0, K, inplace, snap_fit, gp, tstop, bkey, adm);
  }
  spec32_finish(P, So, C, sc32, s_key, s_adm, s_last, t_end, kmax, rec_out, tl, bkey, adm);
}

// Wide FP32 swarms (d > 8, up to 256): G lanes per particle, 8 axis slots each
// (the last lane group ragged when d < 8 G), as k_spec_split -- but the FP32
// engine is statistical, so the lanes' partial fitnesses combine by a
// butterfly (shfl_xor) instead of the FP64 kernels' ordered fold.
template <int F, int DL, int G, int MINB>
__global__ void __launch_bounds__(kSyncThreads, MINB) k_spec32_split(KParams P, KParams32 Q, KState32 S0, KState32 S1,
                                                                    KCtl C, SpecCtl32* sc32, uint32_t t_end,
                                                                    uint32_t kmax, unsigned char* rec_out) {
  static_assert(32 % G == 0, "G must divide the warp");
  __shared__ float s_gpos[DL * G];
  __shared__ unsigned long long s_key, s_adm;
  __shared__ uint32_t s_ctl[4];
  __shared__ int s_last;
  SpecCtl* sc = &sc32->ctl;
  const uint32_t tid = threadIdx.x, lane = tid & 31, sub = lane % G, a0 = sub * DL;
  if (tid == 0) {
    s_ctl[0] = ld_volatile_u32(&sc->t0);
    s_ctl[1] = ld_volatile_u32(&sc->K);
    s_ctl[2] = ld_volatile_u32(&sc->parity);
    s_ctl[3] = ld_volatile_u32(&sc->kspec);
    s_key = 0;
    s_adm = 0;
  }
  for (uint32_t a = tid; a < DL * G; a += blockDim.x) s_gpos[a] = a < P.d ? static_cast<float>(C.snap_pos[a]) : 0.f;
  __syncthreads();
  const uint32_t t0 = s_ctl[0], K = s_ctl[1], par = s_ctl[2];
  if (t0 >= t_end) return;
  const bool inplace = K == 1;
  const KState32 Si = par ? S1 : S0;
  const KState32 So = inplace ? Si : (par ? S0 : S1);
  const float snap_fit = static_cast<float>(C.snap->fit);
  const uint32_t tl = t0 + K - 1;
  auto valid = [&](int a) { return a0 + a < P.d; };
  unsigned long long bkey = 0;
  uint32_t adm = 0;
  uint32_t tstop = warp_tmin(&sc->tmin);
  const uint32_t stride = gridDim.x * (blockDim.x / G);
  const size_t ld = P.ld;
  for (uint32_t u0 = (blockIdx.x * blockDim.x + (tid & ~31u)) / G; u0 < P.n; u0 += stride) {  // warp-uniform
    tstop = min(tstop, warp_tmin(&sc->tmin));
    uint32_t te = min(t0 + K, tstop);
    if (te <= t0) break;
    const uint32_t li = u0 + lane / G;
    const bool live = li < P.n;
    const uint32_t gi = P.base + li;
    float x[DL], v[DL], pb[DL], pbf = -INFINITY;
#pragma unroll
    for (int a = 0; a < DL; ++a) {
      x[a] = v[a] = pb[a] = 0.f;
      if (live && valid(a)) {
        const size_t at = static_cast<size_t>(a0 + a) * ld + li;
        x[a] = Si.pos[at];
        v[a] = Si.vel[at];
        pb[a] = Si.pb[at];
      }
    }
    if (live) pbf = Si.pbf[li];
    uint32_t t = t0;
    bool bad = false, dirty = false;
    uint32_t odd_w[DL][2];
    for (; t < te; ++t) {
      const bool fresh = !(t & 1u) || t == t0;
#pragma unroll
      for (int a = 0; a < DL; ++a) {
        if (!valid(a)) continue;
        float r1, r2;
        if (fresh) {
          uint32_t w0, w1;
          philox_pair(P, t, gi, a0 + a, w0, w1, odd_w[a][0], odd_w[a][1]);
          r1 = u24((t & 1u) ? odd_w[a][0] : w0);
          r2 = u24((t & 1u) ? odd_w[a][1] : w1);
        } else {
          r1 = u24(odd_w[a][0]);
          r2 = u24(odd_w[a][1]);
        }
        const float xv = x[a];
        float nv = __fmaf_rn(Q.c2 * r2, s_gpos[a0 + a] - xv, __fmaf_rn(Q.c1 * r1, pb[a] - xv, Q.w * v[a]));
        nv = fminf(fmaxf(nv, Q.min_v), Q.max_v);
        v[a] = nv;
        x[a] = fminf(fmaxf(xv + nv, Q.min_pos), Q.max_pos);
      }
      Fit32<F> acc;
      if constexpr (F == kRosenbrock) acc.prev = __shfl_up_sync(0xffffffffu, x[DL - 1], 1, G);  // left lane's last axis
#pragma unroll
      for (int a = 0; a < DL; ++a)
        if (valid(a)) acc.add(x[a], a0 + a);
#pragma unroll
      for (int off = 1; off < G; off <<= 1) acc.merge_xor(off, G);
      const float f = acc.value();
      if (live && f > pbf) {
        dirty = true;
        pbf = f;
#pragma unroll
        for (int a = 0; a < DL; ++a) pb[a] = x[a];
      }
      bool early = false;
      if (live && f > snap_fit) {
        if (t < tl) {
          early = true;
        } else if (sub == 0) {
          ++adm;
          const unsigned long long kk = key32(f, gi);
          bkey = kk > bkey ? kk : bkey;
        }
      }
      if (__any_sync(0xffffffffu, early)) {
        if (lane == 0) atomicMin(&sc->tmin, t);
        tstop = t;
        bad = true;
        break;
      }
      if (((t - t0) & 15u) == 15u) {
        tstop = min(tstop, warp_tmin(&sc->tmin));
        te = min(te, tstop);
      }
    }
    if (!bad && t == t0 + K && live) {
#pragma unroll
      for (int a = 0; a < DL; ++a) {
        if (!valid(a)) continue;
        const size_t at = static_cast<size_t>(a0 + a) * ld + li;
        So.pos[at] = x[a];
        So.vel[at] = v[a];
        if (!inplace || dirty) So.pb[at] = pb[a];
      }
      if (sub == 0 && (!inplace || dirty)) So.pbf[li] = pbf;
    }
  }
  spec32_finish(P, So, C, sc32, s_key, s_adm, s_last, t_end, kmax, rec_out, tl, bkey, adm);
}

// Any dims: one launch per iteration, one particle per thread, state in HBM
// (the dims without a register-resident k_spec32 instantiation). Same RNG,
// arithmetic and packed-key aggregation; the last block adopts the winner.
template <int F>
__global__ void __launch_bounds__(kSyncThreads) k_wave32(KParams P, KParams32 Q, KState32 S, KCtl C,
                                                         SpecCtl32* sc32, uint32_t t) {
  __shared__ unsigned long long s_key, s_adm;
  __shared__ int s_last;
  extern __shared__ float s_g[];  // [d] snapshot position
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    s_key = 0;
    s_adm = 0;
  }
  for (uint32_t a = tid; a < P.d; a += blockDim.x) s_g[a] = static_cast<float>(C.snap_pos[a]);
  __syncthreads();
  const float snap_fit = static_cast<float>(C.snap->fit);
  const size_t ld = P.ld;
  unsigned long long bkey = 0;
  uint32_t adm = 0;
  for (uint32_t li = blockIdx.x * blockDim.x + tid; li < P.n; li += gridDim.x * blockDim.x) {
    const uint32_t gi = P.base + li;
    Fit32<F> acc;
    for (uint32_t a = 0; a < P.d; ++a) {
      const size_t at = static_cast<size_t>(a) * ld + li;
      float r1, r2;
      uniform2_f32(P, t, gi, a, r1, r2);
      const float xv = S.pos[at];
      float nv = __fmaf_rn(Q.c2 * r2, s_g[a] - xv, __fmaf_rn(Q.c1 * r1, S.pb[at] - xv, Q.w * S.vel[at]));
      nv = fminf(fmaxf(nv, Q.min_v), Q.max_v);
      const float nx = fminf(fmaxf(xv + nv, Q.min_pos), Q.max_pos);
      S.vel[at] = nv;
      S.pos[at] = nx;
      acc.add(nx, a);
    }
    const float f = acc.value();
    if (f > S.pbf[li]) {
      S.pbf[li] = f;
      for (uint32_t a = 0; a < P.d; ++a) {
        const size_t at = static_cast<size_t>(a) * ld + li;
        S.pb[at] = S.pos[at];
      }
    }
    if (f > snap_fit) {
      ++adm;
      const unsigned long long kk = key32(f, gi);
      bkey = kk > bkey ? kk : bkey;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, bkey, off);
    bkey = o > bkey ? o : bkey;
  }
  const uint32_t wadm = __reduce_add_sync(0xffffffffu, adm);
  if (lane == 0) {
    if (bkey) atomicMax(&s_key, bkey);
    if (wadm) atomicAdd(&s_adm, static_cast<unsigned long long>(wadm));
  }
  __syncthreads();
  if (tid == 0) {
    if (s_key) atomicMax(&sc32->key, s_key);
    if (s_adm) atomicAdd(&C.admitted[t], s_adm);
    __threadfence();
    s_last = last_block_done(C);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(&sc32->key);
  if (key) {
    const uint32_t wi = key_idx(key);
    for (uint32_t a = tid; a < P.d; a += blockDim.x)
      C.snap_pos[a] = static_cast<double>(__ldcg(&S.pos[static_cast<size_t>(a) * ld + (wi - P.base)]));
  }
  __syncthreads();
  if (tid == 0) {
    if (key) {  // every admitted key beat the snapshot: adopt the max
      C.snap->fit = static_cast<double>(key_fit(key));
      C.snap->particle = key_idx(key);
    }
    C.trace[t] = C.snap->fit;
    C.trace_idx[t] = C.snap->particle;
    sc32->key = 0;
  }
}

// FP64 <-> FP32 state conversion (rows of ld, all 3d+1 arrays).
__global__ void k_to_f32(KParams P, KState S, KState32 T) {
  const size_t cells = static_cast<size_t>(P.d) * P.ld;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    T.pos[i] = static_cast<float>(S.pos[i]);
    T.vel[i] = static_cast<float>(S.vel[i]);
    T.pb[i] = static_cast<float>(S.pb[i]);
    if (i < P.ld) T.pbf[i] = static_cast<float>(S.pbf[i]);
  }
}
__global__ void k_to_f64(KParams P, KState32 T, KState S) {
  const size_t cells = static_cast<size_t>(P.d) * P.ld;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    S.pos[i] = T.pos[i];
    S.vel[i] = T.vel[i];
    S.pb[i] = T.pb[i];
    if (i < P.ld) S.pbf[i] = T.pbf[i];
  }
}

}  // namespace cupso
