// cupso_device.cuh -- device-side building blocks of the PSO step (sm_100a).
//
// Every function here restates one reference function bit for bit:
//   philox10 / uniform01  <- rng.hpp:36-62
//   clampd / vel_step / pos_step <- swarm.hpp:56-77
//   Fit* accumulators     <- fitness.hpp:47-85 (+ harness Rastrigin)
//   beats                 <- engine.hpp:38-41
// FP64 arithmetic uses explicit _rn intrinsics in the reference's evaluation
// order, and the whole library is compiled with -fmad=false: the reference
// builds with -ffp-contract=off (proj/CMakeLists.txt:17-20), so an FMA
// contraction here would change the trajectory's last bits.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cupso {

constexpr uint32_t kNoParticle = 0xffffffffu;  // swarm.hpp:16

// Kernel-uniform run parameters, passed by value (lives in the constant bank).
struct KParams {
  double w, c1, c2;                 // inertia, cognitive, social
  double min_pos, max_pos, min_v, max_v;
  uint64_t ld;                      // padded leading dimension (particles per axis row)
  uint32_t n;                       // particles in this swarm / shard
  uint32_t d;                       // dims
  uint32_t base;                    // global index of local particle 0 (multi-GPU shards)
  uint32_t gs;                      // group_size for the classic engines
  uint32_t k0[10], k1[10];          // Philox key schedule (seed-only, precomputed on host)
  // c1 * 2^-53 and c2 * 2^-53 (exact power-of-two scalings; scaled_ok when no
  // underflow): c1 * r1 == c1s * b1 bit for bit where r1 = b1 * 2^-53, so the
  // register-resident kernels skip the two scaling multiplies per particle-axis
  double c1s, c2s;
  uint32_t scaled_ok;
};

// Axis-major SoA state, row stride ld (flat index = axis*ld + i).
struct KState {
  double* pos;
  double* vel;
  double* pb;    // pbest positions
  double* pbf;   // pbest fitness
};

// ---------------------------------------------------------------- RNG
__device__ __forceinline__ void philox10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                         const KParams& P) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ P.k0[r];
    const uint32_t n2 = hi0 ^ c3 ^ P.k1[r];
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
}

// uniform01(key, {t, i, axis, slot}) = ((w0<<32 | w1) >> 11) * 2^-53, exact.
__device__ __forceinline__ double uniform01(const KParams& P, uint32_t t, uint32_t i, uint32_t axis,
                                            uint32_t slot) {
  uint32_t c0 = t, c1 = i, c2 = axis, c3 = slot;
  philox10(c0, c1, c2, c3, P);
  const uint64_t bits53 = (static_cast<uint64_t>(c0) << 21) | (c1 >> 11);
  return __dmul_rn(__ull2double_rn(bits53), 0x1.0p-53);
}

// The 53-bit integer behind uniform01 as a double (exact: < 2^53): uniform01 ==
// uniform53 * 2^-53 exactly.
__device__ __forceinline__ double uniform53(const KParams& P, uint32_t t, uint32_t i, uint32_t axis,
                                            uint32_t slot) {
  uint32_t c0 = t, c1 = i, c2 = axis, c3 = slot;
  philox10(c0, c1, c2, c3, P);
  return __ull2double_rn((static_cast<uint64_t>(c0) << 21) | (c1 >> 11));
}

// ---------------------------------------------------------- kinematics
// std::clamp(v, lo, hi): v < lo ? lo : (hi < v ? hi : v)  -- keeps -0.0 and NaN as the CPU does
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}

// ((w*v) + ((c1*r1)*(pb-x))) + ((c2*r2)*(g-x)), saturated (swarm.hpp:67-72)
__device__ __forceinline__ double vel_step(const KParams& P, double v, double x, double pb, double g,
                                           double r1, double r2) {
  const double a = __dmul_rn(P.w, v);
  const double b = __dmul_rn(__dmul_rn(P.c1, r1), __dsub_rn(pb, x));
  const double c = __dmul_rn(__dmul_rn(P.c2, r2), __dsub_rn(g, x));
  return clampd(__dadd_rn(__dadd_rn(a, b), c), P.min_v, P.max_v);
}

// vel_step with the draws as 53-bit integers (uniform53) and c1s / c2s:
// (c1s * b1) == (c1 * r1) exactly, so the result is vel_step's bit for bit.
__device__ __forceinline__ double vel_step53(const KParams& P, double v, double x, double pb, double g,
                                             double b1, double b2) {
  const double a = __dmul_rn(P.w, v);
  const double b = __dmul_rn(__dmul_rn(P.c1s, b1), __dsub_rn(pb, x));
  const double c = __dmul_rn(__dmul_rn(P.c2s, b2), __dsub_rn(g, x));
  return clampd(__dadd_rn(__dadd_rn(a, b), c), P.min_v, P.max_v);
}

__device__ __forceinline__ double pos_step(const KParams& P, double x, double v) {
  return clampd(__dadd_rn(x, v), P.min_pos, P.max_pos);
}

// ------------------------------------------------------------- cos
// cos(p) for the griewank / rastrigin terms (|p| <= 600 in the registered
// boxes), ONE polynomial per call: reduce by pi -- k = rint(p / pi), r = p - k*pi
// by a 3-part Cody-Waite with FMA (exact for |k| < 2^20) -- then
// cos(p) = (-1)^k cos(r) with |r| <= pi/2, and cos(r) = P(r^2), P the degree-8
// Chebyshev-node interpolant of cos(sqrt z) on [0, (pi/2)^2] (max error 4e-18,
// fitted in 80-bit long double by tools/cos_poly_fit.py). 14 FP64
// instructions and no quadrant select, where fdlibm-style sin+cos kernels cost
// ~30 (both polynomials, then a select). Max error 3.2e-16 absolute against
// glibc over |p| <= 600 -- the same class as CUDA's own cos; the reference's
// glibc cos is not reproducible bit for bit on the GPU either way (DESIGN.md
// section 2). The FP64 constants live in the constant bank: DFMA reads a
// c[][] operand directly, whereas a 64-bit immediate costs two IMAD.MOV per use.
__constant__ double kCos[13] = {
    0x1.8p52,                  // 0: rint shifter
    0.31830988618379067154,    // 1: 1/pi
    3.14159265358979311600e+00,  // 2: pi (Cody-Waite, 3 parts)
    1.22464679914735317723e-16,  // 3
    -2.99476980971833966425e-33, // 4
    4.609001524865924e-14,     // 5: P8 .. P0 (Horner order)
    -1.1462904621323729e-11,   // 6
    2.087656196355758e-09,     // 7
    -2.755731639398695e-07,    // 8
    2.4801587277454882e-05,    // 9
    -0.001388888888877329,     // 10
    0.041666666666663896,      // 11
    -0.4999999999999997,       // 12   (P0 = 1.0)
};

__device__ __forceinline__ double cos_pso(double p) {
  const double big = kCos[0];
  const double t = __fma_rn(p, kCos[1], big);  // rint(p / pi) in the low bits
  const double k = __dsub_rn(t, big);
  const uint32_t odd = static_cast<uint32_t>(__double2loint(t)) & 1u;
  double r = __fma_rn(-k, kCos[2], p);
  r = __fma_rn(-k, kCos[3], r);
  r = __fma_rn(-k, kCos[4], r);
  const double z = __dmul_rn(r, r);
  double c = __fma_rn(z, kCos[5], kCos[6]);
#pragma unroll
  for (int j = 7; j <= 12; ++j) c = __fma_rn(c, z, kCos[j]);
  c = __fma_rn(c, z, 1.0);
  // (-1)^k: flip the sign bit (an integer op on the high word, no select)
  return __hiloint2double(__double2hiint(c) ^ static_cast<int>(odd << 31), __double2loint(c));
}

// fitness constants that are not 32-bit-immediate encodable (see kCos)
__constant__ double kFitK[2] = {0.8, 6.283185307179586};

// ------------------------------------------------------------- fitness
// Accumulators fed one axis at a time in ascending order (fitness.hpp:26-27).
// add(v, axis) == accum(term(v, axis), v, axis) bit for bit: term() is the
// per-axis work that does not depend on the running sum (the expensive cos of
// griewank/rastrigin), accum() the strictly ordered fold. Split kernels compute
// terms of different axes in different lanes and pass the accumulator along
// (shfl_up) so the fold keeps the reference's order.
enum FitId : int { kCubic = 0, kSphere = 1, kRosenbrock = 2, kGriewank = 3, kRastrigin = 4 };

template <int F>
struct Fit;

template <>
struct Fit<kCubic> {  // fitness.hpp:47-54
  double acc = 0.0;
  using Term = double;
  __device__ __forceinline__ static Term term(double v, uint32_t) {
    return __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(__dsub_rn(v, kFitK[0]), v), 1000.0), v), 8000.0);
  }
  __device__ __forceinline__ void accum(Term t, double, uint32_t) { acc = __dadd_rn(acc, t); }
  __device__ __forceinline__ void add(double v, uint32_t a) { accum(term(v, a), v, a); }
  // axis 0 of a fresh accumulator: 0.0 + t == t bit for bit unless t is -0.0,
  // and the term's last operation (+ 8000) cannot round to -0.0
  __device__ __forceinline__ void add_first(double v) { acc = term(v, 0); }
  __device__ __forceinline__ double value() const { return acc; }
  __device__ __forceinline__ void shfl_up(unsigned m, int w) { acc = __shfl_up_sync(m, acc, 1, w); }
};

template <>
struct Fit<kSphere> {  // fitness.hpp:57-61
  double acc = 0.0;
  using Term = double;
  __device__ __forceinline__ static Term term(double v, uint32_t) { return __dmul_rn(v, v); }
  __device__ __forceinline__ void accum(Term t, double, uint32_t) { acc = __dadd_rn(acc, t); }
  __device__ __forceinline__ void add(double v, uint32_t a) { accum(term(v, a), v, a); }
  __device__ __forceinline__ void add_first(double v) { acc = term(v, 0); }  // v*v is never -0.0
  __device__ __forceinline__ double value() const { return -acc; }
  __device__ __forceinline__ void shfl_up(unsigned m, int w) { acc = __shfl_up_sync(m, acc, 1, w); }
};

template <>
struct Fit<kRosenbrock> {  // fitness.hpp:65-73: pairs (x_d, x_{d+1}) in ascending d
  double acc = 0.0;
  double prev = 0.0;
  struct Term {};
  __device__ __forceinline__ static Term term(double, uint32_t) { return {}; }
  __device__ __forceinline__ void accum(Term, double v, uint32_t axis) {
    if (axis > 0) {
      const double a = __dsub_rn(v, __dmul_rn(prev, prev));
      const double b = __dsub_rn(1.0, prev);
      acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(__dmul_rn(100.0, a), a), __dmul_rn(b, b)));
    }
    prev = v;
  }
  __device__ __forceinline__ void add(double v, uint32_t a) { accum(term(v, a), v, a); }
  __device__ __forceinline__ void add_first(double v) { prev = v; }
  __device__ __forceinline__ double value() const { return -acc; }
  __device__ __forceinline__ void shfl_up(unsigned m, int w) {
    acc = __shfl_up_sync(m, acc, 1, w);
    prev = __shfl_up_sync(m, prev, 1, w);
  }
};

template <>
struct Fit<kGriewank> {  // fitness.hpp:77-85 (cos_pso: <= 2 ulp from glibc)
  double sum = 0.0;
  double prod = 1.0;
  struct Term {
    double s, c;
  };
  __device__ __forceinline__ static Term term(double v, uint32_t axis) {
    return {__ddiv_rn(__dmul_rn(v, v), 4000.0), cos_pso(__ddiv_rn(v, __dsqrt_rn(static_cast<double>(axis + 1))))};
  }
  __device__ __forceinline__ void accum(Term t, double, uint32_t) {
    sum = __dadd_rn(sum, t.s);
    prod = __dmul_rn(prod, t.c);
  }
  __device__ __forceinline__ void add(double v, uint32_t a) { accum(term(v, a), v, a); }
  // 0.0 + v*v/4000 (never -0.0) and 1.0 * c are exact identities
  __device__ __forceinline__ void add_first(double v) {
    const Term t = term(v, 0);
    sum = t.s;
    prod = t.c;
  }
  __device__ __forceinline__ double value() const { return -__dsub_rn(__dadd_rn(1.0, sum), prod); }
  __device__ __forceinline__ void shfl_up(unsigned m, int w) {
    sum = __shfl_up_sync(m, sum, 1, w);
    prod = __shfl_up_sync(m, prod, 1, w);
  }
};

template <>
struct Fit<kRastrigin> {  // harness fitness_fn (oracle/pso_oracle.c:rastrigin)
  double acc = 0.0;
  using Term = double;
  __device__ __forceinline__ static Term term(double v, uint32_t) {
    return __dadd_rn(__dsub_rn(__dmul_rn(v, v), __dmul_rn(10.0, cos_pso(__dmul_rn(kFitK[1], v)))), 10.0);
  }
  __device__ __forceinline__ void accum(Term t, double, uint32_t) { acc = __dadd_rn(acc, t); }
  __device__ __forceinline__ void add(double v, uint32_t a) { accum(term(v, a), v, a); }
  __device__ __forceinline__ void add_first(double v) { acc = term(v, 0); }  // (...) + 10 is never -0.0
  __device__ __forceinline__ double value() const { return -acc; }
  __device__ __forceinline__ void shfl_up(unsigned m, int w) { acc = __shfl_up_sync(m, acc, 1, w); }
};

// ------------------------------------------------------ (fit, idx) order
// engine.hpp:38-41: fitness descending, ties to the lower particle index.
__device__ __forceinline__ bool beats(double f, uint32_t i, double F, uint32_t I) {
  return f > F || (f == F && i < I);
}

// Butterfly argmax over a full warp; every lane ends with the winner.
__device__ __forceinline__ void warp_argmax(double& f, uint32_t& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double of = __shfl_xor_sync(0xffffffffu, f, off);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (beats(of, oi, f, i)) {
      f = of;
      i = oi;
    }
  }
}

__device__ __forceinline__ void warp_argmax3(double& f, uint32_t& i, uint32_t& s) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double of = __shfl_xor_sync(0xffffffffu, f, off);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, i, off);
    const uint32_t os = __shfl_xor_sync(0xffffffffu, s, off);
    if (beats(of, oi, f, i)) {
      f = of;
      i = oi;
      s = os;
    }
  }
}

// --------------------------------------------------- one particle's step
// advance_particle (swarm.hpp:115-131) for one particle, scalar accesses.
// Returns the new fitness; updates pbest in place on strict improvement.
template <int F>
__device__ __forceinline__ double advance_one(const KParams& P, const KState& S, uint32_t t,
                                              uint32_t li, const double* __restrict__ gpos) {
  const uint32_t gi = P.base + li;
  Fit<F> fit;
  for (uint32_t a = 0; a < P.d; ++a) {
    const size_t at = static_cast<size_t>(a) * P.ld + li;
    const double r1 = uniform01(P, t, gi, a, 0);
    const double r2 = uniform01(P, t, gi, a, 1);
    const double x = S.pos[at];
    const double v = vel_step(P, S.vel[at], x, S.pb[at], gpos[a], r1, r2);
    const double nx = pos_step(P, x, v);
    S.vel[at] = v;
    S.pos[at] = nx;
    fit.add(nx, a);
  }
  const double f = fit.value();
  if (f > S.pbf[li]) {  // update_pbest, strict > (swarm.hpp:100-108)
    S.pbf[li] = f;
    for (uint32_t a = 0; a < P.d; ++a) {
      const size_t at = static_cast<size_t>(a) * P.ld + li;
      S.pb[at] = S.pos[at];
    }
  }
  return f;
}

// Fitness of particle li's current position (for state export / init).
template <int F>
__device__ __forceinline__ double eval_position(const KParams& P, const double* __restrict__ pos,
                                                uint32_t li) {
  Fit<F> fit;
  for (uint32_t a = 0; a < P.d; ++a) fit.add(pos[static_cast<size_t>(a) * P.ld + li], a);
  return fit.value();
}

}  // namespace cupso
