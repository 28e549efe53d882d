/*
 * pso_oracle.c -- TEST INFRASTRUCTURE ONLY (see pso_oracle.h).
 *
 * CPU restatement of the reference's serial PSO path. Compile with
 * -ffp-contract=off (as the reference does, proj/CMakeLists.txt:17-20):
 * every floating-point expression below keeps the reference's evaluation
 * order so results are bit-identical to psokit::run_serial.
 */
#include "pso_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* rng.hpp:36-49 -- Philox-4x32-10 keyed counter permutation */
void orc_philox4x32(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = 0xD2511F53ull * (uint64_t)c0;
    const uint64_t p1 = 0xCD9E8D57ull * (uint64_t)c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.hpp:56-62 -- top 53 bits of (w0<<32 | w1) times 2^-53 */
double orc_uniform01(uint64_t seed, uint32_t iteration, uint32_t particle, uint32_t axis,
                     uint32_t slot) {
  const uint32_t ctr[4] = {iteration, particle, axis, slot};
  uint32_t w[4];
  orc_philox4x32(ctr, (uint32_t)seed, (uint32_t)(seed >> 32), w);
  const uint64_t bits = ((uint64_t)w[0] << 32) | w[1];
  return (double)(bits >> 11) * 0x1.0p-53;
}

/* rng.hpp:65-68 */
int orc_uniform_range(uint64_t seed, uint32_t iteration, uint32_t particle, uint32_t axis,
                      uint32_t slot, double lo, double hi, double* out) {
  if (lo > hi) return -1;
  *out = lo + orc_uniform01(seed, iteration, particle, axis, slot) * (hi - lo);
  return 0;
}

/* ---- fitness.hpp:47-85 (+ the harness Rastrigin) ---- */

static double cubic(const double* x, size_t n, size_t stride) {
  double acc = 0.0;
  for (size_t d = 0; d < n; ++d) {
    const double v = x[d * stride];
    acc += ((v - 0.8) * v - 1000.0) * v + 8000.0;
  }
  return acc;
}

static double sphere(const double* x, size_t n, size_t stride) {
  double acc = 0.0;
  for (size_t d = 0; d < n; ++d) acc += x[d * stride] * x[d * stride];
  return -acc;
}

static double rosenbrock(const double* x, size_t n, size_t stride) {
  double acc = 0.0;
  for (size_t d = 0; d + 1 < n; ++d) {
    const double a = x[(d + 1) * stride] - x[d * stride] * x[d * stride];
    const double b = 1.0 - x[d * stride];
    acc += 100.0 * a * a + b * b;
  }
  return -acc;
}

static double griewank(const double* x, size_t n, size_t stride) {
  double sum = 0.0;
  double prod = 1.0;
  for (size_t d = 0; d < n; ++d) {
    sum += x[d * stride] * x[d * stride] / 4000.0;
    prod *= cos(x[d * stride] / sqrt((double)(d + 1)));
  }
  return -(1.0 + sum - prod);
}

/* Rastrigin is not in the reference registry (fitness.hpp:87-95); the harness
 * supplies it as a fitness_fn{"rastrigin", -5.12, 5.12, eval} (oracle/ref_shim.cpp
 * builds the identical lambda). Negated for maximisation, ascending axis order. */
#define ORC_TWO_PI 6.283185307179586
static double rastrigin(const double* x, size_t n, size_t stride) {
  double acc = 0.0;
  for (size_t d = 0; d < n; ++d) {
    const double v = x[d * stride];
    acc += v * v - 10.0 * cos(ORC_TWO_PI * v) + 10.0;
  }
  return -acc;
}

static const char* const kNames[] = {"cubic", "sphere", "rosenbrock", "griewank", "rastrigin"};
static const double kLo[] = {-100.0, -100.0, -2.048, -600.0, -5.12};
static const double kHi[] = {100.0, 100.0, 2.048, 600.0, 5.12};

int orc_fitness_id(const char* name) {
  for (int i = 0; i < 5; ++i)
    if (strcmp(name, kNames[i]) == 0) return i;
  return -1;
}

int orc_fitness_box(int fid, double* lo, double* hi) {
  if (fid < 0 || fid > 4) return -1;
  *lo = kLo[fid];
  *hi = kHi[fid];
  return 0;
}

double orc_fitness_eval(int fid, const double* x, size_t n, size_t stride) {
  switch (fid) {
    case ORC_CUBIC: return cubic(x, n, stride);
    case ORC_SPHERE: return sphere(x, n, stride);
    case ORC_ROSENBROCK: return rosenbrock(x, n, stride);
    case ORC_GRIEWANK: return griewank(x, n, stride);
    case ORC_RASTRIGIN: return rastrigin(x, n, stride);
    default: return NAN;
  }
}

/* swarm.hpp:56-62: std::clamp(v, lo, hi) == v < lo ? lo : (hi < v ? hi : v) */
static inline double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}

/* swarm.hpp:67-72 */
double orc_velocity_step(double v, double x, double pbest_x, double gbest_x,
                         const orc_params* p, double r1, double r2) {
  const double next =
      p->inertia * v + p->cognitive * r1 * (pbest_x - x) + p->social * r2 * (gbest_x - x);
  return clampd(next, p->min_v, p->max_v);
}

/* swarm.hpp:75-77 */
double orc_position_step(double x, double v, const orc_params* p) {
  return clampd(x + v, p->min_pos, p->max_pos);
}

/* params.hpp:33-47: same checks, same order, same message text */
int orc_validate(const orc_params* p, char* msg, size_t cap) {
  char buf[256];
  buf[0] = 0;
  if (!(p->min_pos < p->max_pos))
    snprintf(buf, sizeof buf, "pso_params: min_pos (%f) must be < max_pos (%f)", p->min_pos,
             p->max_pos);
  else if (!(p->min_v <= p->max_v))
    snprintf(buf, sizeof buf, "pso_params: min_v (%f) must be <= max_v (%f)", p->min_v,
             p->max_v);
  else if (p->particle_cnt < 1)
    snprintf(buf, sizeof buf, "pso_params: particle_cnt must be >= 1");
  else if (p->dims < 1)
    snprintf(buf, sizeof buf, "pso_params: dims must be >= 1");
  else if (p->max_iter < 1)
    snprintf(buf, sizeof buf, "pso_params: max_iter must be >= 1");
  else if (p->group_size < 1)
    snprintf(buf, sizeof buf, "pso_params: group_size must be >= 1");
  if (!buf[0]) return 0;
  if (msg && cap) {
    strncpy(msg, buf, cap - 1);
    msg[cap - 1] = 0;
  }
  return -1;
}

/* params.hpp:52-66 */
int orc_make_params(int fid, uint32_t particle_cnt, uint32_t dims, uint32_t max_iter,
                    uint32_t group_size, orc_params* p, char* msg, size_t cap) {
  double lo, hi;
  if (orc_fitness_box(fid, &lo, &hi) != 0) return -2;
  p->inertia = 1.0;
  p->cognitive = 2.0;
  p->social = 2.0;
  p->min_pos = lo;
  p->max_pos = hi;
  p->max_v = (hi - lo) / 2.0;
  p->min_v = -p->max_v;
  p->particle_cnt = particle_cnt;
  p->dims = dims;
  p->max_iter = max_iter;
  p->group_size = group_size;
  return orc_validate(p, msg, cap);
}

static inline size_t soa(uint32_t i, uint32_t d, uint32_t n) { return (size_t)d * n + i; }

/* swarm.hpp:136-171 */
void orc_init_swarm(const orc_params* p, uint64_t seed, int fid, orc_state* s,
                    double* gb_fit, uint32_t* gb_particle, double* gb_pos) {
  const uint32_t n = p->particle_cnt;
  s->particle_cnt = n;
  s->dims = p->dims;
  for (uint32_t d = 0; d < p->dims; ++d) {
    for (uint32_t i = 0; i < n; ++i) {
      const size_t at = soa(i, d, n);
      orc_uniform_range(seed, 0, i, d, 2, p->min_pos, p->max_pos, &s->positions[at]);
      orc_uniform_range(seed, 0, i, d, 3, p->min_v, p->max_v, &s->velocities[at]);
    }
  }
  memcpy(s->pbest_pos, s->positions, sizeof(double) * (size_t)n * p->dims);
  for (uint32_t i = 0; i < n; ++i) {
    s->fitness[i] = orc_fitness_eval(fid, s->positions + i, p->dims, n);
    s->pbest_fit[i] = s->fitness[i];
  }
  *gb_fit = -INFINITY;
  *gb_particle = 0xffffffffu;
  for (uint32_t d = 0; d < p->dims; ++d) gb_pos[d] = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    if (s->pbest_fit[i] > *gb_fit) {
      *gb_fit = s->pbest_fit[i];
      *gb_particle = i;
      for (uint32_t d = 0; d < p->dims; ++d) gb_pos[d] = s->pbest_pos[soa(i, d, n)];
    }
  }
}

/* swarm.hpp:115-131 (velocity, position, fitness, pbest in one particle pass) */
static double advance_particle(orc_state* s, const orc_params* p, int fid, uint64_t seed,
                               uint32_t iteration, uint32_t i, const double* gbest_pos) {
  const uint32_t n = s->particle_cnt;
  for (uint32_t d = 0; d < s->dims; ++d) {
    const size_t at = soa(i, d, n);
    const double r1 = orc_uniform01(seed, iteration, i, d, 0);
    const double r2 = orc_uniform01(seed, iteration, i, d, 1);
    const double v = orc_velocity_step(s->velocities[at], s->positions[at], s->pbest_pos[at],
                                       gbest_pos[d], p, r1, r2);
    s->velocities[at] = v;
    s->positions[at] = orc_position_step(s->positions[at], v, p);
  }
  const double fit = orc_fitness_eval(fid, s->positions + i, s->dims, n);
  s->fitness[i] = fit;
  if (fit > s->pbest_fit[i]) { /* update_pbest, swarm.hpp:100-108 (strict >) */
    s->pbest_fit[i] = fit;
    for (uint32_t d = 0; d < s->dims; ++d) s->pbest_pos[soa(i, d, n)] = s->positions[soa(i, d, n)];
  }
  return fit;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* engine_serial.hpp:13-44 */
int orc_run_serial(const orc_params* p, int fid, uint64_t seed, orc_result* r,
                   orc_state* final_state, orc_observer obs, void* user) {
  if (orc_validate(p, NULL, 0) != 0) return -1;
  if (fid < 0 || fid > 4) return -2;
  const uint32_t n = p->particle_cnt, dims = p->dims;
  const size_t cells = (size_t)n * dims;
  orc_state s;
  s.particle_cnt = n;
  s.dims = dims;
  s.positions = (double*)malloc(sizeof(double) * cells);
  s.velocities = (double*)malloc(sizeof(double) * cells);
  s.pbest_pos = (double*)malloc(sizeof(double) * cells);
  s.fitness = (double*)malloc(sizeof(double) * n);
  s.pbest_fit = (double*)malloc(sizeof(double) * n);
  double* gb_pos = (double*)malloc(sizeof(double) * dims);
  double* snap_pos = (double*)malloc(sizeof(double) * dims);
  double gb_fit;
  uint32_t gb_particle;
  orc_init_swarm(p, seed, fid, &s, &gb_fit, &gb_particle, gb_pos);
  r->initial_gbest_fit = gb_fit;
  r->initial_gbest_particle = gb_particle;

  const double t0 = now_seconds();
  for (uint32_t t = 0; t < p->max_iter; ++t) {
    memcpy(snap_pos, gb_pos, sizeof(double) * dims);
    for (uint32_t i = 0; i < n; ++i) {
      advance_particle(&s, p, fid, seed, t, i, snap_pos);
      if (s.pbest_fit[i] > gb_fit) {
        gb_fit = s.pbest_fit[i];
        gb_particle = i;
        for (uint32_t d = 0; d < dims; ++d) gb_pos[d] = s.pbest_pos[soa(i, d, n)];
      }
    }
    r->trace[t] = gb_fit;
    if (r->trace_particle) r->trace_particle[t] = gb_particle;
    if (obs) obs(t, &s, gb_fit, gb_particle, gb_pos, user);
  }
  r->compute_seconds = now_seconds() - t0;
  r->gbest_fit = gb_fit;
  r->gbest_particle = gb_particle;
  memcpy(r->gbest_pos, gb_pos, sizeof(double) * dims);
  if (final_state) {
    memcpy(final_state->positions, s.positions, sizeof(double) * cells);
    memcpy(final_state->velocities, s.velocities, sizeof(double) * cells);
    memcpy(final_state->pbest_pos, s.pbest_pos, sizeof(double) * cells);
    memcpy(final_state->fitness, s.fitness, sizeof(double) * n);
    memcpy(final_state->pbest_fit, s.pbest_fit, sizeof(double) * n);
  }
  free(s.positions); free(s.velocities); free(s.pbest_pos); free(s.fitness); free(s.pbest_fit);
  free(gb_pos); free(snap_pos);
  return 0;
}

/* TEST ONLY -- one iteration of the particles [first, first+count) of a
 * full-size state, returning the shard's best candidate that passes the
 * snapshot filter (engine_queue.hpp:44,91) in beats() order (engine.hpp:38-41).
 * Lets the 2-rank gloo test replay the multi-GPU exchange protocol on CPU. */
int orc_shard_step(const orc_params* p, int fid, uint64_t seed, uint32_t t, orc_state* s,
                   uint32_t first, uint32_t count, const double* snap_pos, double snap_fit,
                   double* best_fit, uint32_t* best_idx, double* best_pos, uint32_t* admitted) {
  double bf = -INFINITY;
  uint32_t bi = 0xffffffffu;
  uint32_t adm = 0;
  for (uint32_t i = first; i < first + count; ++i) {
    const double fit = advance_particle(s, p, fid, seed, t, i, snap_pos);
    if (fit > snap_fit) {
      ++adm;
      if (fit > bf || (fit == bf && i < bi)) {
        bf = fit;
        bi = i;
      }
    }
  }
  *best_fit = bf;
  *best_idx = bi;
  *admitted = adm;
  for (uint32_t d = 0; d < s->dims; ++d)
    best_pos[d] = bi == 0xffffffffu ? 0.0 : s->positions[soa(bi, d, s->particle_cnt)];
  return 0;
}

/* bench.hpp:31-44 */
void orc_trace_checksum(const double* trace, size_t n, char out[17]) {
  uint64_t h = 1469598103934665603ull;
  for (size_t k = 0; k < n; ++k) {
    uint64_t bits;
    memcpy(&bits, &trace[k], 8);
    for (int b = 0; b < 8; ++b) {
      h ^= bits & 0xffu;
      h *= 1099511628211ull;
      bits >>= 8;
    }
  }
  snprintf(out, 17, "%016llx", (unsigned long long)h);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* bench.hpp:20-28 */
double orc_trimmed_mean(const double* xs, size_t n) {
  if (n < 3) return NAN;
  double* sorted = (double*)malloc(sizeof(double) * n);
  memcpy(sorted, xs, sizeof(double) * n);
  qsort(sorted, n, sizeof(double), cmp_double);
  double sum = 0.0;
  for (size_t i = 1; i + 1 < n; ++i) sum += sorted[i];
  free(sorted);
  return sum / (double)(n - 2);
}
