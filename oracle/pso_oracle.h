/*
 * pso_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU solver (psokit, header-only C++20
 * under /root/reference/proj/include/psokit) for the per-iteration PSO step.
 * It is the *checker* for the CUDA path: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. The product library
 * (libcupso.so) never links or calls anything in oracle/.
 *
 * Parity of this restatement is pinned two ways (see tests/test_oracle.py):
 *   1. the reference's own known-answer vectors (Philox KATs test_rng.cpp:18-23,
 *      fitness pins test_fitness.cpp:15-23, kinematics pins test_swarm.cpp:102-141),
 *   2. bitwise comparison against the reference itself, compiled unmodified
 *      from /root/reference by oracle/Makefile into oracle/_ref/ (ref_shim.cpp),
 *      and the golden fixtures under tests/golden/ generated from it.
 */
#ifndef PSO_ORACLE_H
#define PSO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field order and meaning as psokit::pso_params (params.hpp:14-25) and
 * cupso_params (include/cupso.h). */
typedef struct orc_params {
  double inertia, cognitive, social;
  double min_pos, max_pos, min_v, max_v;
  uint32_t particle_cnt, dims, max_iter, group_size;
} orc_params;

/* fitness ids, identical to cupso_fitness_id() numbering */
enum { ORC_CUBIC = 0, ORC_SPHERE = 1, ORC_ROSENBROCK = 2, ORC_GRIEWANK = 3, ORC_RASTRIGIN = 4 };

typedef struct orc_state {
  uint32_t particle_cnt, dims;
  double* positions;  /* particle_cnt*dims, axis-major (swarm.hpp:21-24) */
  double* velocities;
  double* fitness;    /* particle_cnt */
  double* pbest_pos;
  double* pbest_fit;
} orc_state;

typedef struct orc_result {
  double gbest_fit;
  uint32_t gbest_particle;
  double initial_gbest_fit;
  uint32_t initial_gbest_particle;
  double* gbest_pos;        /* [dims], caller-owned */
  double* trace;            /* [max_iter], caller-owned */
  uint32_t* trace_particle; /* [max_iter], caller-owned, may be NULL */
  double compute_seconds;
} orc_result;

typedef void (*orc_observer)(uint32_t iteration, const orc_state* s, double gb_fit,
                             uint32_t gb_particle, const double* gb_pos, void* user);

void orc_philox4x32(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]);
double orc_uniform01(uint64_t seed, uint32_t iteration, uint32_t particle, uint32_t axis,
                     uint32_t slot);
/* returns 0, or -1 when lo > hi (reference throws invalid_argument) */
int orc_uniform_range(uint64_t seed, uint32_t iteration, uint32_t particle, uint32_t axis,
                      uint32_t slot, double lo, double hi, double* out);

int orc_fitness_id(const char* name);
int orc_fitness_box(int fid, double* lo, double* hi);
double orc_fitness_eval(int fid, const double* x, size_t n, size_t stride);

double orc_velocity_step(double v, double x, double pbest_x, double gbest_x,
                         const orc_params* p, double r1, double r2);
double orc_position_step(double x, double v, const orc_params* p);

/* 0 = valid; else writes the reference's message ("pso_params: ...") */
int orc_validate(const orc_params* p, char* msg, size_t cap);
int orc_make_params(int fid, uint32_t particle_cnt, uint32_t dims, uint32_t max_iter,
                    uint32_t group_size, orc_params* out, char* msg, size_t cap);

/* init_swarm: state arrays caller-allocated */
void orc_init_swarm(const orc_params* p, uint64_t seed, int fid, orc_state* s,
                    double* gb_fit, uint32_t* gb_particle, double* gb_pos);

/* run_serial (engine_serial.hpp:13-44). final_state may be NULL. */
int orc_run_serial(const orc_params* p, int fid, uint64_t seed, orc_result* r,
                   orc_state* final_state, orc_observer obs, void* user);

/* TEST ONLY: one iteration of particles [first, first+count), shard candidate out */
int orc_shard_step(const orc_params* p, int fid, uint64_t seed, uint32_t t, orc_state* s,
                   uint32_t first, uint32_t count, const double* snap_pos, double snap_fit,
                   double* best_fit, uint32_t* best_idx, double* best_pos, uint32_t* admitted);

/* bench.hpp:31-44 FNV-1a over trace bits; writes 16 hex digits + NUL */
void orc_trace_checksum(const double* trace, size_t n, char out[17]);
/* bench.hpp:20-28; returns NaN when n < 3 (reference throws) */
double orc_trimmed_mean(const double* xs, size_t n);

#ifdef __cplusplus
}
#endif
#endif
