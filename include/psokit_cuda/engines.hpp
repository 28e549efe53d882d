// psokit_cuda/engines.hpp -- drop-in psokit engines backed by libcupso.so.
//
// Header-only C++20 adapter between the reference's plugin API and the C-ABI
// in include/cupso.h. Include it after the reference headers:
//
//   #include "psokit/psokit.hpp"          // the reference (engines.hpp:12-48)
//   #include "psokit_cuda/engines.hpp"    // this file
//
//   const auto& e = psokit_cuda::find_engine("cuda-sync");   // or any psokit name
//   psokit::run_result r = e.run(params, fitness, psokit::rng_key{1}, {}, {});
//
// and link with -lcupso. Every entry is a psokit::engine_entry
// {name, parallel, run} (engines.hpp:15-19) whose run has the exact engine_fn
// signature (engines.hpp:12-13), so run_bench-style drivers, the acceptance
// checks and the CLI can take them unchanged. Errors surface as the
// reference's exception types (cupso_status -> invalid_argument /
// runtime_error / logic_error / domain_error). There is no CPU fallback.
//
// Fitness functions cross the boundary by name (fitness.hpp:87-95 plus the
// harness "rastrigin"); a fitness_fn whose name/box is not a device fitness
// -- e.g. a test-only lambda -- throws std::invalid_argument.
// exec_options.threads / schedule_jitter have no GPU meaning; the device is
// chosen with CUPSO_DEVICE (default 0).
#pragma once

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "cupso.h"

namespace psokit_cuda {

inline void check(cupso_status st) {
  if (st == CUPSO_OK) return;
  const std::string msg = cupso_last_error();
  switch (st) {
    case CUPSO_EINVAL: throw std::invalid_argument(msg);
    case CUPSO_ELOGIC: throw std::logic_error(msg);
    case CUPSO_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline cupso_params to_c(const psokit::pso_params& p) {
  cupso_params c{};
  c.inertia = p.inertia;
  c.cognitive = p.cognitive;
  c.social = p.social;
  c.min_pos = p.min_pos;
  c.max_pos = p.max_pos;
  c.min_v = p.min_v;
  c.max_v = p.max_v;
  c.particle_cnt = p.particle_cnt;
  c.dims = p.dims;
  c.max_iter = p.max_iter;
  c.group_size = p.group_size;
  return c;
}

inline int fitness_id(const psokit::fitness_fn& f) {
  const int id = cupso_fitness_id(f.name.c_str());
  double lo = 0.0, hi = 0.0;
  if (id < 0 || cupso_fitness_box(id, &lo, &hi) != CUPSO_OK || lo != f.lo || hi != f.hi)
    throw std::invalid_argument("fitness '" + f.name +
                                "' has no device implementation (custom fitness_fn lambdas cannot "
                                "run on the GPU); known: cubic sphere rosenbrock griewank rastrigin");
  return id;
}

inline int device_from_env() {
  const char* e = std::getenv("CUPSO_DEVICE");
  return e ? std::atoi(e) : 0;
}

namespace detail {

struct observer_ctx {
  const psokit::iteration_observer* obs;
  std::exception_ptr error;
};

inline void observer_trampoline(uint32_t t, const cupso_state_view* v, void* user) {
  auto* ctx = static_cast<observer_ctx*>(user);
  if (ctx->error) return;
  try {
    const std::size_t n = v->particle_cnt, cells = n * v->dims;
    psokit::swarm_state s;
    s.particle_cnt = v->particle_cnt;
    s.dims = v->dims;
    s.positions.assign(v->positions, v->positions + cells);
    s.velocities.assign(v->velocities, v->velocities + cells);
    s.fitness.assign(v->fitness, v->fitness + n);
    s.pbest_pos.assign(v->pbest_pos, v->pbest_pos + cells);
    s.pbest_fit.assign(v->pbest_fit, v->pbest_fit + n);
    psokit::global_best gb;
    gb.fit = v->gbest_fit;
    gb.particle = v->gbest_particle;
    gb.pos.assign(v->gbest_pos, v->gbest_pos + v->dims);
    (*ctx->obs)(t, s, gb);
  } catch (...) {
    ctx->error = std::current_exception();
  }
}

}  // namespace detail

// The engine_fn body: one full run (init_swarm + max_iter iterations) on the GPU.
inline psokit::run_result run(const psokit::pso_params& p, const psokit::fitness_fn& f,
                              psokit::rng_key key, int variant,
                              const psokit::iteration_observer& observe = {}) {
  p.validate();  // the reference's own messages (params.hpp:33-47)
  const cupso_params c = to_c(p);
  const int fid = fitness_id(f);
  psokit::run_result r;
  r.gbest_pos.resize(p.dims);
  r.trace.resize(p.max_iter);
  std::vector<uint32_t> trace_particle(p.max_iter);
  std::vector<double> occupancy(p.max_iter);
  cupso_result out{};
  out.gbest_pos = r.gbest_pos.data();
  out.trace = r.trace.data();
  out.trace_particle = trace_particle.data();
  out.queue_occupancy = occupancy.data();
  detail::observer_ctx ctx{&observe, nullptr};
  const cupso_status st =
      cupso_run(&c, fid, key.seed, variant, device_from_env(),
                observe ? detail::observer_trampoline : nullptr, observe ? &ctx : nullptr, &out);
  if (ctx.error) std::rethrow_exception(ctx.error);
  check(st);
  r.gbest_fit = out.gbest_fit;
  r.gbest_particle = out.gbest_particle;
  r.initial_gbest_fit = out.initial_gbest_fit;
  r.compute_seconds = out.compute_seconds;  // device time of the iteration loop
  if (out.has_occupancy) r.queue_occupancy = std::move(occupancy);
  return r;
}

// engines.hpp:21-40 for the GPU. The asynchronous engine is not bitwise
// reproducible, so it is not a `parallel` entry (acceptance.cpp:57-58 checks
// every parallel entry bit for bit against serial).
inline const std::vector<psokit::engine_entry>& engine_registry() {
  static const std::vector<psokit::engine_entry> engines = [] {
    std::vector<psokit::engine_entry> v;
    for (int k = 0; k < cupso_variant_count(); ++k) {
      v.push_back({cupso_variant_name(k), cupso_variant_deterministic(k) != 0,
                   [k](const psokit::pso_params& p, const psokit::fitness_fn& f, psokit::rng_key key,
                       const psokit::exec_options&, const psokit::iteration_observer& obs) {
                     return run(p, f, key, k, obs);
                   }});
    }
    return v;
  }();
  return engines;
}

// engines.hpp:42-48 over the CUDA engines first, then the reference's own.
inline const psokit::engine_entry& find_engine(std::string_view name) {
  for (const auto& e : engine_registry())
    if (e.name == name) return e;
  for (const auto& e : psokit::engine_registry())
    if (e.name == name) return e;
  std::string known;
  for (const auto& e : psokit::engine_registry()) known += " " + e.name;
  for (const auto& e : engine_registry()) known += " " + e.name;
  throw std::invalid_argument("unknown engine '" + std::string(name) + "'; known:" + known);
}

}  // namespace psokit_cuda
