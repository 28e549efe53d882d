// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference solver. It is compiled
// by oracle/Makefile directly against the reference headers where they lie
// (-I/root/reference/proj/include) into oracle/_ref/libpsokit_ref.so, which is
// git-ignored and travels to the GPU box with the snapshot. Nothing of the
// reference is copied into this repo; this file only calls its public API:
//   psokit::find_engine / engine_registry (engines.hpp:21-48),
//   psokit::find_fitness / make_params (fitness.hpp:97-103, params.hpp:52-66),
//   psokit::init_swarm (swarm.hpp:136-171), detail::philox4x32 (rng.hpp:36-49).
// Rastrigin is not in the reference registry; like the survey harness it is
// injected as a fitness_fn lambda with the same expression as
// oracle/pso_oracle.c:rastrigin.
#include <cmath>
#include <cstring>
#include <string>

#include "psokit/psokit.hpp"

namespace {

thread_local std::string g_err;

const psokit::fitness_fn& lookup_fitness(const char* name) {
  static const psokit::fitness_fn rastrigin{
      "rastrigin", -5.12, 5.12, [](psokit::strided_view x) {
        double acc = 0.0;
        for (std::size_t d = 0; d < x.size; ++d) {
          const double v = x[d];
          acc += v * v - 10.0 * std::cos(6.283185307179586 * v) + 10.0;
        }
        return -acc;
      }};
  if (std::string(name) == "rastrigin") return rastrigin;
  return psokit::find_fitness(name);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_philox4x32(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  const auto w = psokit::detail::philox4x32({ctr[0], ctr[1], ctr[2], ctr[3]}, k0, k1);
  for (int i = 0; i < 4; ++i) out[i] = w[i];
}

double ref_uniform01(uint64_t seed, uint32_t it, uint32_t particle, uint32_t axis, uint32_t slot) {
  return psokit::uniform01(psokit::rng_key{seed},
                           {it, particle, axis, static_cast<psokit::draw_slot>(slot)});
}

double ref_fitness_eval(const char* name, const double* x, size_t n) {
  return lookup_fitness(name).eval(psokit::strided_view{x, n, 1});
}

// Runs one engine through its registry entry. Any output pointer may be NULL.
// trace_particle and the final state are captured with an iteration observer
// (so pass NULL for both when timing). threads: exec_options.threads (0 = all).
int ref_run(const char* engine, const char* fitness, uint32_t particles, uint32_t dims,
            uint32_t iters, uint32_t group_size, uint64_t seed, uint32_t threads,
            double* trace, uint32_t* trace_particle, double* occupancy, double* gbest_pos,
            double* gbest_fit, uint32_t* gbest_particle, double* initial_gbest_fit,
            double* compute_seconds, double* positions, double* velocities, double* fit_out,
            double* pbest_pos, double* pbest_fit) {
  try {
    const auto& e = psokit::find_engine(engine);
    const auto& f = lookup_fitness(fitness);
    const auto p = psokit::make_params(f, particles, dims, iters, group_size);
    psokit::exec_options opts;
    opts.threads = threads;
    const bool want_state = positions || velocities || fit_out || pbest_pos || pbest_fit;
    psokit::iteration_observer obs;
    if (trace_particle || want_state) {
      obs = [&](std::uint32_t t, const psokit::swarm_state& s, const psokit::global_best& gb) {
        if (trace_particle) trace_particle[t] = gb.particle;
        if (want_state && t + 1 == iters) {
          const std::size_t cells = s.positions.size();
          if (positions) std::memcpy(positions, s.positions.data(), cells * 8);
          if (velocities) std::memcpy(velocities, s.velocities.data(), cells * 8);
          if (pbest_pos) std::memcpy(pbest_pos, s.pbest_pos.data(), cells * 8);
          if (fit_out) std::memcpy(fit_out, s.fitness.data(), s.fitness.size() * 8);
          if (pbest_fit) std::memcpy(pbest_fit, s.pbest_fit.data(), s.pbest_fit.size() * 8);
        }
      };
    }
    const auto r = e.run(p, f, psokit::rng_key{seed}, opts, obs);
    if (trace) std::memcpy(trace, r.trace.data(), r.trace.size() * 8);
    if (occupancy && !r.queue_occupancy.empty())
      std::memcpy(occupancy, r.queue_occupancy.data(), r.queue_occupancy.size() * 8);
    if (gbest_pos) std::memcpy(gbest_pos, r.gbest_pos.data(), r.gbest_pos.size() * 8);
    if (gbest_fit) *gbest_fit = r.gbest_fit;
    if (gbest_particle) *gbest_particle = r.gbest_particle;
    if (initial_gbest_fit) *initial_gbest_fit = r.initial_gbest_fit;
    if (compute_seconds) *compute_seconds = r.compute_seconds;
    return 0;
  } catch (const std::invalid_argument& ex) {
    g_err = ex.what();
    return 1;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return 2;
  }
}

// Initial state exactly as init_swarm produces it (for init-kernel parity).
int ref_init(const char* fitness, uint32_t particles, uint32_t dims, uint64_t seed,
             double* positions, double* velocities, double* fit_out, double* gbest_fit,
             uint32_t* gbest_particle, double* gbest_pos) {
  try {
    const auto& f = lookup_fitness(fitness);
    const auto p = psokit::make_params(f, particles, dims, 1, 128);
    psokit::swarm_state s;
    psokit::global_best gb;
    psokit::init_swarm(p, psokit::rng_key{seed}, f, s, gb);
    std::memcpy(positions, s.positions.data(), s.positions.size() * 8);
    std::memcpy(velocities, s.velocities.data(), s.velocities.size() * 8);
    std::memcpy(fit_out, s.fitness.data(), s.fitness.size() * 8);
    *gbest_fit = gb.fit;
    *gbest_particle = gb.particle;
    std::memcpy(gbest_pos, gb.pos.data(), gb.pos.size() * 8);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return 1;
  }
}

// The reference's determinism-audited checksum (bench.hpp:31-44).
void ref_trace_checksum(const double* trace, size_t n, char out[17]) {
  const std::string s = psokit::trace_checksum(std::span<const double>(trace, n));
  std::memcpy(out, s.c_str(), 17);
}

}  // extern "C"
