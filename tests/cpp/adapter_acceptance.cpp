// The reference's acceptance criteria (tests/acceptance.cpp:40-124) run
// against the CUDA engines through the drop-in adapter, with the unmodified
// reference's run_serial as the oracle. Built by tests/cpp/Makefile against
// /root/reference/proj/include; the binary travels to the GPU box.
//
//   adapter_acceptance --list     registry only (no GPU needed)
//   adapter_acceptance            all checks (needs a GPU)
#include <bit>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "psokit/psokit.hpp"
#include "psokit_cuda/engines.hpp"

namespace {

bool bits_equal(const std::vector<double>& a, const std::vector<double>& b) {
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if (std::bit_cast<std::uint64_t>(a[i]) != std::bit_cast<std::uint64_t>(b[i])) return false;
  return true;
}

int failures = 0;

void report(bool ok, const char* name, const std::string& detail) {
  std::printf("%s: %s -- %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
  std::fflush(stdout);
  if (!ok) ++failures;
}

// criterion 1 (acceptance.cpp:40-76), the reference's 5 seeds (acceptance.cpp:47)
void cross_engine_equivalence() {
  const auto& cubic = psokit::find_fitness("cubic");
  std::size_t runs = 0, bad = 0;
  std::string first;
  for (const std::uint32_t particles : {33u, 128u, 256u, 1024u})
    for (const std::uint32_t dims : {1u, 120u})
      for (const std::uint64_t seed : {11ull, 22ull, 33ull, 44ull, 55ull}) {
        const auto base = psokit::run_serial(psokit::make_params(cubic, particles, dims, 100, 128), cubic,
                                             psokit::rng_key{seed});
        for (const std::uint32_t gs : {32u, 128u}) {
          const auto p = psokit::make_params(cubic, particles, dims, 100, gs);
          for (const auto& e : psokit_cuda::engine_registry()) {
            if (!e.parallel) continue;
            const auto r = e.run(p, cubic, psokit::rng_key{seed}, {}, {});
            ++runs;
            if (!bits_equal(r.trace, base.trace) || !bits_equal(r.gbest_pos, base.gbest_pos)) {
              if (!bad++) first = e.name + " n=" + std::to_string(particles) + " d=" + std::to_string(dims);
            }
          }
        }
      }
  report(bad == 0, "cross-engine-equivalence",
         std::to_string(runs) + " CUDA engine runs vs psokit::run_serial, " + std::to_string(bad) +
             " mismatches" + (bad ? " (first: " + first + ")" : ""));
}

// criterion 2 (acceptance.cpp:79-105), every CUDA engine incl. async
void per_iteration_oracle() {
  const auto& cubic = psokit::find_fitness("cubic");
  std::size_t checked = 0, violations = 0;
  for (const auto& e : psokit_cuda::engine_registry())
    for (const std::uint32_t dims : {1u, 3u}) {
      const auto p = psokit::make_params(cubic, 256, dims, 50, 64);
      const psokit::rng_key key{101 + dims};
      psokit::swarm_state fresh;
      psokit::global_best init;
      psokit::init_swarm(p, key, cubic, fresh, init);
      double prev = init.fit;
      e.run(p, cubic, key, {}, [&](std::uint32_t, const psokit::swarm_state& s, const psokit::global_best& gb) {
        double best = psokit::fit_sentinel;
        for (std::uint32_t i = 0; i < s.particle_cnt; ++i)
          best = std::max(best, cubic.eval(s.particle_position(i)));
        if (gb.fit != std::max(prev, best)) ++violations;
        prev = gb.fit;
        ++checked;
      });
    }
  report(violations == 0, "per-iteration-oracle",
         std::to_string(checked) + " iterations, " + std::to_string(violations) + " violations");
}

// criterion 3 (acceptance.cpp:108-124)
void convergence() {
  const auto& cubic = psokit::find_fitness("cubic");
  const auto p = psokit::make_params(cubic, 1024, 1, 1000, 128);
  std::string note;
  bool ok = true;
  for (const auto& e : psokit_cuda::engine_registry()) {
    int hits = 0;
    for (std::uint64_t seed = 1; seed <= 10; ++seed)
      if (e.run(p, cubic, psokit::rng_key{seed}, {}, {}).gbest_fit >= 899999.0) ++hits;
    note += e.name + "=" + std::to_string(hits) + "/10 ";
    ok = ok && hits >= 9;
  }
  report(ok, "convergence-1d-cubic", note);
}

// error conventions (params.hpp:33-47, engines.hpp:47, fitness.hpp:102)
void errors() {
  bool ok = true;
  std::string note;
  try {
    psokit_cuda::find_engine("warpspeed");
    ok = false;
  } catch (const std::invalid_argument& e) {
    ok = ok && std::string(e.what()).find("cuda-sync") != std::string::npos;
  }
  const psokit::fitness_fn flat{"flat", -1.0, 1.0, [](psokit::strided_view) { return 1.0; }};
  try {
    psokit_cuda::find_engine("cuda-sync").run(psokit::make_params(flat, 8, 1, 2), flat, {1}, {}, {});
    ok = false;
  } catch (const std::invalid_argument&) {
  }
  psokit::pso_params bad;
  bad.particle_cnt = 0;
  try {
    psokit_cuda::find_engine("cuda-sync").run(bad, psokit::find_fitness("cubic"), {1}, {}, {});
    ok = false;
  } catch (const std::invalid_argument& e) {
    ok = ok && std::string(e.what()) == "pso_params: particle_cnt must be >= 1";
  }
  report(ok, "error-conventions", "unknown engine / custom lambda / invalid params -> std::invalid_argument");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && !std::strcmp(argv[1], "--list")) {
    for (const auto& e : psokit_cuda::engine_registry())
      std::printf("%s parallel=%d\n", e.name.c_str(), e.parallel ? 1 : 0);
    // engines from both registries resolve through find_engine
    std::printf("serial -> %s\n", psokit_cuda::find_engine("serial").name.c_str());
    try {
      const auto& cubic = psokit::find_fitness("cubic");
      psokit_cuda::find_engine("cuda-sync").run(psokit::make_params(cubic, 8, 1, 2), cubic, {1}, {}, {});
      std::printf("gpu: available\n");
    } catch (const std::runtime_error& e) {
      std::printf("gpu: %s\n", e.what());
    }
    return 0;
  }
  cross_engine_equivalence();
  per_iteration_oracle();
  convergence();
  errors();
  return failures;
}
