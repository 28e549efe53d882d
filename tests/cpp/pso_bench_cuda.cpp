// pso_bench_cuda.cpp -- the reference's benchmark front-end protocol with the
// CUDA engines next to psokit's CPU engines, in C++ (SURVEY.md 8(f) #4).
//
// The reference CLI (tools/pso_bench.cpp:44-156) needs CLI11, which this image
// lacks; this binary takes the same flags with a small hand-written parser and
// drives the reference's own protocol pieces from psokit/bench.hpp --
// trimmed_mean / trace_checksum (:20-44), write_csv_row + csv_header (:83-94),
// read_csv (:145), render_table (:191-238), sweep_1d / sweep_120d (:247-265) --
// over psokit_cuda::find_engine, which resolves "cuda-*" names to libcupso and
// every other name to psokit's registry. So one run can time `serial` on the
// host and `cuda-sync` on the GPU and print the reference's speedup table, and
// a deterministic CUDA engine prints the same trace checksum as serial.
//
//   build/pso_bench_cuda --engine serial --engine cuda-sync --particles 65536 \
//       --iters 1000 --repeat 3 --out bench.csv --table
//
// Exit codes as the reference: 2 for usage errors (unknown engine / fitness /
// flag, bad numbers), 1 for runtime failures.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "psokit/psokit.hpp"
#include "psokit_cuda/engines.hpp"

namespace {

struct Options {
  std::vector<std::string> engines;
  std::uint32_t particles = 1024, dims = 1, iters = 1000, group_size = 128, repeat = 10;
  std::vector<std::uint64_t> seeds;
  std::string fitness = "cubic", out_path = "bench.csv", sweep, from_csv, occupancy_out;
  bool paper_scale = false, table = false, csv_table = false;
  std::size_t threads = 0;
};

std::uint64_t to_u64(const std::string& flag, const std::string& v) {
  std::size_t pos = 0;
  unsigned long long x = 0;
  try {
    x = std::stoull(v, &pos);
  } catch (const std::exception&) {
    pos = 0;
  }
  if (pos != v.size() || v.empty() || v[0] == '-')
    throw std::invalid_argument(flag + ": not a non-negative integer: '" + v + "'");
  return x;
}

std::uint32_t positive(const std::string& flag, const std::string& v) {
  const std::uint64_t x = to_u64(flag, v);
  if (x == 0 || x > 0xffffffffull) throw std::invalid_argument(flag + ": must be a positive 32-bit value");
  return static_cast<std::uint32_t>(x);
}

Options parse(int argc, char** argv) {
  Options o;
  const std::map<std::string, std::function<void(const std::string&)>> valued = {
      {"--engine", [&](const std::string& v) { o.engines.push_back(v); }},
      {"--particles", [&](const std::string& v) { o.particles = positive("--particles", v); }},
      {"--dims", [&](const std::string& v) { o.dims = positive("--dims", v); }},
      {"--iters", [&](const std::string& v) { o.iters = positive("--iters", v); }},
      {"--group-size", [&](const std::string& v) { o.group_size = positive("--group-size", v); }},
      {"--repeat", [&](const std::string& v) { o.repeat = static_cast<std::uint32_t>(to_u64("--repeat", v)); }},
      {"--seed", [&](const std::string& v) { o.seeds.push_back(to_u64("--seed", v)); }},
      {"--fitness", [&](const std::string& v) { o.fitness = v; }},
      {"--out", [&](const std::string& v) { o.out_path = v; }},
      {"--sweep", [&](const std::string& v) {
         if (v != "1d" && v != "120d") throw std::invalid_argument("--sweep: one of 1d, 120d");
         o.sweep = v;
       }},
      {"--from-csv", [&](const std::string& v) { o.from_csv = v; }},
      {"--threads", [&](const std::string& v) { o.threads = to_u64("--threads", v); }},
      {"--occupancy-out", [&](const std::string& v) { o.occupancy_out = v; }},
  };
  const std::map<std::string, bool*> flags = {
      {"--paper-scale", &o.paper_scale}, {"--table", &o.table}, {"--csv-table", &o.csv_table}};
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i], v;
    const auto eq = a.find('=');
    const bool inline_value = eq != std::string::npos;
    if (inline_value) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    if (auto f = flags.find(a); f != flags.end() && !inline_value) {
      *f->second = true;
    } else if (auto s = valued.find(a); s != valued.end()) {
      if (!inline_value) {
        if (i + 1 >= argc) throw std::invalid_argument(a + ": missing value");
        v = argv[++i];
      }
      s->second(v);
    } else {
      throw std::invalid_argument("unknown option: " + a);
    }
  }
  if (o.engines.empty()) o.engines = {"serial"};
  if (o.seeds.empty()) o.seeds = {1};
  return o;
}

// Engine names: "all" = psokit's CPU engines, then the CUDA engines.
std::vector<std::string> resolve_engines(const std::vector<std::string>& asked) {
  std::vector<std::string> out;
  for (const auto& name : asked) {
    if (name == "all") {
      for (const auto& e : psokit::engine_registry()) out.push_back(e.name);
      for (const auto& e : psokit_cuda::engine_registry()) out.push_back(e.name);
    } else {
      psokit_cuda::find_engine(name);  // invalid_argument naming the known engines
      out.push_back(name);
    }
  }
  return out;
}

// bench.hpp:99-141's loop over one engine and cell: `repeat` timed runs per
// seed, CSV rows as they complete, and the determinism audit for every engine
// whose trace is reproducible (psokit's own, and the CUDA entries marked
// parallel, i.e. bitwise run_serial; cuda-async / cuda-sync-f32 are exempt).
std::vector<psokit::bench_record> bench_cell(const Options& o, const std::string& name, std::uint32_t particles,
                                             std::uint32_t iters) {
  const psokit::engine_entry& engine = psokit_cuda::find_engine(name);
  bool audited = engine.parallel;
  for (const auto& e : psokit::engine_registry()) audited = audited || e.name == name;
  const psokit::fitness_fn& fitness = psokit::find_fitness(o.fitness);
  const psokit::pso_params params = psokit::make_params(fitness, particles, o.dims, iters, o.group_size);
  psokit::exec_options opts;
  opts.threads = o.threads;
  std::ofstream csv;
  if (!o.out_path.empty()) {
    const bool fresh = !std::ifstream(o.out_path).good();
    csv.open(o.out_path, std::ios::app);
    if (!csv) throw std::runtime_error("cannot open output file: " + o.out_path);
    if (fresh) csv << psokit::csv_header << '\n';
  }
  if (o.repeat < 3) throw std::invalid_argument("--repeat must be >= 3 (the trimmed mean drops min and max)");
  std::vector<psokit::bench_record> out;
  for (const std::uint64_t seed : o.seeds) {
    psokit::bench_record rec;
    rec.engine = name;
    rec.particles = particles;
    rec.dims = o.dims;
    rec.iters = iters;
    rec.seed = seed;
    for (std::uint32_t k = 0; k < o.repeat; ++k) {
      const psokit::run_result r = engine.run(params, fitness, psokit::rng_key{seed}, opts, {});
      rec.seconds.push_back(r.compute_seconds);
      const std::string sum = psokit::trace_checksum(r.trace);
      if (k == 0) {
        rec.final_gbest_fit = r.gbest_fit;
        rec.checksum = sum;
      } else if (audited && sum != rec.checksum) {
        throw std::runtime_error("determinism violation: engine " + name + " seed " + std::to_string(seed) +
                                 " produced differing traces");
      }
      if (csv.is_open()) psokit::write_csv_row(csv, rec, k);
    }
    std::printf("%-16s particles=%-7u dims=%-3u iters=%-6u seed=%-4llu trimmed_mean=%.6fs final_gbest=%.17g "
                "checksum=%s\n",
                rec.engine.c_str(), rec.particles, rec.dims, rec.iters, static_cast<unsigned long long>(rec.seed),
                rec.trimmed_mean_seconds(), rec.final_gbest_fit, rec.checksum.c_str());
    out.push_back(std::move(rec));
  }
  return out;
}

void occupancy_dump(const Options& o, const std::vector<std::string>& engines, std::uint32_t particles,
                    std::uint32_t iters) {
  std::string queue;
  for (const auto& e : engines)
    if (queue.empty() && (e.rfind("queue", 0) == 0 || e.rfind("cuda-queue", 0) == 0 || e == "cuda-sync"))
      queue = e;
  if (queue.empty()) throw std::invalid_argument("--occupancy-out needs a queue engine among --engine");
  const psokit::fitness_fn& fitness = psokit::find_fitness(o.fitness);
  const auto params = psokit::make_params(fitness, particles, o.dims, iters, o.group_size);
  psokit::exec_options opts;
  opts.threads = o.threads;
  const auto r = psokit_cuda::find_engine(queue).run(params, fitness, psokit::rng_key{o.seeds.front()}, opts, {});
  std::ofstream f(o.occupancy_out);
  if (!f) throw std::runtime_error("cannot open output file: " + o.occupancy_out);
  f << "iteration,occupancy\n";
  char line[64];
  for (std::size_t t = 0; t < r.queue_occupancy.size(); ++t) {
    std::snprintf(line, sizeof line, "%zu,%.17g\n", t, r.queue_occupancy[t]);
    f << line;
  }
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Options o = parse(argc, argv);
    if (!o.from_csv.empty()) {
      std::ifstream in(o.from_csv);
      if (!in) throw std::runtime_error("cannot open input file: " + o.from_csv);
      std::cout << psokit::render_table(psokit::read_csv(in), !o.csv_table);
      return 0;
    }
    psokit::find_fitness(o.fitness);  // usage error before any run
    const std::vector<std::string> engines = resolve_engines(o.engines);
    std::vector<psokit::sweep_cell> cells{{o.particles, o.iters}};
    Options run = o;
    if (o.sweep == "1d") {
      run.dims = 1;
      cells = psokit::sweep_1d(o.paper_scale);
    } else if (o.sweep == "120d") {
      run.dims = 120;
      cells = psokit::sweep_120d(o.paper_scale);
    }
    std::vector<psokit::bench_record> all;
    for (const auto& cell : cells)
      for (const auto& name : engines) {
        auto recs = bench_cell(run, name, cell.particles, cell.iters);
        all.insert(all.end(), std::make_move_iterator(recs.begin()), std::make_move_iterator(recs.end()));
      }
    if (!o.occupancy_out.empty()) occupancy_dump(run, engines, cells.front().particles, cells.front().iters);
    if (o.table || o.csv_table) std::cout << psokit::render_table(all, !o.csv_table);
  } catch (const std::invalid_argument& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
