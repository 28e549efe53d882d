#!/usr/bin/env python
"""bench.py -- particle-updates/sec of the B200-native PSO step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg3|cfg4|cfg5] [--variant cuda-sync]

One bench "step" = one full optimisation run of the workload's T iterations
(init_swarm excluded, exactly like the reference's compute_seconds,
engine_serial.hpp:25-40), with the swarm resident in HBM. The default
workload is BASELINE.json configs[1]: 1-D cubic, 2^20 particles, 1000
iterations, synchronous variant (cuda-sync).

value   = particles * iterations * steps / max-over-ranks device seconds
e2e     = the same metric through the reference-facing C-ABI call cupso_run
          (host params in, host trace/gbest out, init + H2D/D2H inside the
          timed region), wall clock
roofline: the binding roof of the dominant kernel. The temporally blocked
          kernels (k_spec, k_async_reg) keep the swarm in registers for a whole
          pass, so HBM does not bind them: their roof is instruction issue --
          warp-instructions of the exact timed schedule (ncu capture committed in
          profiles/ncu_bench_r02.json) / device time / (SMs x 4 x SM clock). The
          HBM model of SURVEY 8(d) ((5d+1)*8 algorithmic bytes per
          particle-update / launch time / MEASURED_PEAKS hbm_gbs) stays as
          roofline.hbm_model; `traffic` is the captured DRAM bytes per launch.
paper_engines: the paper's per-iteration engines (reduction, unrolled, queue,
          queue-lock) and cuda-sync without temporal blocking (wave mode) on the
          same workload, so the gain splits into aggregation and blocking.
strong_cfg5: BASELINE configs[4] as a strong-scaling sub-record on every line:
          sphere d=8, 2^28 particles in total, 2^28/N per GPU (+ the reduction
          kernel on the same swarm at N=1).
other_workloads: BASELINE configs[2] (cfg3, cuda-async) and configs[3] (cfg4,
          cuda-sync) timed in the same run at N=1, each with its roof and the
          reduction kernel on the same swarm; plus the FP32 engine on the cfg2
          swarm (cfg2_fp32, dtype f32: evidence for that engine, not the headline).
cpu_baseline: the unmodified reference (oracle/_ref, queue-lock engine, all
          host threads) on a bounded sample of the same workload, rank 0 only.
Multi-GPU: `--gpus N` without WORLD_SIZE re-launches itself under
torch.distributed.run (N ranks, one per GPU); under torchrun it checks
WORLD_SIZE == N. cuda-sync shards one swarm across the ranks (contiguous
global-index ranges; one NCCL all-gather of a pass record per pass);
engines without a sharded form (cuda-async -- SURVEY 8(e): replicas only --,
cuda-sync-f32, the classic engines) run one independent swarm per rank.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (fitness, particles, dims, iters, default variant, description)
    "cfg2": ("cubic", 1 << 20, 1, 1000, "cuda-sync", "BASELINE configs[1]: 1-D cubic, 2^20 particles, 1000 iterations"),
    "cfg3": ("cubic", 1 << 24, 1, 100, "cuda-async", "BASELINE configs[2]: 1-D cubic, 2^24 particles, async persistent"),
    "cfg4": ("rastrigin", 1 << 20, 32, 1000, "cuda-sync", "BASELINE configs[3]: Rastrigin d=32, 2^20 particles, 1000 iterations"),
    "cfg5": ("sphere", 1 << 28, 8, 200, "cuda-sync", "BASELINE configs[4]: sphere d=8, 2^28 particles (per GPU: 2^28/N), 200 iterations"),
}
STRONG = ("sphere", 1 << 28, 8, 200)  # the strong_cfg5 sub-record
STRONG_MAX_STEPS = 5
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2
PAPER_ENGINES = ("cuda-reduction", "cuda-unrolled", "cuda-queue", "cuda-queue-lock")
NCU_BENCH = os.path.join(ROOT, "profiles", "ncu_bench_r02.json")


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args_list, n) -> int:
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) under
    torch.distributed.run and pass rank 0's JSON line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + args_list
    return subprocess.call(cmd)


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every 5 ms through NVML
    (the nvidia-smi query fields clocks.sm / clocks_event_reasons.*) during the
    timed region; nvidia-smi itself is too slow for a ~100 ms region."""

    REASONS = {  # nvmlClocksEventReason* bit -> nvidia-smi field name
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, device: int, period_s: float = 0.005):
        self.device = device
        self.period = period_s
        self.sm, self.reasons, self.power = [], set(), []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.error = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # reported, never fatal
            self.error = str(e)
        return self

    def _run(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
                self.power.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
            except Exception as e:
                self.error = str(e)
                return
            self._stop.wait(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [],
                    "samples": 0, "error": self.error or "no samples"}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(self.sm), "reasons": sorted(self.reasons), "samples": len(self.sm),
                "power_w_max": max(self.power) if self.power else None, "source": "NVML, 5 ms"}


def measured_peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_bench_entry(workload: str, variant: str) -> dict:
    """The committed ncu capture of the exact timed schedule (tools/ncu_bench.py), or {}."""
    try:
        with open(NCU_BENCH) as fh:
            return json.load(fh).get(workload, {}).get(variant, {})
    except Exception:
        return {}


# ------------------------------------------------------------ CPU reference
def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _reference_runner():
    """(kind, threads, run(fitness, n, d, iters) -> compute seconds, engine name).
    The unmodified reference (oracle/_ref, queue-lock, all host threads) where it
    was built, else the C restatement's serial loop. Checker/baseline only."""
    import oracle as orc
    if not os.path.exists(orc.REF_SO) and os.path.isdir(orc.REF_INC):
        orc.build(ref=True)
    if os.path.exists(orc.REF_SO):
        ref = orc.Reference()
        threads = os.cpu_count() or 1

        def run(fitness, n, d, iters):
            r, _ = ref.run("queue-lock", fitness, n, d, iters, 1, threads=threads, want_particles=False)
            return r.compute_seconds
        return "reference", threads, run, "queue-lock (oracle/_ref, the unmodified reference)"
    o = orc.Oracle()

    def run(fitness, n, d, iters):
        return o.run_serial(fitness, n, d, iters, 1, want_state=False).compute_seconds
    return "port", 1, run, "serial (oracle/pso_oracle.c)"


def cpu_reference_leg(fitness, n, d, T, max_seconds=12.0):
    """The reference on a bounded sample of the workload (~max_seconds), plus its
    other CPU engines (serial on 1 core, reduction on all host
    cores) on ~3 s samples each."""
    kind, threads, run, engine = _reference_runner()
    per_iter = max(run(fitness, n, d, 2) / 2, 1e-6)
    iters = max(2, min(T, int(max_seconds / per_iter)))
    secs = run(fitness, n, d, iters)
    out = {"value": n * iters / secs, "unit": "particle-updates/s", "cores": threads, "kind": kind,
           "sample": f"{engine}: {fitness} d={d}, {n} particles x {iters} of {T} iterations "
                     f"(compute loop {secs:.2f} s, seed 1, cpu={_cpu_model()})"}
    if kind == "reference":
        import oracle as orc
        ref = orc.Reference()
        engines = {}
        for name, thr in (("serial", 1), ("reduction", threads)):
            try:
                def go(it):
                    r, _ = ref.run(name, fitness, n, d, it, 1, threads=thr, want_particles=False)
                    return r.compute_seconds
                pi = max(go(2) / 2, 1e-6)
                it = max(2, min(T, int(3.0 / pi)))
                sec = go(it)
                engines[f"{name} ({thr} thread{'s' if thr > 1 else ''})"] = {
                    "value": n * it / sec, "unit": "particle-updates/s", "iterations": it}
            except Exception as e:  # reported, never fatal
                engines[name] = {"error": str(e)}
        out["other_engines"] = engines
    return out


def run_reference_arm(args, world, rank):
    """The reference's own CPU implementation on the same workload: the full T
    iterations per step when a step fits STEP_BUDGET seconds (cfg2: ~8 s on 16
    host cores), else a bounded sample of the iterations (a rate: the
    per-iteration cost is flat)."""
    if rank != 0:
        return 0
    step_budget = 15.0
    fitness, n, d, T, _, desc = WORKLOADS[args.workload]
    if args.iters:
        T = args.iters
    n_rank = n if args.workload != "cfg5" else (1 << 24)  # 2^28 FP64 state would need ~56 GB of host RAM
    kind, threads, run, engine = _reference_runner()
    per_iter = max(run(fitness, n_rank, d, 2) / 2, 1e-6)
    iters = T if per_iter * T <= step_budget else max(2, int(step_budget / per_iter))
    vals = []
    for k in range(args.warmup + args.steps):
        s = run(fitness, n_rank, d, iters)
        if k >= args.warmup:
            vals.append(s)
    secs = sum(vals)
    value = n_rank * iters * len(vals) / secs
    same = iters == T and n_rank == n
    line = {
        "impl": "reference", "metric": "particle-updates/sec", "value": value, "unit": "particle-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / len(vals), "higher_is_better": True,
        "scaling": "strong" if args.workload == "cfg5" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox init of the reference)",
        "config": {"workload": desc, "fitness": fitness, "particles": n_rank, "dims": d,
                   "iterations_per_step": iters, "iterations_of_workload": T, "same_config": same,
                   "engine": f"reference {engine}, {threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "particle-updates/s", "cores": threads, "kind": kind,
                         "sample": f"{fitness} d={d}, {n_rank} particles x {iters} iterations per step, "
                                   f"cpu={_cpu_model()}"},
        "e2e": {"value": value, "unit": "particle-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def flush_l2(torch, dev):
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
        flush_l2.buf = buf
    buf.random_(0, 1 << 30)


class Job:
    """One swarm (or shard / replica) per rank and the timing protocol: W untimed
    warm-up steps, then K steps, each = init_swarm + L2 flush (untimed) + the T
    iterations timed with CUDA events on the launching stream; barrier + sync on
    both sides; max over ranks of the summed device seconds."""

    def __init__(self, cp, torch, pg, dev, local, world, rank, fitness, n_total, d, T, variant, sharded_total):
        self.cp, self.torch, self.pg, self.dev, self.local = cp, torch, pg, dev, local
        self.world, self.rank = world, rank
        self.engine = cp.find_engine(variant)
        self.variant = variant
        self.f = cp.find_fitness(fitness)
        self.T, self.d = T, d
        # cuda-sync shards one swarm; the other engines run one swarm per rank
        self.replicas = world > 1 and variant != "cuda-sync"
        if self.replicas:
            n_rank = n_total // world if sharded_total else n_total
            self.p = cp.make_params(self.f, n_rank, d, T)
            self.seed, first, self.count = 1 + rank, 0, n_rank
            self.n_total = n_rank * world
            self.sw = cp.Swarm(self.p, self.f, self.seed, device=local)
        else:
            self.n_total = n_total if sharded_total else n_total * world
            self.p = cp.make_params(self.f, self.n_total, d, T)
            self.seed = 1
            first, self.count = cp.shard_range(self.n_total, world, rank)
            self.sw = cp.Swarm(self.p, self.f, self.seed, device=local, first=first, count=self.count)
            if world > 1:
                uid = [cp.nccl_unique_id() if rank == 0 else None]
                pg.broadcast_object_list(uid, src=0)
                self.sw.nccl_init(uid[0], world, rank)

    def barrier(self):
        if self.pg:
            self.pg.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if not self.pg:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def run(self, warmup: int, steps: int, variant=None, clocks=None):
        v = (variant or self.engine).variant
        for _ in range(warmup):
            self.sw.init()
            flush_l2(self.torch, self.dev)
            self.barrier()
            self.sw.step(v, self.T)
        per = []
        self.barrier()
        self.spec_at_start = self.sw.spec_stats()  # pass counters of the timed steps only
        ctx = clocks if clocks is not None else _Null()
        with ctx:
            for _ in range(steps):
                self.sw.init()
                flush_l2(self.torch, self.dev)
                self.barrier()
                per.append(self.sw.step(v, self.T))
            self.barrier()
        return self.max_over_ranks(sum(per)), len(per)

    def close(self):
        self.sw.close()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def roofline_of(job, workload, variant, dev_secs, K, clocks, spec_delta, torch):
    """Binding roof of the dominant kernel, see the module docstring."""
    cp, sw, T, d = job.cp, job.sw, job.T, job.d
    f32 = variant == "cuda-sync-f32"
    bytes_per_pu = (5 * d + 1) * (4 if f32 else 8)
    mode = sw.sync_mode() if variant == "cuda-sync" else ("spec" if f32 else None)
    amode = sw.async_mode() if variant == "cuda-async" else None
    passes, fails, launches = (x / K for x in spec_delta)
    spec = mode in ("spec", "nccl-sharded-spec")
    grid = sw.sync_grid_blocks()
    persistent = variant == "cuda-async" or (variant == "cuda-sync" and job.world == 1 and grid > 0 and not spec)
    launches_per_step = {"cuda-sync": (launches * (2 if job.world > 1 else 1)) if spec else
                         (1 if persistent else (2 * T if job.world > 1 else T)), "cuda-async": 1,
                         "cuda-queue-lock": T, "cuda-queue": 2 * T, "cuda-reduction": 2 * T,
                         "cuda-unrolled": 2 * T, "cuda-sync-f32": launches}[variant]
    iters_per_launch = T if persistent else (T / passes if spec and passes else 1)
    launch_secs = (dev_secs / K) / (T / iters_per_launch)
    alg_bytes = job.count * iters_per_launch * bytes_per_pu
    peak, peak_src = measured_peak_gbs()
    achieved = alg_bytes / launch_secs / 1e9
    fit = job.f.name
    kernel = {"resident": f"k_sync_res<{fit},{d}>", "persistent": f"k_sync<{fit}>", "wave": f"k_wave<{fit}>",
              "spec": f"k_spec<{fit},{d}>" if d in (1, 2, 4, 8) and not (fit == "rastrigin" and d == 8)
              else f"k_spec_split<{fit},d={d}>", "nccl-sharded-spec": f"k_spec<{fit},{d}>+k_spec_commit"}.get(
                  mode, f"k_propose<{fit}>+k_commit")
    if f32:
        kernel = f"k_spec32<{fit},{d}>"
    if variant == "cuda-async":
        kernel = {"reg": f"k_async_reg<{fit},{d}>", "tiled": f"k_async_tiled<{fit}>"}.get(amode, f"k_async<{fit}>")
    elif variant not in ("cuda-sync", "cuda-sync-f32"):
        kernel = f"k_classic_step<{fit}>"
    hbm = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "peak_source": peak_src, "alg_bytes_per_launch": alg_bytes, "launch_ms": launch_secs * 1e3,
           "bytes_per_particle_update": bytes_per_pu}
    e = ncu_bench_entry(workload, variant) if job.world == 1 else {}
    traffic = None
    if e.get("dram_bytes_per_step") is not None and e.get("launches_per_step"):
        traffic = e["dram_bytes_per_step"] / e["launches_per_step"]
    blocked = mode in ("resident", "spec", "nccl-sharded-spec") or amode == "reg"
    sm_hz = ((clocks or {}).get("sm_mhz") or 1965.0) * 1e6
    nsm = torch.cuda.get_device_properties(job.dev).multi_processor_count
    roof = None
    if blocked and e.get("warp_inst_per_step"):
        ach = e["warp_inst_per_step"] * K / dev_secs  # warp-instructions per second, live device time
        peak_i = nsm * 4 * sm_hz
        roof = {"bound": "issue", "achieved": ach / 1e9, "peak": peak_i / 1e9, "unit": "G warp-instructions/s",
                "frac": ach / peak_i, "traffic": traffic,
                "inst_per_particle_update": e["warp_inst_per_step"] * 32 / (job.count * T),
                "peak_source": f"{nsm} SMs x 4 schedulers x SM clock {sm_hz / 1e6:.0f} MHz (NVML, timed region)",
                "source": f"smsp__inst_executed.sum over the exact timed schedule ({e.get('capture', '?')})"}
    if roof is not None and e.get("fmaheavy_cycles_per_step"):
        # the pipe Philox saturates: IMAD.WIDE.U32 holds the fma-heavy pipe 4 cycles per
        # warp-instruction per SMSP (tools/micro/pipes.cu); busy SMSP-cycles of the exact
        # schedule (ncu) over the live SMSP-cycles of the timed region
        busy = e["fmaheavy_cycles_per_step"] * K
        roof["pipe_fmaheavy"] = {"frac": busy / (4 * nsm * sm_hz * dev_secs),  # the .sum counts per SMSP
                                 "busy_smsp_cycles_per_step": e["fmaheavy_cycles_per_step"],
                                 "ncu_pct_of_active": e.get("fmaheavy_pct_of_active_ncu"),
                                 "source": "sm__pipe_fmaheavy_cycles_active.sum over the exact timed schedule"}
    if roof is None:  # streaming kernels: the HBM model binds
        roof = dict(hbm, traffic=traffic)
    roof.update({"kernel": kernel, "mode": mode or amode, "hbm_model": hbm,
                 "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over "
                                 "the launches of one timed step (profiles/ncu_bench_r02.json)"})
    if blocked:
        roof["note"] = ("temporally blocked: each pass reads and writes the state once for K iterations held "
                        "in registers, so the HBM model (hbm_model.frac > 1) does not bind; instruction issue does")
    # RNG ceiling: the reference's two Philox-4x32-10 calls per particle-axis alone
    # run at 3.11e11 draw pairs/s on a B200 (profiles/micro_philox_r01.txt); the
    # FP32 engine draws one call per particle-axis and iteration pair (4x fewer)
    draws_ps = 3.114e11 * (4.0 if f32 else 1.0)
    value = job.n_total * T * K / dev_secs
    rng_peak = draws_ps / d * job.world
    roof["rng_ceiling"] = {"bound": "issue (Philox IMAD.WIDE/LOP3)", "achieved": value, "peak": rng_peak,
                           "unit": "particle-updates/s", "frac": value / rng_peak,
                           "source": "profiles/micro_philox_r01.txt (draw-only microbenchmark, 1 GPU)"}
    if spec:
        roof["spec"] = {"passes_per_step": passes, "launches_per_step": launches, "falsified_per_step": fails,
                        "iters_per_pass": T / passes if passes else None}
    return roof, launches_per_step


def paper_engines_leg(job, K):
    """The paper's per-iteration engines and cuda-sync without temporal blocking on
    the same swarm (rank 0, N=1): aggregation vs blocking."""
    cp = job.cp
    out = {}
    steps = max(2, min(K, 5))
    for name in PAPER_ENGINES:
        secs, k = job.run(2, steps, cp.find_engine(name))
        out[name] = {"value": job.n_total * job.T * k / secs, "unit": "particle-updates/s"}
    if job.variant == "cuda-sync":
        os.environ["CUPSO_SYNC_MODE"] = "wave"  # read when a handle picks its mode
        try:
            wave = Job(cp, job.torch, None, job.dev, job.local, 1, 0, job.f.name, job.n_total, job.d, job.T,
                       "cuda-sync", True)
            secs, k = wave.run(2, steps)
            wave.close()
            out["cuda-sync (wave: one fused launch per iteration, no temporal blocking)"] = {
                "value": job.n_total * job.T * k / secs, "unit": "particle-updates/s"}
        finally:
            del os.environ["CUPSO_SYNC_MODE"]
    out["note"] = ("reduction/unrolled/queue/queue-lock: engine_reduction.hpp / engine_queue.hpp restated as one "
                   "or two launches per iteration (CUDA graph); the queue-lock / reduction ratio is the paper's "
                   "aggregation claim (PAPER.md:442); wave / queue-lock isolates the fused step + B200 "
                   "aggregation; headline / wave is the temporal blocking")
    return out


def strong_cfg5_leg(cp, torch, pg, dev, local, world, rank, warmup, steps):
    """BASELINE configs[4] strong-scaled: 2^28 particles in total, 2^28/N per GPU."""
    fitness, n, d, T = STRONG
    job = Job(cp, torch, pg, dev, local, world, rank, fitness, n, d, T, "cuda-sync", True)
    K = max(1, min(steps, STRONG_MAX_STEPS))
    clk = ClockSampler(local)
    secs, K = job.run(max(3, min(warmup, 3)), K, clocks=clk)
    clocks = clk.summary()
    s0, s1 = job.spec_at_start, job.sw.spec_stats()
    rec = {"metric": "particle-updates/sec", "value": n * T * K / secs, "unit": "particle-updates/s",
           "n_gpus": world, "steps": K, "warmup": 3, "ms_per_step": 1e3 * secs / K, "scaling": "strong",
           "config": {"fitness": fitness, "particles_total": n, "particles_per_gpu": job.count, "dims": d,
                      "iterations_per_step": T, "variant": "cuda-sync", "parallelism": f"dp{world} (particle shards)",
                      "mode": job.sw.sync_mode(), "passes_per_step": (s1[0] - s0[0]) / K,
                      "falsified_per_step": (s1[1] - s0[1]) / K},
           "final_gbest_fit": job.sw.gbest().fit, "clocks": clocks}
    if world == 1:  # binding roof from the exact-schedule capture of this workload (ncu_bench_r02 cfg5)
        roof, _ = roofline_of(job, "cfg5", "cuda-sync", secs, K, clocks, [b - a for a, b in zip(s0, s1)], torch)
        keep = ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel", "pipe_fmaheavy")
        rec["roofline"] = {k: v for k, v in roof.items() if k in keep}
        rec["hbm_model_frac"] = roof["hbm_model"]["frac"]
    if world == 1:  # the in-repo reduction kernel on the same 2^28 swarm (~4 s per step)
        rsecs, rk = job.run(1, 2, cp.find_engine("cuda-reduction"))
        red = n * T * rk / rsecs
        rec["reduction_baseline"] = {"variant": "cuda-reduction", "value": red, "unit": "particle-updates/s",
                                     "speedup": rec["value"] / red}
    job.close()
    return rec


def workload_leg(cp, torch, dev, local, name, warmup, steps, variant=None, with_reduction=True):
    """Another BASELINE workload on the same GPU in the same run (rank 0, N=1):
    its default engine, timed exactly like the headline (device time, L2
    flushed, clocks sampled), its binding roof, and the in-repo reduction kernel
    on the same swarm -- so every configs[] row is measured by the driver's own
    bench run, not only the headline."""
    fitness, n, d, T, default_variant, desc = WORKLOADS[name]
    variant = variant or default_variant
    job = Job(cp, torch, None, dev, local, 1, 0, fitness, n, d, T, variant, True)
    try:
        clk = ClockSampler(local)
        secs, K = job.run(max(3, min(warmup, 3)), max(2, min(steps, 5)), clocks=clk)
        clocks = clk.summary()
        s0, s1 = job.spec_at_start, job.sw.spec_stats()
        roof, launches = roofline_of(job, name, variant, secs, K, clocks, [b - a for a, b in zip(s0, s1)], torch)
        value = n * T * K / secs
        red = None
        if with_reduction:
            rsecs, rk = job.run(1, 2, cp.find_engine("cuda-reduction"))
            red = n * T * rk / rsecs
        keep = ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel", "mode", "inst_per_particle_update",
                "pipe_fmaheavy")
        return {"metric": "particle-updates/sec", "value": value, "unit": "particle-updates/s", "steps": K,
                "ms_per_step": 1e3 * secs / K, "dtype": "f32" if variant == "cuda-sync-f32" else "f64",
                "config": {"workload": desc, "fitness": fitness, "particles": n, "dims": d,
                           "iterations_per_step": T, "variant": variant},
                "roofline": {k: v for k, v in roof.items() if k in keep},
                "hbm_model_frac": roof["hbm_model"]["frac"], "clocks": clocks, "gpu_launches": launches * K,
                "reduction_baseline": None if red is None else {
                    "variant": "cuda-reduction", "value": red, "unit": "particle-updates/s", "speedup": value / red},
                "final_gbest_fit": job.sw.gbest().fit}
    finally:
        job.close()


def dry_run(args, world, rank):
    """CPU check of the launch plumbing (no GPU work): ranks, gloo rendezvous,
    max-over-ranks reduction and the line's shape."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo", init_method="env://", world_size=world, rank=rank)
        import torch
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mx = float(t.item())
        dist.destroy_process_group()
    else:
        mx = 1.0
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": "particle-updates/sec", "value": None, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "max_over_ranks_check": mx,
                          "workload": args.workload,
                          "strong_cfg5": {"dry_run": True, "n_gpus": world, "particles_total": STRONG[1],
                                          "particles_per_gpu": STRONG[1] // world}}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default=None)
    ap.add_argument("--iters", type=int, default=None, help="override iterations per step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-baseline-kernel", action="store_true", help="skip the paper_engines leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-strong", action="store_true", help="skip the strong_cfg5 sub-record")
    ap.add_argument("--no-others", action="store_true", help="skip the cfg3 / cfg4 sub-records")
    ap.add_argument("--dry-run", action="store_true", help="launch plumbing only (CPU)")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(sys.argv[1:], args.gpus)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.dry_run:
        return dry_run(args, world, rank)
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)

    import torch
    import paper_2205_01313_b200 as cp

    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise RuntimeError("bench.py: no CUDA device (the product has no CPU path)")
    local = local % ndev  # more ranks than GPUs: replicas share devices
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fitness, n_base, d, T, default_variant, desc = WORKLOADS[args.workload]
    if args.iters:
        T = args.iters
    variant = args.variant or default_variant
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://", world_size=world, rank=rank)
        pg = dist

    job = Job(cp, torch, pg, dev, local, world, rank, fitness, n_base, d, T, variant, args.workload == "cfg5")
    clk = ClockSampler(local)
    dev_secs, K = job.run(args.warmup, args.steps, clocks=clk)
    clocks = clk.summary()
    spec0, spec1 = job.spec_at_start, job.sw.spec_stats()
    value = job.n_total * T * K / dev_secs
    gb = job.sw.gbest()
    roofline, launches_per_step = roofline_of(job, args.workload, variant, dev_secs, K, clocks,
                                              [b - a for a, b in zip(spec0, spec1)], torch)

    extra = {}
    if world == 1 and not args.no_baseline_kernel:
        extra["paper_engines"] = paper_engines_leg(job, K)
        red = extra["paper_engines"]["cuda-reduction"]["value"]
        extra["reduction_baseline"] = {"variant": "cuda-reduction", "value": red, "unit": "particle-updates/s",
                                       "speedup_of_headline": value / red}

    # ---- e2e through the reference-facing C-ABI call (cupso_run), host buffers ----
    e2e = None
    job.close()  # cupso_run owns its own device swarm
    if not args.no_e2e and world == 1:
        e2e_secs = []
        for k in range(1 + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = job.engine.run(job.p, job.f, cp.rng_key(job.seed), cp.exec_options(device=local))
            e2e_secs.append(time.perf_counter() - t0)
        e2e_secs = e2e_secs[1:]
        h2d = C.sizeof(cp._lib.cupso_params) + 8  # params + seed; the swarm is initialised on device
        d2h = T * (8 + 4 + 8 + 8) + (16 + 8 * d) + 16  # trace, particle, admitted, async key; gbest record; initial
        e2e = {"value": job.n_total * T * len(e2e_secs) / sum(e2e_secs), "unit": "particle-updates/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "cupso_run via find_engine(...).run (init_swarm + T iterations + result D2H; "
                       "device swarm reused across calls of the same shape)",
               "final_gbest_fit": r.gbest_fit}
    elif not args.no_e2e:
        # N > 1: the shard handle API end to end (init_swarm + NCCL gbest exchange +
        # T iterations + trace/gbest D2H), wall clock, max over ranks
        job2 = Job(cp, torch, pg, dev, local, world, rank, fitness, n_base, d, T, variant, args.workload == "cfg5")
        e2e_secs = []
        for k in range(1 + args.steps):
            job2.barrier()
            t0 = time.perf_counter()
            job2.sw.init()
            job2.sw.step(job2.engine.variant, T)
            job2.sw.trace()
            job2.sw.gbest()
            e2e_secs.append(time.perf_counter() - t0)
        job2.close()
        tot = job.max_over_ranks(sum(e2e_secs[1:]))
        e2e = {"value": job.n_total * T * args.steps / tot, "unit": "particle-updates/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": T * (8 + 4 + 8 + 8) + 16 + 8 * d,
               "path": ("Swarm API per rank (independent replicas)" if job.replicas else
                        "Swarm shard API per rank: init (with NCCL adopt)") + " + step + trace + gbest; max over ranks"}

    strong = None
    if not args.no_strong:
        try:
            strong = strong_cfg5_leg(cp, torch, pg, dev, local, world, rank, args.warmup, args.steps)
        except Exception as e:  # reported, never fatal for the headline line
            strong = {"error": str(e)}

    others = None
    if world == 1 and args.workload == "cfg2" and not args.no_others:
        others = {}
        for name in ("cfg3", "cfg4"):
            try:
                others[name] = workload_leg(cp, torch, dev, local, name, args.warmup, args.steps)
            except Exception as e:  # reported, never fatal for the headline line
                others[name] = {"error": str(e)}
        try:  # the FP32 engine on the headline swarm: reduced precision, not the headline
            others["cfg2_fp32"] = workload_leg(cp, torch, dev, local, "cfg2", args.warmup, args.steps,
                                               variant="cuda-sync-f32", with_reduction=False)
        except Exception as e:
            others["cfg2_fp32"] = {"error": str(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_leg(fitness, min(job.count, 1 << 24), d, T)
        except Exception as e:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": "particle-updates/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": "particle-updates/sec", "value": value, "unit": "particle-updates/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * dev_secs / K,
            "higher_is_better": True, "scaling": "strong" if args.workload == "cfg5" else "weak",
            "vs_baseline": None, "dtype": "f32" if variant == "cuda-sync-f32" else "f64",
            "data": "synthetic (Philox-initialised swarm, reference make_params defaults)",
            "config": {"workload": desc, "fitness": fitness, "particles_total": job.n_total,
                       "particles_per_gpu": job.count, "dims": d, "iterations_per_step": T,
                       "variant": variant,
                       "parallelism": f"replicas{world} (independent swarms, seeds 1..{world})" if job.replicas
                       else f"dp{world} (particle shards)",
                       "l2": "flushed (512 MiB write) before every step; within a step the swarm stays resident "
                             "as in a real run"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * K, "final_gbest_fit": gb.fit,
            "strong_cfg5": strong,
            "other_workloads": others,
            **extra,
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
