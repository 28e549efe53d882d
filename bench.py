#!/usr/bin/env python
"""bench.py -- particle-updates/sec of the B200-native PSO step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg3|cfg4|cfg5] [--variant cuda-sync]

One bench "step" = one full optimisation run of the workload's T iterations
(init_swarm excluded, exactly like the reference's compute_seconds,
engine_serial.hpp:25-40), with the swarm resident in HBM. The default
workload is BASELINE.json configs[1]: 1-D cubic, 2^20 particles, 1000
iterations, synchronous atomic variant (cuda-sync); the in-repo reduction
baseline kernel (cuda-reduction) is timed on the same workload in the same run.

value   = particles * iterations * steps * world / max-over-ranks device seconds
e2e     = the same metric through the reference-facing C-ABI call cupso_run
          (host params in, host trace/gbest out, allocation + init + H2D/D2H
          inside the timed region), wall clock
roofline: algorithmic bytes (5d+1)*8 per particle-update per
          launch / CUDA-event duration of that launch, against MEASURED_PEAKS.json
cpu_baseline: the unmodified reference (oracle/_ref, queue-lock engine, all
          host threads) on a bounded sample of the same workload, rank 0 only
Multi-GPU (torchrun): weak scaling, each rank holds a contiguous shard of one
swarm of world*N particles; the per-iteration gbest exchange is an NCCL
all-gather of one (16+8d)-byte record per rank issued by libcupso on its stream.
Engines without a sharded form (cuda-async -- SURVEY 8(e): replicas only --,
cuda-sync-f32, the classic engines) run one independent swarm per rank instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
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
    "cfg5": ("sphere", 1 << 28, 8, 50, "cuda-sync", "BASELINE configs[4]: sphere d=8, 2^28 particles (per GPU: 2^28/N)"),
}
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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


def ncu_entry(workload: str, variant: str) -> dict:
    """The committed ncu summary entry (profiles/ncu_summary_*.json) for a kernel, or {}."""
    pdir = os.path.join(ROOT, "profiles")
    for name in sorted(os.listdir(pdir), reverse=True) if os.path.isdir(pdir) else []:
        if name.startswith("ncu_summary") and name.endswith(".json"):
            try:
                with open(os.path.join(pdir, name)) as fh:
                    e = json.load(fh).get(workload, {}).get(variant)
                if e and e.get("dram_bytes_per_launch") is not None:
                    return e
            except Exception:
                pass
    return {}


def ncu_traffic(workload: str, variant: str):
    """(dram bytes per iteration, 1) from the committed ncu summary, or (None, None)."""
    e = ncu_entry(workload, variant)
    if not e:
        return None, None
    if e.get("dram_bytes_per_iter") is not None:
        return e["dram_bytes_per_iter"], 1
    return e["dram_bytes_per_launch"], e.get("iters_per_launch")


def cpu_reference_leg(fitness, n, d, max_seconds=12.0, sample_iters=None):
    """The unmodified reference (oracle/_ref) queue-lock engine on all host threads,
    timed on a bounded sample of the workload. Checker/baseline only."""
    import oracle as orc
    if not os.path.exists(orc.REF_SO):
        if os.path.isdir(orc.REF_INC):
            orc.build(ref=True)
    if os.path.exists(orc.REF_SO):
        kind = "reference"
        ref = orc.Reference()
        threads = os.cpu_count() or 1
        # calibrate: 2 iterations, then size the sample to ~max_seconds
        r, _ = ref.run("queue-lock", fitness, n, d, 2, 1, threads=threads, want_particles=False)
        per_iter = max(r.compute_seconds / 2, 1e-6)
        iters = sample_iters or max(2, min(1000, int(max_seconds / per_iter)))
        r, _ = ref.run("queue-lock", fitness, n, d, iters, 1, threads=threads, want_particles=False)
        secs = r.compute_seconds
        engine = "queue-lock"
    else:  # the C restatement, single thread
        kind = "port"
        o = orc.Oracle()
        threads = 1
        r = o.run_serial(fitness, n, d, 2, 1, want_state=False)
        per_iter = max(r.compute_seconds / 2, 1e-6)
        iters = sample_iters or max(2, min(1000, int(max_seconds / per_iter)))
        r = o.run_serial(fitness, n, d, iters, 1, want_state=False)
        secs = r.compute_seconds
        engine = "serial (oracle/pso_oracle.c)"
    return {"value": n * iters / secs, "unit": "particle-updates/s", "cores": threads, "kind": kind,
            "sample": f"{engine}: {fitness} d={d}, {n} particles x {iters} iterations "
                      f"(compute loop {secs:.2f} s, seed 1, cpu={_cpu_model()})"}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference_arm(args, world, rank):
    if rank != 0:
        return 0
    fitness, n, d, T, _, desc = WORKLOADS[args.workload]
    n_rank = n if args.workload != "cfg5" else (1 << 24)  # 2^28 FP64 state does not fit host RAM budget
    import oracle as orc
    if not os.path.exists(orc.REF_SO) and os.path.isdir(orc.REF_INC):
        orc.build(ref=True)
    base = cpu_reference_leg(fitness, n_rank, d, max_seconds=3.0)
    # each step: a bounded sample run of the same workload
    iters = int(base["sample"].split(" x ")[1].split(" ")[0])
    vals = []
    if base["kind"] == "reference":
        ref = orc.Reference()
        for k in range(args.warmup + args.steps):
            r, _ = ref.run("queue-lock", fitness, n_rank, d, iters, 1, threads=base["cores"], want_particles=False)
            if k >= args.warmup:
                vals.append(r.compute_seconds)
    else:
        o = orc.Oracle()
        for k in range(args.warmup + args.steps):
            r = o.run_serial(fitness, n_rank, d, iters, 1, want_state=False)
            if k >= args.warmup:
                vals.append(r.compute_seconds)
    secs = sum(vals)
    value = n_rank * iters * len(vals) / secs
    line = {
        "impl": "reference", "metric": "particle-updates/sec", "value": value, "unit": "particle-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / len(vals), "higher_is_better": True, "scaling": "strong" if args.workload == "cfg5" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox init of the reference)",
        "config": {"workload": desc, "fitness": fitness, "particles": n_rank, "dims": d,
                   "iterations_per_step": iters, "engine": "reference queue-lock (all host threads)"},
        "cpu_baseline": {**base, "value": value},
        "e2e": {"value": value, "unit": "particle-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def flush_l2(torch, dev):
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
        flush_l2.buf = buf
    buf.random_(0, 1 << 30)


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
    ap.add_argument("--no-baseline-kernel", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)

    import torch
    import paper_2205_01313_b200 as cp

    local = local % max(1, torch.cuda.device_count())  # more ranks than GPUs: replicas share devices
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fitness, n_per_rank, d, T, default_variant, desc = WORKLOADS[args.workload]
    if args.workload == "cfg5":
        n_total = n_per_rank
        n_per_rank = n_total // world
    else:
        n_total = n_per_rank * world
    if args.iters:
        T = args.iters
    variant_name = args.variant or default_variant
    engine = cp.find_engine(variant_name)
    f = cp.find_fitness(fitness)
    p = cp.make_params(f, n_total, d, T)
    seed = 1

    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://", world_size=world, rank=rank)
        pg = dist
    # cuda-sync shards one swarm across the ranks (NCCL pass-record exchange);
    # the other engines have no sharded form (cuda-async: SURVEY 8(e) "replicas
    # only"), so at N > 1 every rank runs an independent swarm of n_per_rank
    # particles with its own seed and no data-path collective.
    replicas = world > 1 and variant_name != "cuda-sync"
    if replicas:
        p = cp.make_params(f, n_per_rank, d, T)
        seed = 1 + rank
        first, count = 0, n_per_rank
    else:
        first, count = cp.shard_range(n_total, world, rank)

    def barrier():
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    sw = cp.Swarm(p, f, seed, device=local, first=first, count=count) if not replicas else \
        cp.Swarm(p, f, seed, device=local)
    if world > 1 and not replicas:
        uid = [cp.nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(uid, src=0)
        sw.nccl_init(uid[0], world, rank)

    # ---- W warmup steps, then exactly K timed steps. Each step: init_swarm and an
    # L2 flush (untimed), then the T iterations timed with CUDA events recorded by
    # libcupso on the stream that launches the kernels (device seconds). ----
    for k in range(args.warmup):
        sw.init()
        flush_l2(torch, dev)
        barrier()
        sw.step(engine.variant, T)
    per_step = []
    spec0 = sw.spec_stats()
    barrier()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            sw.init()
            flush_l2(torch, dev)
            barrier()
            per_step.append(sw.step(engine.variant, T))
        barrier()
    clocks = clk.summary()
    dev_secs = sum(per_step)
    if pg:
        t = torch.tensor([dev_secs], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        dev_secs = float(t.item())
    K = len(per_step)
    value = n_total * T * K / dev_secs
    gb = sw.gbest()
    grid = sw.sync_grid_blocks()

    # ---- roofline of the dominant kernel (one launch = T iterations for the persistent kernels) ----
    f32 = variant_name == "cuda-sync-f32"
    bytes_per_pu = (5 * d + 1) * (4 if f32 else 8)
    # cuda-sync runs as speculative passes (k_spec: ~T/K launches per step),
    # persistent (1 cooperative launch per step) or as a graph of one wave per
    # iteration; shards: propose+commit per iteration
    mode = sw.sync_mode() if variant_name == "cuda-sync" else ("spec" if f32 else None)
    amode = sw.async_mode() if variant_name == "cuda-async" else None
    spec1 = sw.spec_stats()
    spec_passes = (spec1[0] - spec0[0]) / K
    spec_launches = (spec1[2] - spec0[2]) / K
    spec = mode in ("spec", "nccl-sharded-spec")
    persistent = variant_name == "cuda-async" or (variant_name == "cuda-sync" and world == 1 and grid > 0
                                                  and not spec)
    # sharded spec: k_spec + k_spec_commit per pass (the all-gather is NCCL's)
    launches_per_step = {"cuda-sync": (spec_launches * (2 if world > 1 else 1)) if spec else
                         (1 if persistent else (2 * T if world > 1 else T)), "cuda-async": 1,
                         "cuda-queue-lock": T, "cuda-queue": 2 * T, "cuda-reduction": 2 * T,
                         "cuda-unrolled": 2 * T, "cuda-sync-f32": spec_launches}[variant_name]
    iters_per_launch = T if persistent else (T / spec_passes if spec else 1)
    launch_secs = (dev_secs / K) / (T / iters_per_launch)
    alg_bytes = count * iters_per_launch * bytes_per_pu
    peak, peak_src = measured_peak_gbs()
    achieved = alg_bytes / launch_secs / 1e9
    traffic, traffic_iters = ncu_traffic(args.workload, variant_name)
    if traffic is not None and traffic_iters:
        traffic = traffic * iters_per_launch / traffic_iters
    sync_kernel = {"resident": f"k_sync_res<{fitness},{d if d == 1 else 0}>", "persistent": f"k_sync<{fitness}>",
                   "wave": f"k_wave<{fitness}>", "spec": f"k_spec<{fitness},{d}>",
                   "nccl-sharded-spec": f"k_spec<{fitness},{d}>+k_spec_commit"}.get(
                       mode, f"k_propose<{fitness}>+k_commit")
    if f32:
        sync_kernel = f"k_spec32<{fitness},{d}>"
    async_kernel = {"reg": f"k_async_reg<{fitness},{d}>", "tiled": f"k_async_tiled<{fitness}>"}.get(
        amode, f"k_async<{fitness}>")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src,
                "kernel": {"cuda-sync": sync_kernel, "cuda-sync-f32": sync_kernel,
                           "cuda-async": async_kernel}.get(variant_name, f"k_classic_step<{fitness}>"),
                "mode": mode or amode,
                "traffic_note": "ncu dram read+write per launch (profiles/ncu_summary_r01.json); "
                                "below alg bytes = L2-resident state, above = pbest write-backs",
                "alg_bytes_per_launch": alg_bytes, "launch_ms": launch_secs * 1e3,
                "bytes_per_particle_update": bytes_per_pu}
    # RNG ceiling: the reference's two Philox-4x32-10 calls per particle-axis alone
    # run at 3.11e11 draw pairs/s on a B200 (profiles/micro_philox_r01.txt); the
    # FP32 engine draws one call per particle-axis and iteration pair (4x fewer)
    draws_ps = 3.114e11 * (4.0 if f32 else 1.0)
    rng_peak = draws_ps / d * world  # whole job
    roofline["rng_ceiling"] = {"bound": "issue (Philox IMAD.WIDE/LOP3)", "achieved": value,
                               "peak": rng_peak, "unit": "particle-updates/s", "frac": value / rng_peak,
                               "source": "profiles/micro_philox_r01.txt (draw-only microbenchmark, 1 GPU)"}
    if spec:
        roofline["spec"] = {"passes_per_step": spec_passes, "launches_per_step": spec_launches,
                            "falsified_per_step": (spec1[1] - spec0[1]) / K,
                            "iters_per_pass": T / spec_passes if spec_passes else None}
    if mode in ("resident", "spec", "nccl-sharded-spec") or amode == "reg":
        # The swarm lives in SMEM for the whole launch: HBM carries ~0 bytes per
        # iteration, so the algorithmic-bytes figure above can exceed
        # the HBM roof. The binding roof is instruction issue (Philox IMAD/LOP3 +
        # FP64): executed warp-instructions per iteration from the committed ncu
        # capture vs 148 SMs x 4 schedulers x SM clock.
        e = ncu_entry(args.workload, variant_name)
        if e.get("warp_inst_per_launch"):
            winst_iter = e.get("warp_inst_per_iter") or e["warp_inst_per_launch"] / e["iters_per_launch"]
            sm_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
            nsm = torch.cuda.get_device_properties(dev).multi_processor_count
            ach = winst_iter * T * K / dev_secs
            roofline["issue_roofline"] = {
                "bound": "issue", "achieved": ach / 1e9, "peak": nsm * 4 * sm_hz / 1e9,
                "unit": "G warp-instructions/s", "frac": ach / (nsm * 4 * sm_hz),
                "inst_per_particle_update": winst_iter * 32 / count,
                "source": "smsp__inst_executed.sum of " + e.get("capture", "?")}
        roofline["note"] = {
            "resident": "SMEM-resident swarm (k_sync_res): state read/written once per launch, not per iteration",
            "spec": "temporally blocked (k_spec): each pass reads/writes the state once for K iterations held in "
                    "registers",
            "nccl-sharded-spec": "temporally blocked shards (k_spec): one all-gather of a pass record per pass",
        }.get(mode, "temporally blocked (k_async_reg): state read/written once per K iterations held in registers") \
            + "; frac > 1 means the HBM model does not bind -- see issue_roofline"

    extra = {}
    # ---- the in-repo reduction baseline kernel on the same workload (rank 0, N=1) ----
    if world == 1 and not args.no_baseline_kernel and variant_name != "cuda-reduction":
        red = cp.find_engine("cuda-reduction")
        rs = []
        for k in range(2 + max(2, args.steps // 2)):
            sw.init()
            flush_l2(torch, dev)
            torch.cuda.synchronize()
            s = sw.step(red.variant, T)
            if k >= 2:
                rs.append(s)
        rv = n_total * T * len(rs) / sum(rs)
        extra["reduction_baseline"] = {"variant": "cuda-reduction", "value": rv, "unit": "particle-updates/s",
                                       "speedup_of_headline": value / rv}

    # ---- e2e through the reference-facing C-ABI call (cupso_run), host buffers ----
    e2e = None
    if world == 1:
        sw.close()  # cupso_run owns its own device swarm (cfg5: 2 x 52 GB double-buffered)
        e2e_secs = []
        for k in range(1 + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = engine.run(p, f, cp.rng_key(seed), cp.exec_options(device=local))
            e2e_secs.append(time.perf_counter() - t0)
        e2e_secs = e2e_secs[1:]
        h2d = C.sizeof(cp._lib.cupso_params) + 8  # params + seed; the swarm is initialised on device
        d2h = T * (8 + 4 + 8 + 8) + (16 + 8 * d) + 16  # trace, particle, admitted, async key; gbest record; initial
        e2e = {"value": n_total * T * len(e2e_secs) / sum(e2e_secs), "unit": "particle-updates/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "cupso_run via find_engine(...).run (init_swarm + T iterations + result D2H; "
                       "device swarm reused across calls of the same shape)",
               "final_gbest_fit": r.gbest_fit}
    else:
        # N > 1: the shard handle API end to end (init_swarm + NCCL gbest exchange +
        # T iterations + trace/gbest D2H), wall clock, max over ranks
        e2e_secs = []
        for k in range(1 + args.steps):
            barrier()
            t0 = time.perf_counter()
            sw.init()
            sw.step(engine.variant, T)
            sw.trace()
            sw.gbest()
            e2e_secs.append(time.perf_counter() - t0)
        t = torch.tensor([sum(e2e_secs[1:])], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e = {"value": n_total * T * args.steps / float(t.item()), "unit": "particle-updates/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": T * (8 + 4 + 8 + 8) + 16 + 8 * d,
               "path": ("Swarm API per rank (independent replicas)" if replicas else
                        "Swarm shard API per rank: init (with NCCL adopt)") + " + step + trace + gbest; max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_leg(fitness, min(n_per_rank, 1 << 24), d)
        except Exception as e:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": "particle-updates/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": "particle-updates/sec", "value": value, "unit": "particle-updates/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * dev_secs / K,
            "higher_is_better": True, "scaling": "strong" if args.workload == "cfg5" else "weak", "vs_baseline": None,
            "dtype": "f32" if f32 else "f64",
            "data": "synthetic (Philox-initialised swarm, reference make_params defaults)",
            "config": {"workload": desc, "fitness": fitness, "particles_total": n_total,
                       "particles_per_gpu": count, "dims": d, "iterations_per_step": T,
                       "variant": variant_name, "parallelism": f"replicas{world} (independent swarms, seeds 1..{world})" if replicas
                       else f"dp{world} (particle shards)",
                       "sync_grid_blocks": grid,
                       "l2": "flushed (512 MiB write) before every step; within a step the swarm stays resident as in a real run"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * K, "final_gbest_fit": gb.fit,
            **extra,
        }
        print(json.dumps(line), flush=True)
    sw.close()
    if pg:
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
