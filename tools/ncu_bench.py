"""ncu counters of the EXACT schedule bench.py times (run on the GPU box).

    python tools/ncu_bench.py <tag> [workload[:variant] ...]

For each workload: one timed step of `bench.py --steps 1 --warmup 0` (the same
T, the same device-side pass schedule as a bench step) under

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
                  smsp__inst_executed.sum,gpu__time_duration.sum
        --clock-control none -k regex:<the workload's pass kernels>

(single-pass counters: no kernel replay, so the device-side schedule runs as
in the bench), summed over the step's launches into
gpurun_out/ncu_bench_<tag>.json (copy to profiles/ncu_bench_<tag>.json; read
by bench.py for roofline.traffic / the issue roof) plus the raw CSV.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,gpu__time_duration.sum,"
           "sm__pipe_fmaheavy_cycles_active.sum,sm__pipe_fp64_cycles_active.sum,sm__pipe_alu_cycles_active.sum,"
           "sm__cycles_active.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active")
KERNELS = {  # variant -> kernel regex of its timed launches
    "cuda-sync": "k_spec|k_wave|k_sync|k_propose|k_commit",
    "cuda-async": "k_async",
    "cuda-sync-f32": "k_spec32|k_wave32",
    "cuda-reduction": "k_classic",
    "cuda-queue-lock": "k_classic",
}
DEFAULT_VARIANT = {"cfg2": "cuda-sync", "cfg3": "cuda-async", "cfg4": "cuda-sync", "cfg5": "cuda-sync"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "Kinst": 1e3, "Minst": 1e6,
         "Ginst": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1, "ms": 1}


def capture(tag, workload, variant):
    csv_path = os.path.join(OUT, f"ncu_bench_{tag}_{workload}_{variant}.csv")
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--replay-mode", "application", "-k", f"regex:{KERNELS[variant]}", "--csv",
           "--log-file", csv_path, sys.executable, os.path.join(ROOT, "bench.py"), "--workload", workload,
           "--variant", variant, "--steps", "1", "--warmup", "0", "--no-cpu", "--no-baseline-kernel", "--no-e2e",
           "--no-strong", "--no-others"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    if r.returncode != 0:
        print(r.stdout[-2000:], r.stderr[-2000:])
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    return csv_path, line


def summarise(csv_path):
    launches = {}
    with open(csv_path) as fh:
        rows = [r for r in csv.reader(fh) if len(r) > 10]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    for r in rows[1:]:
        lid = r[ix["ID"]]
        e = launches.setdefault(lid, {"kernel": r[ix["Kernel Name"]]})
        v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1)
        e[r[ix["Metric Name"]]] = v
    return list(launches.values())


def main():
    tag = sys.argv[1]
    targets = sys.argv[2:] or list(DEFAULT_VARIANT)
    out = {}
    for t in targets:
        wl, _, var = t.partition(":")
        var = var or DEFAULT_VARIANT[wl]
        csv_path, line = capture(tag, wl, var)
        ls = summarise(csv_path)
        # the bench step is the last `launches_per_step` launches captured (Job's
        # constructor runs none of these kernels; warm-up is 0)
        tot = {m: sum(x.get(m, 0.0) for x in ls) for m in METRICS.split(",")}
        kernels = sorted({x["kernel"].split("(")[0] for x in ls})
        T = line["config"]["iterations_per_step"]
        out.setdefault(wl, {})[var] = {
            "kernels": kernels, "launches_per_step": len(ls), "iters_per_step": T,
            "particles": line["config"]["particles_per_gpu"],
            "dram_bytes_per_step": tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"],
            "dram_read_per_step": tot["dram__bytes_read.sum"], "dram_write_per_step": tot["dram__bytes_write.sum"],
            "warp_inst_per_step": tot["smsp__inst_executed.sum"],
            "kernel_ms_per_step_ncu": tot["gpu__time_duration.sum"],
            # SM-cycles per step each pipe was busy (summed over SMs) and SM-active cycles:
            # the fma-heavy pipe runs IMAD/IMAD.WIDE (Philox), 4 cycles per IMAD.WIDE.U32
            # warp-instruction per SMSP on sm_100a (tools/micro/pipes.cu)
            "fmaheavy_cycles_per_step": tot.get("sm__pipe_fmaheavy_cycles_active.sum"),
            "fp64_cycles_per_step": tot.get("sm__pipe_fp64_cycles_active.sum"),
            "alu_cycles_per_step": tot.get("sm__pipe_alu_cycles_active.sum"),
            "sm_active_cycles_per_step": tot.get("sm__cycles_active.sum"),
            "fmaheavy_pct_of_active_ncu": sum(x.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", 0)
                                              * x.get("sm__cycles_active.sum", 0) for x in ls)
            / max(1.0, tot.get("sm__cycles_active.sum", 0.0)),
            "bench_ms_per_step_under_ncu": line["ms_per_step"],
            "capture": f"profiles/ncu_bench_{tag}_{wl}_{var}.csv (tools/ncu_bench.py: one bench.py step, "
                       f"--metrics {METRICS}, --clock-control none)",
        }
        e = out[wl][var]
        print(f"{wl} {var}: {e['launches_per_step']} launches, DRAM {e['dram_bytes_per_step'] / 1e6:.1f} MB/step, "
              f"{e['warp_inst_per_step'] * 32 / (e['particles'] * T):.1f} thread-inst per particle-update", flush=True)
    path = os.path.join(OUT, f"ncu_bench_{tag}.json")
    old = {}
    if os.path.exists(path):
        with open(path) as fh:
            old = json.load(fh)
    for wl, v in out.items():
        old.setdefault(wl, {}).update(v)
    with open(path, "w") as fh:
        json.dump(old, fh, indent=1)


if __name__ == "__main__":
    main()
