"""Turn this round's ncu captures + launch list into the committed profiles/.

    python tools/make_profiles.py r01
writes profiles/<r>_ncu_summary.txt, profiles/ncu_summary_<r>.json (read by
bench.py for roofline.traffic) and profiles/<r>_launches_cfg2.txt.
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import METRICS, raw, to_bytes  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

# capture -> (workload, variant, iterations covered by the captured launch(es), particles scale to the workload, desc)
# A capture may hold several launches (all passes of a short k_spec run): metrics are summed over them and
# the JSON carries per-iteration figures next to the per-launch average.
CAPTURES = {
    "cfg2_spec": ("cfg2", "cuda-sync", 64, 1.0,
                  "k_spec<cubic,1> speculative pass, 2^20 x d=1, one launch = one 64-iteration pass"),
    "cfg2_sync": ("cfg2", "cuda-sync-resident", 200, 1.0,
                  "k_sync_res<cubic,1> SMEM-resident persistent, 2^20 x d=1, one launch = 200 iterations"),
    "cfg2_reduction_step": ("cfg2", "cuda-reduction", 1, 1.0, "k_classic_step<cubic,tree> (reduction phase 1), one iteration"),
    "cfg2_reduction_fold": ("cfg2", "cuda-reduction-fold", 1, 1.0, "k_classic_fold<tree> (reduction phase 2), one iteration"),
    "cfg3_async": ("cfg3", "cuda-async", 100, 1.0, "k_async_reg<cubic,1> (registers, K=32), 2^24 x d=1, one launch = 100 iterations"),
    "cfg4_spec": ("cfg4", "cuda-sync", 60, 1.0,
                  "k_spec_split<rastrigin,8x4> (4 lanes x 8 axes per particle), 2^20 x d=32, every pass of a 60-iteration run summed"),
    "cfg4_f32": ("cfg4", "cuda-sync-f32", 60, 1.0,
                 "k_spec32_split<rastrigin,8x4> (FP32 engine), 2^20 x d=32, every pass of a 60-iteration run summed"),
    "cfg4_wave": ("cfg4", "cuda-sync-wave", 1, 1.0, "k_wave<rastrigin> (cos_pso), 2^20 x d=32, one iteration (iteration 5)"),
    "cfg5proxy_spec": ("cfg5", "cuda-sync", 20, 16.0,
                       "k_spec<sphere,8>, 2^24 x d=8 proxy of 2^28 (x16), every pass of a 20-iteration run summed"),
    "cfg5proxy_wave": ("cfg5", "cuda-sync-wave", 1, 16.0, "k_wave<sphere>, 2^24 x d=8 proxy of 2^28 (x16 per launch), iteration 5"),
}


def main(tag, dest=None):
    """dest: directory for the summaries (default profiles/; on the GPU box use gpurun_out/... so they travel)."""
    pdir = dest or os.path.join(ROOT, "profiles")
    lines = [f"# {tag}: ncu --set full --clock-control none captures (B200, sm_100a); one launch each",
             "# per-launch numbers are cold-cache and serialised under replay; compare shares, not absolutes", ""]
    js = {}
    for key, (wl, var, iters, scale, desc) in CAPTURES.items():
        rep = os.path.join(OUT, f"{tag}_{key}.ncu-rep")
        if not os.path.exists(rep):
            continue
        rows = raw(rep)
        tot = {"rd": 0.0, "wr": 0.0, "inst": 0.0, "ms": 0.0}
        for d in rows:
            lines.append(f"== {key}: {desc}")
            lines.append(f"   kernel: {d['kernel'][:110]}")
            for m in METRICS:
                if m in d:
                    lines.append(f"   {m:62s} {d[m][0]} {d[m][1]}")
            lines.append(f"   top stalls (warps per issue-active): {d['top_stalls']}")
            lines.append("")
            tot["rd"] += to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else 0.0
            tot["wr"] += to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else 0.0
            tot["inst"] += float(d["smsp__inst_executed.sum"][0].replace(",", "")) if "smsp__inst_executed.sum" in d else 0.0
            dur = d.get("gpu__time_duration.sum")
            if dur:
                v = float(dur[0].replace(",", ""))
                tot["ms"] += v * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(dur[1], 1.0)
        if rows:
            n = len(rows)
            js.setdefault(wl, {})[var] = {
                "launches_captured": n, "iters_covered": iters,
                "dram_bytes_per_iter": (tot["rd"] + tot["wr"]) * scale / iters,
                "warp_inst_per_iter": tot["inst"] * scale / iters,
                "dram_bytes_per_launch": (tot["rd"] + tot["wr"]) * scale / n, "iters_per_launch": iters / n,
                "warp_inst_per_launch": tot["inst"] * scale / n,
                "dram_read": tot["rd"] * scale, "dram_write": tot["wr"] * scale,
                "duration_ms_total": tot["ms"], "capture": f"gpurun_out/{tag}_{key}.ncu-rep", "desc": desc}
            if n > 1:
                lines.append(f"-- {key}: {n} launches, {iters} iterations: dram {(tot['rd'] + tot['wr']) / iters / 1e6:.1f} MB/iter, "
                             f"{tot['inst'] / iters / 1e6:.1f} M warp-inst/iter, {tot['ms']:.3f} ms total (serialised replay)")
                lines.append("")
    os.makedirs(pdir, exist_ok=True)
    with open(os.path.join(pdir, f"{tag}_ncu_summary.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(pdir, f"ncu_summary_{tag}.json"), "w") as fh:
        json.dump(js, fh, indent=1)
    # launch list of the default bench command
    lp = os.path.join(OUT, "launches_cfg2.csv")
    if os.path.exists(lp):
        rows = list(csv.reader(open(lp)))
        i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
        hdr = rows[i]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[i + 1:]:
            if len(r) <= vi:
                continue
            try:
                v = float(r[vi].replace(",", ""))
            except ValueError:
                continue
            name = r[ki].split("(")[0]
            a = agg.setdefault(name, [0, 0.0])
            a[0] += 1
            a[1] += v
        tot = sum(a[1] for a in agg.values())
        out = ["# launch list of `python bench.py --steps 3 --warmup 3 --no-cpu` under",
               "# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold: shares only)",
               f"# {'launches':>8} {'total_us':>12} {'share':>6}  kernel"]
        for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            out.append(f"  {c:8d} {t / 1e3:12.1f} {100 * t / tot:5.1f}%  {n}")
        with open(os.path.join(pdir, f"{tag}_launches_cfg2.txt"), "w") as fh:
            fh.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", sys.argv[2] if len(sys.argv) > 2 else None)
