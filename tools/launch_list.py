"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv python bench.py ...
    python tools/launch_list.py L.csv "<the bench command>" > profiles/<tag>_launches_cfg2.txt

ncu serialises launches and runs them cold, so the per-kernel SHARES are what
compare with the bench's own timing, not the absolute times.
"""
import csv
import sys


def main(path, label):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = {}
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        except ValueError:
            continue
        a = agg.setdefault(r[ki].split("(")[0], [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"# launch list of `{label}` under")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold: shares only)")
    print(f"# {'launches':>8} {'total_us':>12} {'share':>6}  kernel")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:8d} {t:12.1f} {100 * t / tot:5.1f}%  {n}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "?")
