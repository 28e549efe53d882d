"""Warp-stall samples of one ncu --set full capture, attributed to SASS opcodes.

    ncu -i <rep> --page source --csv --print-source sass > src.csv
    python tools/ncu_stalls.py src.csv

Prints the kernel's stall-reason totals and, per opcode class, its share of the
samples, its share of executed instructions and its top stall reasons.
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "(Not" not in h]
    tot, execs = collections.Counter(), collections.Counter()
    byop = collections.defaultdict(collections.Counter)
    for r in data:
        if len(r) < len(hdr) or not r[ix["Source"]].strip():
            continue
        toks = r[ix["Source"]].strip().split()
        op = (toks[1] if toks[0].startswith("@") else toks[0]).rstrip(";")
        base = "IMAD.WIDE" if op.startswith("IMAD.WIDE") else op.split(".")[0]
        execs[base] += int(r[ix["Instructions Executed"]] or 0)
        for s in stalls:
            v = int(r[ix[s]] or 0)
            tot[s] += v
            byop[base][s] += v
    T, E = sum(tot.values()), sum(execs.values())
    print(f"{rows[0][1][:110]}\nwarp-state samples: {T}")
    for s, v in tot.most_common():
        if v:
            print(f"  {s:26s} {v:8d} {v / T:6.3f}")
    print("\nopcode       samples  executed  top stall reasons (share of the opcode's samples)")
    for op, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:16]:
        t = sum(c.values())
        if t:
            top = ", ".join(f"{k[6:]}={v / t:.2f}" for k, v in c.most_common(4))
            print(f"  {op:10s} {t / T:7.3f} {execs[op] / E:9.3f}  {top}")


if __name__ == "__main__":
    main(sys.argv[1])
