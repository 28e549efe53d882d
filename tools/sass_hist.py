"""SASS opcode histogram of a kernel's hot loop (the iteration loop).

    python tools/sass_hist.py <lib.so> <mangled-name-substring> [units-per-trip] [--all]

Dumps the function with cuobjdump -sass, finds the innermost backward-branch
loop holding most of the Philox multiplies (the iteration loop), and counts
opcodes inside it, grouped into classes (Philox IMAD/LOP3, FP64, loads,
constant loads, spills, shuffles, ...). units-per-trip divides the counts to
per-particle-axis figures (k_spec<cubic,1,NP=4>: 4; k_spec_split<.,8,G>: 8).
"""
import collections
import re
import subprocess
import sys

LINE = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);")
CLASSES = [
    ("philox: IMAD.WIDE", lambda o: o.startswith("IMAD.WIDE") or o.startswith("UIMAD.WIDE")),
    ("philox: LOP3", lambda o: o.startswith("LOP3") or o.startswith("ULOP3")),
    ("IMAD/IADD/other int", lambda o: o.split(".")[0] in ("IMAD", "IADD3", "IADD", "UIADD3", "UIMAD", "SHF", "USHF",
                                                          "LEA", "ISETP", "UISETP", "IABS", "SEL", "USEL", "PRMT",
                                                          "VIADD", "IMNMX", "MOV", "UMOV", "IMAD.MOV", "R2UR",
                                                          "S2R", "S2UR", "FLO", "POPC", "PLOP3", "P2R", "R2P",
                                                          "VIMNMX", "LOP", "ULEA")),
    ("FP64 (DFMA/DMUL/DADD/DSETP/DMNMX)", lambda o: o[0] == "D" and o.split(".")[0] in
     ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DSET")),
    ("I2F/F2I/F2F conversions", lambda o: o.split(".")[0] in ("I2F", "F2I", "F2F", "I2FP", "F2IP", "FRND")),
    ("FP32", lambda o: o.split(".")[0] in ("FFMA", "FMUL", "FADD", "FSETP", "FSEL", "FMNMX", "MUFU", "FSET")),
    ("LDC (constant reloads)", lambda o: o.startswith("LDC") and not o.startswith("LDCU")),
    ("LDCU (uniform constant)", lambda o: o.startswith("LDCU")),
    ("spill LDL/STL", lambda o: o.split(".")[0] in ("LDL", "STL")),
    ("global LDG/STG", lambda o: o.split(".")[0] in ("LDG", "STG", "LD", "ST", "ATOMG", "RED", "ATOM")),
    ("shared LDS/STS", lambda o: o.split(".")[0] in ("LDS", "STS", "ATOMS")),
    ("SHFL / vote", lambda o: o.split(".")[0] in ("SHFL", "VOTE", "VOTEU", "MATCH")),
    ("control (BRA/BSSY/BSYNC/WARPSYNC/...)", lambda o: o.split(".")[0] in ("BRA", "BSSY", "BSYNC", "WARPSYNC",
                                                                            "EXIT", "CALL", "RET", "BAR", "NOP",
                                                                            "YIELD", "BREAK", "DEPBAR")),
]


def dump(lib, name):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs, cur, buf = {}, None, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                funcs[cur] = buf
            cur, buf = m.group(1), []
        elif cur:
            buf.append(line)
    if cur:
        funcs[cur] = buf
    hits = [f for f in funcs if name in f]
    if not hits:
        raise SystemExit(f"no function matching {name}")
    f = min(hits, key=len)
    ins = []
    for line in funcs[f]:
        m = LINE.search(line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    return f, ins


def hot_loop(ins):
    """The innermost backward-branch loop that still holds >= 75 % of the
    function's Philox multiplies (the iteration loop, not the particle loop)."""
    loops = []
    for addr, op, rest in ins:
        if op.startswith("BRA") and "DIV" not in op:
            m = re.search(r"0x([0-9a-f]+)", rest)
            if m and int(m.group(1), 16) < addr:
                tgt = int(m.group(1), 16)
                loops.append((tgt, addr, sum(1 for a, o, _ in ins if tgt <= a <= addr and "IMAD.WIDE" in o)))
    top = max(c for _, _, c in loops)
    return min(((lo, hi) for lo, hi, c in loops if c >= 0.75 * top), key=lambda r: r[1] - r[0])


def classify(op):
    for name, pred in CLASSES:
        if pred(op):
            return name
    return "other"


def main():
    lib, name = sys.argv[1], sys.argv[2]
    units = float(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("-") else 1.0
    fn, ins = dump(lib, name)
    lo, hi = (0, 1 << 62) if "--all" in sys.argv else hot_loop(ins)
    body = [op for a, op, _ in ins if lo <= a <= hi]
    cls = collections.Counter(classify(op) for op in body)
    ops = collections.Counter(op for op in body)
    print(f"function: {fn}")
    print(f"hot loop: 0x{lo:x}..0x{hi:x}, {len(body)} instructions per trip, {units:g} units per trip "
          f"-> {len(body) / units:.1f} per unit")
    for k, v in cls.most_common():
        print(f"  {k:40s} {v:6d}  {v / units:8.2f} per unit")
    print("top opcodes:", ", ".join(f"{k} {v}" for k, v in ops.most_common(18)))


if __name__ == "__main__":
    main()
