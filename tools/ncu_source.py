"""Aggregate an ncu source page (SASS) into regions: samples per instruction kind and the
hottest instructions (dev tool).  usage: ncu_source.py report.ncu-rep [kernel-regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')
for blk in blocks[1:2 if len(sys.argv) < 3 else None]:
    lines = blk.split("\n")
    name = lines[0][:100]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    data = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(int(r[idx["# Samples"]]) for r in data) or 1
    print(name, "total samples", tot, "instructions", len(data))
    # cumulative profile: position vs samples, in 20 chunks
    kinds = {}
    for r in data:
        op = r[idx["Source"]].split()[0] if r[idx["Source"]].split() else "?"
        if op.startswith("@"): op = r[idx["Source"]].split()[1]
        kinds[op.split(".")[0]] = kinds.get(op.split(".")[0], 0) + int(r[idx["# Samples"]])
    print("by opcode:", {k: round(100 * v / tot, 1) for k, v in sorted(kinds.items(), key=lambda x: -x[1])[:14]})
    stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    top = sorted(range(len(data)), key=lambda i: -int(data[i][idx["# Samples"]]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]
    for i in sorted(top):
        r = data[i]
        st = sorted(((int(r[idx[c]]), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"{i:5d} {100 * int(r[idx['# Samples']]) / tot:5.1f}%  exec {r[idx['Instructions Executed']]:>10}  {r[idx['Source']].strip()[:70]:70s} {st}")
