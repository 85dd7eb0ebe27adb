"""Per-kernel SASS instruction families of the built library -> JSON (dev tool).
    python tools/sass_histogram.py > profiles/r02_sass_histogram.json"""
import collections, json, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1808_00896_b200", "libso3fft_b200.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
FAM = ["DMMA", "DFMA", "DADD", "DMUL", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "LDS", "STS", "LDG", "STG", "SHFL", "BAR", "MUFU"]
res, cur = {}, None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = res.setdefault(name, collections.Counter())
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Za-z0-9_.]+)", line)
    if m and cur is not None:
        op = m.group(1)
        cur["total"] += 1
        for f in FAM:
            if op.startswith(f):
                cur[op if f in ("DMMA", "UTMALDG", "UTMASTG") else f] += 1
print(json.dumps({k: dict(v) for k, v in sorted(res.items())}, indent=1))
