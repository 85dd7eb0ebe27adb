"""Can the HBM-bound torus FFT and the FP64-bound DWT share the GPU?  B=512, existing kernels:
time each stage alone, then both issued on two streams (either order, either priority).

    python tools/overlap_probe.py [-B 512]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1808_00896_b200 as so3  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("-B", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--pads", type=lambda t: [int(x) for x in t.split(",")], default=[0, 60, 100, 130])
ap.add_argument("--dwt-pads", type=lambda t: [int(x) for x in t.split(",")], default=[])
ap.add_argument("--persist", type=lambda t: [int(x) for x in t.split(",")], default=[])
ap.add_argument("--carveout", type=int, default=-1, help="preferred smem carveout of every big kernel (-1: default)")
args = ap.parse_args()
b = args.B
n = 2 * b
dev = torch.device("cuda", 0)
plan = so3.make_plan(b, device=dev)
plan.set_knob("carveout", args.carveout)
g = torch.randn(n ** 3, dtype=torch.complex128, device=dev)
spec_a = torch.randn(n ** 3, dtype=torch.complex128, device=dev)
spec_b = torch.empty_like(spec_a)
coef = torch.empty(so3.coeff_count(b), dtype=torch.complex128, device=dev)
grid2 = torch.empty_like(g)


def timed(fn):
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(args.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def on(stream, fn):
    def run():
        with torch.cuda.stream(stream):
            fn()
    return run


lo = torch.cuda.Stream(device=dev, priority=0)
hi = torch.cuda.Stream(device=dev, priority=-1)
res = {}
fwd_fft = lambda: so3.fft_analysis(plan, g, spec_b)
fwd_dwt = lambda: so3.dwt_analysis(plan, spec_a, coef)
inv_dwt = lambda: so3.dwt_synthesis(plan, coef, spec_b)
inv_fft = lambda: so3.fft_synthesis(plan, spec_a, grid2)
for dpad in args.dwt_pads:
    plan.set_knob("dwt_pad", dpad)
    res[f"dwt_pad{dpad}_analysis"] = timed(fwd_dwt)
    res[f"dwt_pad{dpad}_synthesis"] = timed(inv_dwt)
plan.set_knob("dwt_pad", 0)
for name, f in (("fft_analysis", fwd_fft), ("dwt_analysis", fwd_dwt), ("dwt_synthesis", inv_dwt),
                ("fft_synthesis", inv_fft)):
    res[name] = timed(f)


def pair(first, second, s1, s2):
    def run():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            first()
        with torch.cuda.stream(s2):
            second()
        e1, e2 = torch.cuda.Event(), torch.cuda.Event()
        e1.record(s1)
        e2.record(s2)
        cur.wait_event(e1)
        cur.wait_event(e2)
    return run


for pad in args.pads:
    plan.set_knob("fft_pad", pad)
    for tag, (dwt, fft) in {"forward": (fwd_dwt, fwd_fft), "inverse": (inv_dwt, inv_fft)}.items():
        res[f"pad{pad}_{tag}_fft_alone"] = timed(fft)
        res[f"pad{pad}_{tag}_serial"] = timed(lambda: (dwt(), fft()))
        res[f"pad{pad}_{tag}_dwt_first_fft_hi"] = timed(pair(dwt, fft, lo, hi))
        res[f"pad{pad}_{tag}_fft_first_fft_hi"] = timed(pair(fft, dwt, hi, lo))
        res[f"pad{pad}_{tag}_dwt_first_same_prio"] = timed(pair(dwt, fft, lo, torch.cuda.Stream(device=dev)))
    print(json.dumps({k: v for k, v in res.items() if k.startswith(f"pad{pad}_")}), flush=True)
plan.set_knob("fft_pad", 0)
ref_fwd = torch.empty_like(spec_b)
so3.fft_analysis(plan, g, ref_fwd)
ref_inv = torch.empty_like(grid2)
so3.fft_synthesis(plan, spec_a, ref_inv)
for pc in args.persist:
    plan.set_knob("fft_persist", pc)
    so3.fft_analysis(plan, g, spec_b)
    so3.fft_synthesis(plan, spec_a, grid2)
    torch.cuda.synchronize()
    res[f"persist{pc}_bit_identical"] = bool(torch.equal(spec_b, ref_fwd)) and bool(torch.equal(grid2, ref_inv))
    for tag, (dwt, fft) in {"forward": (fwd_dwt, fwd_fft), "inverse": (inv_dwt, inv_fft)}.items():
        res[f"persist{pc}_{tag}_fft_alone"] = timed(fft)
        res[f"persist{pc}_{tag}_serial"] = timed(lambda: (dwt(), fft()))
        res[f"persist{pc}_{tag}_fft_first_fft_hi"] = timed(pair(fft, dwt, hi, lo))
        res[f"persist{pc}_{tag}_fft_first_same"] = timed(pair(fft, dwt, lo, torch.cuda.Stream(device=dev)))
    print(json.dumps({k: v for k, v in res.items() if k.startswith(f"persist{pc}_")}), flush=True)
plan.set_knob("fft_persist", 0)
print(json.dumps(res, indent=1))
