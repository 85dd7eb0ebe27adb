"""Dev check: FFT stage outputs under two knob settings, bit for bit, both directions.
usage: fft_variant_check.py "k=v,k=v" "k=v" B [B ...]   (first setting is the reference)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1808_00896_b200 as so3

def knobs(spec):
    return [kv.split("=") for kv in spec.split(",") if kv]

ref, alt = knobs(sys.argv[1]), knobs(sys.argv[2])
for b in map(int, sys.argv[3:]):
    n = 2 * b
    plan = so3.make_plan(b)
    g = torch.randn(n ** 3, dtype=torch.complex128, device="cuda")
    res = []
    for ks in (ref, alt):
        for k, v in ref:
            plan.set_knob(k, 0 if k != "fft_tma" else 1)
        for k, v in ks:
            plan.set_knob(k, int(v))
        spec = torch.zeros_like(g)
        so3.fft_analysis(plan, g, spec)
        grid = torch.zeros_like(g)
        so3.fft_synthesis(plan, g, grid)
        torch.cuda.synchronize()
        res.append((spec, grid))
    fe = torch.equal(torch.view_as_real(res[0][0]), torch.view_as_real(res[1][0]))
    ie = torch.equal(torch.view_as_real(res[0][1]), torch.view_as_real(res[1][1]))
    print(f"B={b} {sys.argv[2]} vs {sys.argv[1]}: forward bit-identical {fe}, inverse bit-identical {ie}", flush=True)
    del res
    torch.cuda.empty_cache()
