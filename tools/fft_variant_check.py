"""Dev check: an FFT pass variant knob against the plain two-pass kernels, bit for bit, both
directions.  usage: fft_variant_check.py KNOB B [B ...]   (KNOB=1 vs KNOB=0)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1808_00896_b200 as so3

knob = sys.argv[1]
for b in map(int, sys.argv[2:]):
    n = 2 * b
    plan = so3.make_plan(b)
    g = torch.randn(n ** 3, dtype=torch.complex128, device="cuda")
    res = {}
    for v in (0, 1):
        plan.set_knob(knob, v)
        spec = torch.zeros_like(g)
        so3.fft_analysis(plan, g, spec)
        grid = torch.zeros_like(g)
        so3.fft_synthesis(plan, g, grid)
        torch.cuda.synchronize()
        res[v] = (spec, grid)
        del spec, grid
    fe = torch.equal(torch.view_as_real(res[0][0]), torch.view_as_real(res[1][0]))
    ie = torch.equal(torch.view_as_real(res[0][1]), torch.view_as_real(res[1][1]))
    print(f"B={b} {knob}: forward bit-identical {fe}, inverse bit-identical {ie}", flush=True)
    if not (fe and ie):
        d = (res[0][0] - res[1][0]).abs().view(n, n, n)
        print("forward max diff", float(d.max()), "nonzero rows", int((d.amax(dim=2) > 0).sum()))
        d = (res[0][1] - res[1][1]).abs()
        print("inverse max diff", float(d.max()))
    del res
    torch.cuda.empty_cache()
