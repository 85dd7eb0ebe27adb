"""Profiling driver (dev tool): W+K device-resident iFSOFT->FSOFT steps at bandwidth B, no CPU work."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1808_00896_b200 as so3

b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 2 * b
C = b * (4 * b * b - 1) // 3
F = int(os.environ.get("PROF_BATCH", "1"))
plan = so3.make_plan(b, batch=F)
for kv in filter(None, os.environ.get("SO3_KNOBS", "").split(",")):
    k, v = kv.split("="); plan.set_knob(k, int(v))
rng = np.random.default_rng(b)
c = torch.from_numpy(rng.standard_normal(F * C) + 1j * rng.standard_normal(F * C)).cuda()
grid = torch.empty(F * n ** 3, dtype=torch.complex128, device="cuda")
spec = torch.empty_like(grid)
out = torch.empty_like(c)
for _ in range(steps):
    so3.dwt_synthesis(plan, c, spec)
    so3.fft_synthesis(plan, spec, grid)
    so3.fft_analysis(plan, grid, spec)
    so3.dwt_analysis(plan, spec, out)
torch.cuda.synchronize()
print("max abs round trip", float((out - c).abs().max()))
