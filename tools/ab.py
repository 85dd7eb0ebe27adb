"""A/B timing of kernel configurations in ONE process (dev tool): alternating repetitions of
each stage under each knob setting, median ms.  usage: ab.py B 'name=v,name=v' 'name=v' ..."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1808_00896_b200 as so3

b = int(sys.argv[1])
configs = [dict(kv.split("=") for kv in c.split(",")) if c else {} for c in sys.argv[2:]] or [{}]
n = 2 * b
C = so3.coeff_count(b)
F = int(os.environ.get("AB_BATCH", "1"))
plan = so3.make_plan(b, batch=F)
rng = np.random.default_rng(b)
coef = torch.from_numpy(rng.standard_normal(F * C) + 1j * rng.standard_normal(F * C)).cuda()
grid = torch.empty(F * n ** 3, dtype=torch.complex128, device="cuda")
spec = torch.empty_like(grid)
out = torch.empty_like(coef)
stages = {
    "dwt_synthesis": lambda: so3.dwt_synthesis(plan, coef, spec),
    "fft_synthesis": lambda: so3.fft_synthesis(plan, spec, grid),
    "fft_analysis": lambda: so3.fft_analysis(plan, grid, spec),
    "dwt_analysis": lambda: so3.dwt_analysis(plan, spec, out),
}
res = {i: {s: [] for s in stages} for i in range(len(configs))}
defaults = { "dwt_variant": 0, "syn_jw": 0, "ana_split": 1, "fft_xb": 0, "dwt_batch": 1, "fft_fused": 1, "fft_tma": 1, "fft_bulkin": 1, "fft_bulkout": -1}
for rep in range(int(os.environ.get("AB_REPS", "7"))):
    for i, cfg in enumerate(configs):
        for k, v in defaults.items():
            plan.set_knob(k, int(cfg.get(k, v)))
        for s, fn in stages.items():
            fn(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            if rep > 0:
                res[i][s].append(e0.elapsed_time(e1))
for i, cfg in enumerate(configs):
    print(json.dumps({"B": b, "batch": F, "config": cfg, **{s: round(statistics.median(v), 4) for s, v in res[i].items()}}))
