"""Segment-parallel DWT (dwt_seg.cuh) against the dwt_mma.cuh kernels on the same plan: per-stage
difference (relative to max) and median stage times.  usage: seg_check.py B [B ...]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1808_00896_b200 as so3


SEG = int(os.environ.get('SEG', '3'))


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


for b in [int(x) for x in (sys.argv[1:] or [64, 128, 256])]:
    n, C = 2 * b, so3.coeff_count(b)
    plan = so3.make_plan(b)
    for kv in filter(None, os.environ.get('SO3_KNOBS', '').split(',')):
        k, v = kv.split('='); plan.set_knob(k, int(v))
    rng = np.random.default_rng(b)
    coef = torch.from_numpy(rng.standard_normal(C) + 1j * rng.standard_normal(C)).cuda()
    spec = {s: torch.zeros(n ** 3, dtype=torch.complex128, device="cuda") for s in (0, 1)}
    out = {s: torch.zeros(C, dtype=torch.complex128, device="cuda") for s in (0, 1)}
    res = {"B": b, "plan_GB": round(plan.device_bytes / 1e9, 2) if hasattr(plan, "device_bytes") else None}
    for s in (0, 1):
        plan.set_knob("dwt_seg", SEG * s)
        res[f"syn_ms_seg{s}"] = round(timed(lambda: so3.dwt_synthesis(plan, coef, spec[s])), 4)
    # the analysis of the SAME spectrum (the old kernels' synthesis) under both settings
    for s in (0, 1):
        plan.set_knob("dwt_seg", SEG * s)
        res[f"ana_ms_seg{s}"] = round(timed(lambda: so3.dwt_analysis(plan, spec[0], out[s])), 4)
    d_syn = (spec[1] - spec[0]).abs().max().item() / spec[0].abs().max().item()
    d_ana = (out[1] - out[0]).abs().max().item() / out[0].abs().max().item()
    nz = int((spec[1] != 0).sum().item()), int((spec[0] != 0).sum().item())
    res.update(syn_rel=d_syn, ana_rel=d_ana, nonzero=nz, finite=bool(torch.isfinite(torch.view_as_real(out[1])).all().item()))
    print(json.dumps(res), flush=True)
    del plan, spec, out, coef
    torch.cuda.empty_cache()
