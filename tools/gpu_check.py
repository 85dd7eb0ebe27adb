"""Quick GPU parity probe (dev tool): our CUDA path vs the oracle on seeded inputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1808_00896_b200 as so3
from oracle import so3_oracle as O

def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

for b in [int(x) for x in (sys.argv[1:] or [1, 2, 3, 4, 5, 6, 8, 16, 32, 64])]:
    rng = np.random.default_rng(b)
    C = O.n_coeffs(b)
    c = rng.standard_normal(C) + 1j * rng.standard_normal(C)
    plan = so3.make_plan(b)
    plan.set_dwt_variant(os.environ.get('SO3_DWT', 'mma'))
    for kv in filter(None, os.environ.get('SO3_KNOBS', '').split(',')):
        k, v = kv.split('='); plan.set_knob(k, int(v))
    t0 = time.time()
    g = so3.ifsoft_sequential(so3.So3Coefficients(b, c), plan).data
    f = so3.fsoft_sequential(so3.So3SampleGrid(b, g), plan).data
    tg = time.time() - t0
    g_ref = O.ifsoft(c, b)
    f_ref = O.fsoft(g_ref, b)
    f2 = so3.fsoft_sequential(so3.So3SampleGrid(b, g_ref), plan).data
    ea, er = O.error_metrics(f_ref, f2)
    print(f"B={b}: inv rel {rel(g, g_ref):.2e}  fwd rel {rel(f2, f_ref):.2e} (per-slot {er:.2e})  roundtrip {O.error_metrics(c, f)}  gpu {tg:.3f}s", flush=True)
