"""Small transforms that exercise every kernel family, for compute-sanitizer (memcheck, racecheck,
synccheck -- one tool per run):

  B=16  fused one-pass slices (TMA 4-D box), batched DWT kernels (batch 4), direct route
  B=64  fused slices, MMA DWT (JW=32), SOF device streaming
  B=128 TMA-fed two-pass FFT (2B=256: tensor stores / loads, bulk rows), MMA DWT (JW=64)
  B=256 split analysis (ana_split=2: two CTAs per cluster, partial sums, arrival counters),
        synthesis JW=64 4-warp CTAs
  B=128 sharded row-table passes and chunked DWT, 2 emulated ranks

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_00896_b200 as so3  # noqa: E402


def coeffs(b, seed, batch=1):
    rng = np.random.default_rng(seed)
    c = so3.coeff_count(b) * batch
    return torch.from_numpy(rng.standard_normal(c) + 1j * rng.standard_normal(c)).cuda()


def round_trip(b, **knobs):
    plan = so3.make_plan(b)
    for k, v in knobs.items():
        plan.set_knob(k, v)
    c = coeffs(b, b)
    g = so3.ifsoft_sequential(so3.So3Coefficients(b, c), plan)
    back = so3.fsoft_sequential(g, plan).data
    torch.cuda.synchronize()
    err = float((back - c).abs().max())
    print(f"B={b} {knobs or ''}: round trip {err:.2e}", flush=True)
    assert err < 1e-10
    return g


round_trip(16)
plan = so3.make_plan(16, batch=4)
c4 = coeffs(16, 1, batch=4).view(4, -1)
back = so3.fsoft_batch(so3.ifsoft_batch(c4, plan), plan)
assert float((back - c4).abs().max()) < 1e-10
g = so3.ifsoft_direct(so3.So3Coefficients(4, coeffs(4, 4)))
g64 = round_trip(64)
with tempfile.TemporaryDirectory() as d:
    so3.write_samples(os.path.join(d, "g.sofg"), g64)
    assert torch.equal(so3.read_samples(os.path.join(d, "g.sofg"), device="cuda").data, g64.data)
round_trip(128)
round_trip(256, ana_split=2)
# sharded kernels (row-table FFT passes, chunked DWT), 2 emulated ranks in one process
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_sharded import emulate  # noqa: E402
b = 128
n = 2 * b
c = coeffs(b, 7)
grid = so3.ifsoft_sequential(so3.So3Coefficients(b, c), so3.make_plan(b)).data
out, back = emulate(b, 2, grid, c, chunks=2)
assert float((out - c).abs().max()) < 1e-10 and float((back - grid).abs().max()) < 1e-9
print("sanitize run complete", flush=True)
