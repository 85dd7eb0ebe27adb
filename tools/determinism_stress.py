"""Dev check: repeated B=512 iFSOFT -> FSOFT steps must be bit-identical (per-cluster counters of
the split analysis re-arm themselves; TMA passes, row-table loops and reductions are
deterministic).  usage: determinism_stress.py [B] [repeats]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1808_00896_b200 as so3

b = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
plan = so3.make_plan(b)
rng = np.random.default_rng(b)
C = so3.coeff_count(b)
c = torch.from_numpy(rng.standard_normal(C) + 1j * rng.standard_normal(C)).cuda()
ref_g = ref_f = None
for r in range(reps):
    g = so3.ifsoft_sequential(so3.So3Coefficients(b, c), plan).data
    f = so3.fsoft_sequential(so3.So3SampleGrid(b, g), plan).data
    torch.cuda.synchronize()
    if ref_g is None:
        ref_g, ref_f = g.clone(), f.clone()
        print("round trip max abs", float((f - c).abs().max()), flush=True)
    else:
        assert torch.equal(g, ref_g) and torch.equal(f, ref_f), f"repeat {r} differs"
    del g, f
print(f"B={b}: {reps} repeats bit-identical")
