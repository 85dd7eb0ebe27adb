"""Round-trip accuracy of the REFERENCE arithmetic (the bit-identical oracle port) on the
bench's seeded inputs, to set the GPU path's per-slot errors against (dev tool, CPU only).

  python tools/reference_accuracy.py 64 128 256  > profiles/r01_reference_accuracy.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import so3_oracle as O  # noqa: E402


def seeded(b: int) -> np.ndarray:   # bench.py seeded_coefficients(b, seed=b)
    rng = np.random.default_rng(b)
    C = O.n_coeffs(b)
    return rng.standard_normal(C) + 1j * rng.standard_normal(C)


out = []
workers = os.cpu_count() or 1
for b in [int(x) for x in sys.argv[1:]] or [64, 128]:
    c = seeded(b)
    t0 = time.time()
    g = O.ifsoft(c, b, workers=workers)
    back = O.fsoft(g, b, workers=workers)
    d = np.abs(back - c)
    nz = np.abs(c) > 0
    rec = {"bandwidth": b, "roundtrip_max_abs": float(d.max()),
           "roundtrip_max_rel_per_slot": float((d[nz] / np.abs(c[nz])).max()),
           "roundtrip_max_rel_of_max": float(d.max() / np.abs(c).max()),
           "min_abs_coefficient": float(np.abs(c).min()), "seconds": time.time() - t0, "workers": workers}
    print(json.dumps(rec), flush=True)
    out.append(rec)
