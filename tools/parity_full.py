"""Per-direction parity at one bandwidth (oracle/parity.py protocol) -> JSON.

    python tools/parity_full.py -B 512 --out profiles/r02_parity_B512.json

Runs the oracle (bit-identical to the reference arithmetic) on every host core with the
reference's fork-pool scheme, so the oracle stage times it records are also a MEASURED whole
CPU run of the reference arithmetic at that bandwidth (bench.py reads them for cpu_baseline).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1808_00896_b200 as so3  # noqa: E402
from oracle import so3_oracle as O  # noqa: E402
from oracle.parity import run_parity  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("-B", type=int, required=True)
ap.add_argument("--workers", type=int, default=O.default_workers())
ap.add_argument("--out", required=True)
args = ap.parse_args()
b = args.B
slices = sorted(set([0, b // 3, b - 1, 2 * b - 1]))
clusters = [(0, 0), (1, 0), (b // 2, 0), (b - 1, 0), (b // 3, b // 3), (b - 1, b - 1),
            (b // 2, b // 5), (b - 1, b - 2), ((3 * b) // 4, (2 * b) // 3)]
clusters = [c for c in dict.fromkeys(clusters) if c[0] < b and c[1] <= c[0]]
t0 = time.time()
res = run_parity(b, so3, torch, workers=args.workers, truth_slices=slices, truth_clusters=clusters,
                 log=lambda s: print(s, flush=True))
res["wall_s"] = time.time() - t0
res["host_cores"] = os.cpu_count()
res["gpu"] = torch.cuda.get_device_name(0)
with open(args.out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: res[k] for k in ("inverse", "forward", "round_trip_gpu", "round_trip_reference",
                                        "oracle_inverse_s", "oracle_forward_s")}, default=str)[:3000])
