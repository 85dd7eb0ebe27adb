"""Streamed SOFG throughput at B=512 (row 8(f).2): a 17 GB iFSOFT grid written from the device
to a file and read back to the device through 2 x STAGING_BYTES of pinned host memory, checked
bit-exact on the device; host RSS growth reported (the reference's reader holds the 17 GB bytes
object plus a 17 GB converted copy).

    python tools/sof_stream.py [-B 512] [--dir /tmp] [--out profiles/r02_sof_stream_B512.json]
"""
import argparse
import json
import os
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_00896_b200 as so3  # noqa: E402
from paper_1808_00896_b200 import core  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("-B", type=int, default=512)
ap.add_argument("--dir", default="/tmp")
ap.add_argument("--out", default=None)
args = ap.parse_args()
b = args.B
plan = so3.make_plan(b, device="cuda:0")
rng = np.random.default_rng(b)
c = torch.from_numpy(rng.standard_normal(so3.coeff_count(b)) + 1j * rng.standard_normal(so3.coeff_count(b))).cuda()
grid = so3.ifsoft_sequential(so3.So3Coefficients(b, c), plan)
torch.cuda.synchronize()
del c
path = os.path.join(args.dir, f"so3_stream_B{b}.sofg")
nbytes = 16 * (2 * b) ** 3
rss0 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
t0 = time.perf_counter()
so3.write_samples(path, grid)
os.sync()
t_write = time.perf_counter() - t0
t0 = time.perf_counter()
back = so3.read_samples(path, device="cuda:0")
torch.cuda.synchronize()
t_read = time.perf_counter() - t0
equal = bool(torch.equal(back.data, grid.data))
rss1 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
res = {"bandwidth": b, "bytes": nbytes, "staging_bytes_per_buffer": core.STAGING_BYTES, "buffers": 2,
       "write_s": t_write, "write_GBps": nbytes / t_write / 1e9, "read_s": t_read, "read_GBps": nbytes / t_read / 1e9,
       "bit_exact": equal, "host_max_rss_growth_MB": (rss1 - rss0) / 1024.0, "file": path,
       "note": "write includes os.sync(); the read is served from the page cache where the box kept the file"}
os.unlink(path)
print(json.dumps(res))
if args.out:
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
