"""Time one rank's sharded DWT stages (dev tool): so3_shard_dwt_* of rank 0 of G at bandwidth B."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1808_00896_b200 as so3
from paper_1808_00896_b200.distributed import NativeShardBackend, ShardMap

b, world = int(sys.argv[1]), int(sys.argv[2])
m = ShardMap(b, world)
be = NativeShardBackend(b, world, 0)
for kv in sys.argv[3:]:   # knobs, e.g. fft_tab_loop=0
    k, v = kv.split("=")
    so3._native.check(so3._native.lib().so3_plan_set_knob(be.handle, k.encode(), int(v)), "set_knob")
C = so3.coeff_count(b)
rng = np.random.default_rng(1)
coef = torch.from_numpy(rng.standard_normal(C) + 1j * rng.standard_normal(C)).cuda()
send = be.empty(m.layout_b_rows(0) * m.J)
out = be.zeros(C)
for name, fn in (("dwt_synthesis", lambda: be.dwt_synthesis(coef, send)), ("dwt_analysis", lambda: be.dwt_analysis(send, out))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); [fn() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
    print(f"B={b} G={world} rank0 {name}: {e0.elapsed_time(e1) / 3:.3f} ms")
n, J = 2 * b, m.J
slab = torch.from_numpy(rng.standard_normal(n * J * n) + 1j * rng.standard_normal(n * J * n)).cuda()
ex = be.empty(m.exchange_rows(0) * J)   # layout A, then layout B with the own block
out_slab = be.empty(n * J * n)
for name, fn in (("fft_analysis", lambda: be.fft_analysis(slab, ex)), ("fft_synthesis", lambda: be.fft_synthesis(ex, out_slab))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); [fn() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
    print(f"B={b} G={world} rank0 {name}: {e0.elapsed_time(e1) / 3:.3f} ms")
