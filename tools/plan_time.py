"""Plan construction time (dev tool): make_plan(B) wall time, cold and warm, per bandwidth."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1808_00896_b200 as so3

torch.cuda.init(); torch.empty(1, device="cuda")
for b in [int(x) for x in (sys.argv[1:] or [32, 128, 256, 512])]:
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        p = so3.make_plan(b)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"B={b} rep={rep} make_plan {t1 - t0:.3f} s  device_bytes {p.device_bytes / 1e9:.2f} GB", flush=True)
        p.release()
