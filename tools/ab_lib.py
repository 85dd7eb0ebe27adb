"""A/B of the DWT stages between two builds of the library in ONE process (dev tool): each .so
gets its own plan; stages alternate, median of reps.  usage: ab_lib.py B old.so [new.so]"""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

b = int(sys.argv[1])
paths = sys.argv[2:] if os.environ.get("AB_ONLY") else [sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else
         os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1808_00896_b200",
                      "libso3fft_b200.so")]
n = 2 * b
C = b * (4 * b * b - 1) // 3
torch.empty(1, device="cuda")
spec = torch.randn(n ** 3, dtype=torch.complex128, device="cuda")
coef = torch.randn(C, dtype=torch.complex128, device="cuda")
out_s = torch.empty_like(spec)
out_c = torch.empty_like(coef)
libs, plans = [], []
for p in paths:
    lib = ctypes.CDLL(p)
    lib.so3_plan_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    lib.so3_dwt_analysis.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 2 + [ctypes.c_void_p]
    lib.so3_dwt_synthesis.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 2 + [ctypes.c_void_p]
    lib.so3_cluster_count.restype = ctypes.c_int64
    h = ctypes.c_void_p()
    assert lib.so3_plan_create(b, 1, ctypes.byref(h)) == 0
    for kv in filter(None, os.environ.get("SO3_KNOBS", "").split(",")):   # per-plan knobs for every library
        k, v = kv.split("=")
        assert lib.so3_plan_set_knob(h, k.encode(), int(v)) == 0, kv
    libs.append(lib)
    plans.append(h)
ncl = libs[0].so3_cluster_count(b)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr())
res = {p: {"ana": [], "syn": []} for p in paths}
for rep in range(int(os.environ.get("AB_REPS", "9"))):
    for lib, h, p in zip(libs, plans, paths):
        for name, fn in (("ana", lambda: lib.so3_dwt_analysis(h, P(spec), P(out_c), 0, ncl, st)),
                         ("syn", lambda: lib.so3_dwt_synthesis(h, P(coef), P(out_s), 0, ncl, st))):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            assert fn() == 0
            e1.record()
            torch.cuda.synchronize()
            if rep:
                res[p][name].append(e0.elapsed_time(e1))
for p in paths:
    print(os.path.basename(p), {k: round(statistics.median(v), 3) for k, v in res[p].items()})
