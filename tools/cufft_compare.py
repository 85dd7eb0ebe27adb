"""Comparison only (north_star: cuFFT is timed as a comparison, never used on the path):
cuFFT (torch.fft) on the same two torus-FFT passes as our K1a/K1b at bandwidth B."""
import sys, json
import torch
b = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = 2 * b
x = torch.randn(n, n, n, dtype=torch.complex128, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
res = {"B": b}
res["cufft_rows_k_ms"] = t(lambda: torch.fft.fft(x, dim=2))          # contiguous axis, like K1a (no transpose)
res["cufft_cols_i_ms"] = t(lambda: torch.fft.fft(x, dim=0))          # stride n^2 axis, like K1b
res["cufft_2d_ms"] = t(lambda: torch.fft.fft2(x, dim=(0, 2)))        # the whole torus stage
res["copy_ms"] = t(lambda: x.clone())
byt = 2 * 16 * n ** 3
for k in list(res):
    if k.endswith("_ms"):
        res[k.replace("_ms", "_TBps")] = byt / (res[k] * 1e-3) / 1e12
print(json.dumps(res))
