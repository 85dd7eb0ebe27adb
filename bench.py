#!/usr/bin/env python3
"""Benchmark: FSOFT + iFSOFT throughput on B200 (BASELINE.json metric).

One step = one iFSOFT (seeded coefficients -> samples) followed by one FSOFT
(samples -> coefficients) of one function at bandwidth B, the reference
benchmark protocol (pkg/src/so3fft/bench.py:146-209).  Each step is two
transforms; ``value`` = transforms/s of the whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--bandwidth B]
  python bench.py --impl reference ...     # CPU reference arm (oracle port, all host cores)

Rank 0 prints ONE JSON line.  Under torchrun (N > 1) the default is the
sharded pipeline: ONE transform split over the N GPUs (beta slabs for the
torus FFT, cost-balanced cluster groups for the DWT, one NCCL all-to-all per
direction; paper_1808_00896_b200/distributed.py), i.e. strong scaling;
``--mode replicas`` runs N independent single-GPU replicas instead.  The timed
region is bracketed by a barrier + synchronize and the max over ranks is
reported.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")   # reference bench.py:21-24: pin BLAS before numpy loads

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_B = 512


def coeff_count(b: int) -> int:
    return b * (4 * b * b - 1) // 3


def seeded_coefficients(b: int, seed: int) -> np.ndarray:
    """BASELINE.json configs: real and imaginary parts i.i.d. N(0,1), default_rng(seed)."""
    rng = np.random.default_rng(seed)
    c = coeff_count(b)
    return rng.standard_normal(c) + 1j * rng.standard_normal(c)


def dwt_flops(b: int) -> float:
    """Algorithmic DWT flops per transform direction: 8 * B * C(B)."""
    return 8.0 * b * coeff_count(b)


def fft_bytes(b: int) -> float:
    """Algorithmic torus-FFT bytes per direction: read + write (2B)^3 complex128 = 256 B^3."""
    return 256.0 * b ** 3


def measured_peaks() -> dict:
    peaks = {"fp64_tflops": 36.97, "fp64_source": "measured DMMA m8n8k4 burst, profiles/r01_fp64_peak.log",
             "hbm_gbs": 6553.3, "hbm_source": "fallback 6553.3 (MEASURED_PEAKS.json absent)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            mp = json.load(fh)
        if "hbm_gbs" in mp:
            peaks["hbm_gbs"] = float(mp["hbm_gbs"])
            peaks["hbm_source"] = "MEASURED_PEAKS.json hbm_gbs (measured)"
    fp = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(fp):
        with open(fp) as fh:
            peaks.update(json.load(fh))
    return peaks


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"so3_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        load = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# --------------------------------------------------------------------------- CPU baseline (oracle port)

CPU_WHOLE = os.path.join(ROOT, "profiles", "r02_cpu_whole.json")


class ReferenceSample:
    """A bounded, proportional sample of one iFSOFT + FSOFT of the reference arithmetic.

    The oracle (oracle/so3_oracle.py, bit-identical to the reference) runs its four stages
    exactly as the reference's *_parallel does (soft.py:124-173 over run_items,
    schedule.py:200-257: a fork pool per stage, fork-inherited items, dynamic batches, the
    parent-side transpose / scatter into freshly allocated outputs), but on 1/`stride` of the
    work: every stride-th beta slice for the two FFT stages and every stride-th symmetry cluster
    in (m, m') order for the two DWT stages (systematic samples with a per-step offset, so
    every cluster size is represented).  Each stage's time is scaled by its own sampling
    fraction to a whole-transform estimate.  A step is therefore ~1/stride of a transform
    pair, and the line's value = transforms_per_step / step time is consistent with its
    ms_per_step.  profiles/r02_cpu_whole.json holds WHOLE measured runs (B = 64..512 on the
    GPU box's 16 cores) that calibrate this estimate.
    """

    def __init__(self, b: int, workers: int, stride: int):
        from oracle import so3_oracle as O
        self.O, self.b, self.n, self.workers, self.stride = O, b, 2 * b, workers, max(1, stride)
        n = self.n
        O._plan(b)   # plan tables outside the timed region (reference bench.py:156-158)
        self.c = seeded_coefficients(b, b)
        self.bases = sorted(O.base_pairs(b))
        # Stage inputs and outputs are fully populated buffers, as a whole run's are.  A whole
        # run also faults in its freshly allocated outputs (three (2B)^3 arrays and one
        # coefficient array per round trip); a sample writing 1/stride of a fresh array would
        # fault in most of its (transparent huge) pages, so that first-touch cost is measured
        # here, on the output buffers' own first fill, and added unscaled.
        self.grid = np.full((n, n, n), 0.5 - 0.25j, dtype=np.complex128)
        self.spec_in = np.full((n, n, n), 0.25 + 0.5j, dtype=np.complex128)
        self.spec_out = np.empty((n, n, n), dtype=np.complex128)
        t0 = time.perf_counter()
        self.spec_out[...] = 0.0
        self.touch_grid_s = time.perf_counter() - t0
        self.cube_out = np.zeros(n ** 3, dtype=np.complex128)
        self.cube_out[...] = 0.0
        self.coef_out = np.empty(O.n_coeffs(b), dtype=np.complex128)
        t0 = time.perf_counter()
        self.coef_out[...] = 0.0
        self.touch_coef_s = time.perf_counter() - t0

    def step(self, k: int) -> dict:
        O, b, n, st = self.O, self.b, self.n, self.stride
        js = list(range(k % st, n, st))
        cl = self.bases[k % st::st]
        # the per-stage fixed cost (fork a pool of this process, start its workers, collect) is
        # paid once per stage by a whole run too: measured here, and not scaled
        p0 = time.perf_counter()
        O._pool_map(lambda i: i, range(4 * self.workers), self.workers)
        ovh = time.perf_counter() - p0
        t = {"pool_overhead_s": ovh}
        t0 = time.perf_counter()
        O.dwt_synthesis_stage(self.c, b, self.workers, clusters=cl, out=self.spec_out)
        t1 = time.perf_counter()
        O.fft_synthesis_stage(self.spec_in, b, self.workers, slices=js, out=self.cube_out)
        t2 = time.perf_counter()
        O.fft_analysis_stage(self.grid, b, self.workers, slices=js, out=self.spec_out)
        t3 = time.perf_counter()
        O.dwt_analysis_stage(self.spec_in, b, self.workers, clusters=cl, out=self.coef_out)
        t4 = time.perf_counter()
        fs, fc = len(js) / n, len(cl) / len(self.bases)
        t["sample_s"] = t4 - t0
        t["stages_sample_s"] = {"dwt_synthesis": t1 - t0, "fft_synthesis": t2 - t1, "fft_analysis": t3 - t2,
                                "dwt_analysis": t4 - t3}
        scale = lambda dt, f: ovh + max(dt - ovh, 0.0) / f
        t["first_touch_s"] = {"grid": self.touch_grid_s, "coefficients": self.touch_coef_s}
        t["inverse_s"] = scale(t1 - t0, fc) + scale(t2 - t1, fs) + 2 * self.touch_grid_s
        t["forward_s"] = scale(t3 - t2, fs) + scale(t4 - t3, fc) + self.touch_grid_s + self.touch_coef_s
        t["transforms_per_s"] = 2.0 / (t["inverse_s"] + t["forward_s"])
        t["transforms_per_step"] = t["transforms_per_s"] * t["sample_s"]
        t["sample"] = (f"B={b}: {len(js)}/{n} beta slices and {len(cl)}/{len(self.bases)} symmetry clusters "
                       f"(systematic, offset {k % st}) through all four stages of iFSOFT + FSOFT on a "
                       f"{self.workers}-process fork pool; stage times less the measured pool start-up scaled by their sampling fractions, plus the measured first-touch cost of the whole run's fresh outputs")
        return t


def committed_parity(b: int) -> dict:
    """Per-direction parity of this bandwidth against the reference arithmetic, measured by
    tools/parity_full.py (oracle/parity.py) and committed under profiles/; summarised here so the
    bench line carries it (the bench does not re-run the 4-minute oracle)."""
    path = os.path.join(ROOT, "profiles", f"r02_parity_B{b}.json")
    if not os.path.exists(path):
        return {}
    with open(path) as fh:
        r = json.load(fh)
    truth = lambda k: {"gpu_err": r[k]["truth"]["gpu_max_err"], "reference_err": r[k]["truth"]["reference_max_err"]}
    return {"per_direction_vs_reference": {
        "source": f"profiles/r02_parity_B{b}.json",
        "inverse_rel_of_max": r["inverse"]["rel_of_max"],
        "forward_rel_of_max": r["forward"]["rel_of_max"], "forward_per_slot": r["forward"]["per_slot"],
        "vs_long_double": {"inverse": truth("inverse"), "dwt_synthesis": truth("inverse_dwt_stage"),
                           "dwt_analysis": truth("forward_dwt_stage"), "fft_analysis": truth("forward_fft_stage")},
        "round_trip_gpu": {"max_abs": r["round_trip_gpu"]["max_abs"], "per_slot": r["round_trip_gpu"]["per_slot"],
                           "rms_abs": r["round_trip_compare"]["gpu_rms_abs"]},
        "round_trip_reference": {"max_abs": r["round_trip_reference"]["max_abs"],
                                 "per_slot": r["round_trip_reference"]["per_slot"],
                                 "rms_abs": r["round_trip_compare"]["reference_rms_abs"]}}}


def cpu_whole_measured(b: int):
    """Whole measured runs of the reference arithmetic (profiles/r02_cpu_whole.json)."""
    if not os.path.exists(CPU_WHOLE):
        return None
    with open(CPU_WHOLE) as fh:
        rec = json.load(fh)
    run = rec["runs"].get(f"B{b}")
    if run is None:
        return None
    return {"transforms_per_s": run["transforms_per_s"], "inverse_s": run["inverse_s"],
            "forward_s": run["forward_s"], "cores": run["cores"], "host": rec["host"],
            "source": "profiles/r02_cpu_whole.json (tools/parity_full.py)"}


def run_reference_arm(args, rank: int, world: int) -> None:
    """--impl reference: the reference arithmetic (oracle port) on all host cores, rank 0 only.
    Each warm-up or timed step is one bounded ReferenceSample step."""
    if rank != 0:
        return
    from oracle import so3_oracle as O
    b = args.bandwidth
    workers = O.default_workers()
    smp = ReferenceSample(b, workers, args.cpu_stride)
    for k in range(args.warmup):
        smp.step(k)
    steps = [smp.step(args.warmup + k) for k in range(args.steps)]
    total_s = sum(r["sample_s"] for r in steps)
    per_step = sum(r["transforms_per_step"] for r in steps) / len(steps)
    v = per_step * len(steps) / total_s
    whole = cpu_whole_measured(b)
    cpu = {"value": v, "unit": "transforms/s", "cores": workers, "kind": "port", "sample": steps[-1]["sample"],
           "extrapolated": True, "transforms_per_step": per_step,
           "est_seconds": {"inverse": statistics.mean(r["inverse_s"] for r in steps),
                           "forward": statistics.mean(r["forward_s"] for r in steps)}}
    if whole:
        cpu["measured_whole"] = whole
        cpu["estimate_over_measured"] = v / whole["transforms_per_s"]
    line = {
        "impl": "reference", "metric": metric_name(b), "value": v, "unit": "transforms/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total_s / len(steps), "transforms_per_step": per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(b, world),
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm

def metric_name(b: int, batch: int = 1) -> str:
    return f"FSOFT+iFSOFT transforms/sec (B={b}{f', batch {batch}' if batch > 1 else ''}, fp64)"


def workload_config(b: int, world: int, batch: int = 1) -> dict:
    if batch == 1:
        what = f"B={b} single function, complex128, coefficients N(0,1) seed={b}"
    else:
        what = f"B={b}, batch of {batch} functions, coefficients N(0,1) seeds 32000+f scaled by 1/(1+l)"
    return {"workload": f"BASELINE configs: {what}; iFSOFT then FSOFT", "bandwidth": b, "functions_per_step": batch,
            "grid": f"{batch} x {2 * b}^3 complex128 ({batch * 16 * (2 * b) ** 3 / 1e9:.2f} GB)",
            "coefficients": coeff_count(b) * batch,
            "l2": "inputs larger than L2 (126 MB)" if batch * 16 * (2 * b) ** 3 > 126e6 else "L2 flushed between steps",
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


def l2_flush(torch, buf):
    buf.add_(1.0)


def run_gpu_arm(args, rank: int, world: int, dist) -> None:
    import torch
    import paper_1808_00896_b200 as so3

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    b = args.bandwidth
    n = 2 * b
    C = coeff_count(b)
    F = args.batch
    plan = so3.make_plan(b, device=dev, batch=F)
    plan.set_dwt_variant(args.dwt_variant)
    stream = torch.cuda.current_stream(dev)

    if F == 1:
        host_c = seeded_coefficients(b, b)
    else:   # BASELINE configs[1]: seeds 32000 + f, scaled by 1/(1+l)
        scale = 1.0 / (1.0 + np.repeat(np.arange(b), [(2 * l + 1) ** 2 for l in range(b)]))
        host_c = np.concatenate([seeded_coefficients(b, 32000 + f) * scale for f in range(F)])
    coeffs = torch.from_numpy(host_c).to(dev)
    grid = torch.empty(F * n ** 3, dtype=torch.complex128, device=dev)
    spec = torch.empty(F * n ** 3, dtype=torch.complex128, device=dev)
    out = torch.empty(F * C, dtype=torch.complex128, device=dev)
    flush = None
    if 16 * F * n ** 3 <= 126e6 * 2:
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > L2

    n_ev = 5
    def step(evs=None):
        if flush is not None:
            l2_flush(torch, flush)
        if evs is not None:
            evs[0].record(stream)
        so3.dwt_synthesis(plan, coeffs, spec)          # K3
        if evs is not None:
            evs[1].record(stream)
        so3.fft_synthesis(plan, spec, grid)            # K4a + K4b
        if evs is not None:
            evs[2].record(stream)
        so3.fft_analysis(plan, grid, spec)             # K1a + K1b
        if evs is not None:
            evs[3].record(stream)
        so3.dwt_analysis(plan, spec, out)              # K2
        if evs is not None:
            evs[4].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(local).start() if rank == 0 else None
    time.sleep(0.3 if clocks else 0)
    # stage-resolved pass (events between stages on the launching stream)
    stage_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        step(stage_ev[k])
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    clk = clocks.stop() if clocks else None
    stage_names = ["dwt_synthesis", "fft_synthesis", "fft_analysis", "dwt_analysis"]
    stage_ms = {nm: statistics.mean(stage_ev[k][i].elapsed_time(stage_ev[k][i + 1]) for k in range(args.steps))
                for i, nm in enumerate(stage_names)}
    if dist is not None:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = world * F * 2.0 * 1000.0 / ms_step

    # parity of the measured output: round trip recovers the seeded coefficients
    got = out.cpu().numpy()
    diff = np.abs(got - host_c)
    rt_abs = float(diff.max())
    rt_rel = float((diff / np.abs(host_c)).max())
    rt_rel_max = float(diff.max() / np.abs(host_c).max())

    # end to end through the public API (the e2e contract): every step copies its input (the
    # coefficients) in from pinned host memory and reads its result (the coefficients after the
    # round trip) back into pinned host memory; the intermediate grid stays on the device, as a GPU
    # caller keeps it (ifsoft/fsoft on device tensors).  The variant that also moves the 17 GB grid
    # through host memory (numpy in, numpy out) is reported beside it ("grid_via_host").
    e2e = None
    if not args.no_e2e:
        h_c = torch.empty(F * C, dtype=torch.complex128, pin_memory=True)
        h_c.numpy()[:] = host_c
        h_r = torch.empty(F * C, dtype=torch.complex128, pin_memory=True)
        d_r = torch.empty(F * C, dtype=torch.complex128, device=dev)

        def e2e_step():
            c_dev = h_c.to(dev, non_blocking=True)
            if F == 1:
                g = so3.ifsoft_sequential(so3.So3Coefficients(b, c_dev), plan, out=grid)
                r = so3.fsoft_sequential(g, plan, out=d_r).data
            else:
                so3.ifsoft_batch(c_dev, plan, out=grid)
                r = so3.fsoft_batch(grid, plan, out=d_r)
            h_r.copy_(r.reshape(-1), non_blocking=True)
            stream.synchronize()   # the step's result is in host memory when the step ends

        def timed(fn, ksteps):
            fn()
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(ksteps):
                out_ = fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / ksteps
            if dist is not None:
                t = torch.tensor([ms], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            return ms, out_

        ksteps = max(1, min(args.steps, 2 * args.e2e_steps))
        e_ms, _ = timed(e2e_step, ksteps)
        serial = {"value": world * F * 2000.0 / e_ms, "unit": "transforms/s", "ms_per_step": e_ms, "steps": ksteps,
                  "roundtrip_max_abs": float(np.abs(h_r.numpy() - host_c).max()),
                  "api": "the same step, synchronised per step (no overlap between steps: the latency of one round trip)"}

        # The same steps as a stream: every step still copies ITS coefficients in from pinned host
        # memory and ITS result back to pinned host memory, but step k+1's upload and step k-1's
        # download run on two copy streams beside step k's kernels (two device buffers each way,
        # ordered by events; PCIe is full duplex).  Throughput over all steps, the last download included.
        cin, cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        d_c2 = [torch.empty(F * C, dtype=torch.complex128, device=dev) for _ in range(2)]
        d_r2 = [d_r, torch.empty(F * C, dtype=torch.complex128, device=dev)]
        h_r2 = [h_r, torch.empty(F * C, dtype=torch.complex128, pin_memory=True)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def pipelined(ksteps):
            for i in range(2):
                ev_comp[i].record(stream)
                ev_out[i].record(stream)
            for k in range(ksteps):
                i = k & 1
                with torch.cuda.stream(cin):
                    cin.wait_event(ev_comp[i])            # step k-2 no longer reads this input buffer
                    d_c2[i].copy_(h_c, non_blocking=True)
                    ev_in[i].record(cin)
                stream.wait_event(ev_in[i])
                stream.wait_event(ev_out[i])              # step k-2's result has left this output buffer
                if F == 1:
                    g = so3.ifsoft_sequential(so3.So3Coefficients(b, d_c2[i]), plan, out=grid)
                    so3.fsoft_sequential(g, plan, out=d_r2[i])
                else:
                    so3.ifsoft_batch(d_c2[i], plan, out=grid)
                    so3.fsoft_batch(grid, plan, out=d_r2[i])
                ev_comp[i].record(stream)
                with torch.cuda.stream(cout):
                    cout.wait_event(ev_comp[i])
                    h_r2[i].copy_(d_r2[i], non_blocking=True)
                    ev_out[i].record(cout)
            for i in range(2):
                stream.wait_event(ev_out[i])              # the timed region ends when every result is in host memory

        psteps = max(4, ksteps)
        pipelined(2)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for hr in h_r2:
            hr.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pipelined(psteps)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        p_ms = e0.elapsed_time(e1) / psteps
        if dist is not None:
            t = torch.tensor([p_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            p_ms = float(t.item())
        e2e = {"value": world * F * 2000.0 / p_ms, "unit": "transforms/s", "ms_per_step": p_ms,
               "h2d_bytes_per_step": 16 * F * C, "d2h_bytes_per_step": 16 * F * C, "steps": psteps,
               "roundtrip_max_abs": max(float(np.abs(hr.numpy() - host_c).max()) for hr in h_r2),
               "api": ("every step: pinned coefficients -> device, ifsoft_" + ("sequential" if F == 1 else "batch") +
                       " (device grid) -> fsoft, result -> pinned host memory; consecutive steps overlap their "
                       "copies with the kernels (two copy streams, double-buffered device coefficients)"),
               "serial": serial}
        del d_c2, d_r2, h_r2
        del h_r, d_r
        # the grid through host memory as well (numpy in, numpy out, the reference's own contract):
        # pinned numpy buffers, then the pageable arrays the reference's callers pass
        h_cn = h_c.numpy()
        h_g = torch.empty(F * n ** 3, dtype=torch.complex128, pin_memory=True).numpy()
        h_o = torch.empty(F * C, dtype=torch.complex128, pin_memory=True).numpy()

        def host_step():
            if F == 1:
                g = so3.ifsoft_sequential(so3.So3Coefficients(b, h_cn), plan, out=h_g)
                so3.fsoft_sequential(so3.So3SampleGrid(b, g.data), plan, out=h_o)
            else:
                so3.ifsoft_batch(h_cn, plan, out=h_g)
                so3.fsoft_batch(h_g, plan, out=h_o)
        ksteps = max(1, min(args.steps, args.e2e_steps))
        g_ms, _ = timed(host_step, ksteps)
        e2e["grid_via_host"] = {
            "value": world * F * 2000.0 / g_ms, "unit": "transforms/s", "ms_per_step": g_ms,
            "h2d_bytes_per_step": 16 * F * (C + n ** 3), "d2h_bytes_per_step": 16 * F * (n ** 3 + C),
            "steps": ksteps, "roundtrip_max_abs": float(np.abs(h_o - host_c).max()),
            "api": "ifsoft_sequential(So3Coefficients numpy, pinned) -> fsoft_sequential(So3SampleGrid numpy)"}
        del h_c, h_cn, h_g, h_o
        if F == 1:
            p_c = host_c.copy()

            def pageable_step():
                g = so3.ifsoft_sequential(so3.So3Coefficients(b, p_c), plan)
                return so3.fsoft_sequential(g, plan)
            p_ms, back = timed(pageable_step, 1)
            e2e["grid_via_host"]["pageable"] = {
                "value": world * 2000.0 / p_ms, "unit": "transforms/s", "ms_per_step": p_ms, "steps": 1,
                "roundtrip_max_abs": float(np.abs(np.asarray(back.data) - host_c).max()),
                "api": "ifsoft_sequential / fsoft_sequential on pageable numpy arrays (fresh outputs)"}

    if rank != 0:
        return
    peaks = measured_peaks()
    p64 = peaks["fp64_tflops"] * 1e12
    bw = peaks["hbm_gbs"] * 1e9
    fl = dwt_flops(b) * F
    by = fft_bytes(b) * F
    # DWT algorithmic bytes: the spectrum read (written) once and the coefficients written
    # (read) once; below the FP64 ridge (small B) the DWT is HBM-bound
    dwt_bytes = 16.0 * F * (n ** 3 + C)
    dwt_bound = "fp64" if fl / dwt_bytes >= p64 / bw else "hbm"
    fused = n in (16, 32, 64)   # one-pass slice FFT (fft2d_slice_tma_kernel: pair-major side by TMA)
    kernel_of = {
        "dwt_analysis": "dwt_analysis_batch_reg_kernel" if (F >= 2 and n <= 64) else "dwt_analysis_mma_cta_kernel",
        # B a multiple of 64: the segment-parallel synthesis (dwt_seg.cuh) is the library default
        "dwt_synthesis": "dwt_synthesis_batch_kernel" if (F >= 2 and n <= 64) else
                         ("dwt_synthesis_seg_kernel" if (n % 128 == 0 and n <= 1024) else "dwt_synthesis_mma_kernel"),
        # launch_fft2d / launch_fft_tma dispatch: one-pass TMA slices at 2B <= 64, TMA-fed passes
        # (rows in -> tensor store; tensor load -> rows out) at 2B in {256, 512, 1024}, else plain
        "fft_analysis": "fft2d_slice_tma_kernel" if fused else
                        ("fft_pass_tstore_kernel x2" if n in (256, 512, 1024) else "fft_pass_kernel x2"),
        "fft_synthesis": "fft2d_slice_tma_kernel" if fused else
                         ("fft_pass_tload_kernel x2" if n in (256, 512, 1024) else "fft_pass_kernel x2"),
    }
    if kernel_of["dwt_analysis"] == "dwt_analysis_mma_cta_kernel" and n % 128 == 0 and 512 < n <= 1024:
        # library default at B = 320 .. 512 (dwt_seg bit 4): persistent CTAs, two passes per cluster
        kernel_of["dwt_analysis"] = "dwt_analysis_segp_kernel (persistent, segment-parallel)"
    stages = {}
    for nm in stage_names:
        ms = stage_ms[nm]
        if nm.startswith("dwt"):
            stages[nm] = {"ms": ms, "tflops": fl / (ms * 1e-3) / 1e12, "frac_fp64": fl / (ms * 1e-3) / p64,
                          "gbs": dwt_bytes / (ms * 1e-3) / 1e9, "frac_hbm": dwt_bytes / (ms * 1e-3) / bw,
                          "bound": dwt_bound}
        else:
            stages[nm] = {"ms": ms, "gbs": by / (ms * 1e-3) / 1e9, "frac_hbm": by / (ms * 1e-3) / bw, "bound": "hbm",
                          "note": ("one pass" if fused else "two HBM passes") +
                                  "; algorithmic bytes = one read + one write of the grid"}
    # roofline of the dominant stage (longest), against the bound it sits under
    dom = max(stage_names, key=lambda k: stage_ms[k])
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get(f"B{b}" + (f"x{F}" if F > 1 else ""), {}).get(dom)
    if dom.startswith("dwt") and dwt_bound == "fp64":
        achieved = fl / (stage_ms[dom] * 1e-3) / 1e12
        roof = {"kernel": f"{dom} ({kernel_of[dom]}, DMMA)", "bound": "tensor", "pipe": "fp64 DMMA (mma.sync f64)",
                "achieved": achieved,
                "peak": peaks["fp64_tflops"], "unit": "TFLOP/s", "frac": achieved / peaks["fp64_tflops"],
                "traffic": traffic, "peak_source": peaks["fp64_source"],
                "algorithmic": f"8*B*C(B) x {F} functions = {fl:.4g} flop per launch (one transform direction)"}
    else:
        alg = dwt_bytes if dom.startswith("dwt") else by
        achieved = alg / (stage_ms[dom] * 1e-3) / 1e9
        roof = {"kernel": f"{dom} ({kernel_of[dom]})", "bound": "hbm", "achieved": achieved,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "traffic": traffic, "peak_source": peaks["hbm_source"],
                "algorithmic": (f"16*((2B)^3 + C(B)) x {F} functions = {alg:.4g} bytes per direction"
                                if dom.startswith("dwt") else
                                f"256*B^3 x {F} functions = {alg:.4g} bytes per direction (grid read + write)")}
    cpu = None
    if world == 1 and not args.no_cpu and F == 1:
        from oracle import so3_oracle as O
        r = ReferenceSample(b, O.default_workers(), args.cpu_stride).step(0)   # one bounded step
        cpu = {"value": r["transforms_per_s"], "unit": "transforms/s", "cores": O.default_workers(),
               "kind": "port", "sample": r["sample"], "extrapolated": True, "sample_s": r["sample_s"],
               "est_seconds": {"inverse": r["inverse_s"], "forward": r["forward_s"]}}
        whole = cpu_whole_measured(b)
        if whole:
            cpu["measured_whole"] = whole
            cpu["estimate_over_measured"] = r["transforms_per_s"] / whole["transforms_per_s"]
    line = {
        "metric": metric_name(b, F), "value": value, "unit": "transforms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(b, world, F),
        "fsoft_per_s": world * F * 1000.0 / (stage_ms["fft_analysis"] + stage_ms["dwt_analysis"]),
        "ifsoft_per_s": world * F * 1000.0 / (stage_ms["dwt_synthesis"] + stage_ms["fft_synthesis"]),
        "stages": stages, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        # our kernels per step: per direction one DWT launch and one (fused slice) or two FFT
        # passes; the L2 flush between steps is a torch fill, not counted
        "gpu_launches": (2 + 2 * (1 if fused else 2)) * args.steps,
        "clocks": clk,
        "parity": dict({"roundtrip_max_abs": rt_abs, "roundtrip_max_rel_per_slot": rt_rel,
                        "roundtrip_max_rel_of_max": rt_rel_max}, **committed_parity(b) if F == 1 else {}),
        "peaks": peaks,
    }
    print(json.dumps(line), flush=True)


def run_sharded_arm(args, rank: int, world: int, dist) -> None:
    """One B transform pair split over `world` GPUs (strong scaling)."""
    import torch
    from paper_1808_00896_b200.distributed import NativeShardBackend, ShardedSO3

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    b = args.bandwidth
    n = 2 * b
    C = coeff_count(b)
    chunks = args.chunks if args.chunks else (4 if (b >= 128 and world > 1) else 1)
    backend = NativeShardBackend(b, world, rank, device=dev, chunks=chunks)
    sh = ShardedSO3(b, rank, world, backend)
    m = sh.map
    J = m.J
    stream = torch.cuda.current_stream(dev)
    host_c = seeded_coefficients(b, b)
    coeffs = torch.from_numpy(host_c).to(dev)
    # staged step (one chunk): one exchange buffer (layout A, then layout B with the own block)
    # reused across steps; the pipelined step allocates through ShardedSO3 (torch's caching
    # allocator reuses them)
    if chunks == 1:
        ex = backend.empty(m.exchange_rows(rank) * J)
        lay_b = ex[m.b_chunk(rank, 0)[0]:]
        slab = backend.empty(n * J * n)
    out = backend.zeros(C)

    result = {}

    def step_staged(evs=None):
        rec = (lambda i: evs[i].record(stream)) if evs is not None else (lambda i: None)
        rec(0)
        backend.dwt_synthesis(coeffs, lay_b)
        rec(1)
        for w in sh._exchange(ex, 0, forward=False):   # other ranks' blocks only (none for one rank)
            w.wait()
        rec(2)
        backend.fft_synthesis(ex, slab)
        rec(3)
        backend.fft_analysis(slab, ex)
        rec(4)
        for w in sh._exchange(ex, 0, forward=True):
            w.wait()
        rec(5)
        backend.dwt_analysis(lay_b, out)
        rec(6)
        result["coeffs"] = out

    def step_pipelined(evs=None):
        # chunked exchange overlapped with the DWT (ShardedSO3.ifsoft / fsoft)
        rec = (lambda i: evs[i].record(stream)) if evs is not None else (lambda i: None)
        rec(0)
        sl = sh.ifsoft(coeffs)
        rec(1)
        result["coeffs"] = sh.fsoft(sl, out=out)   # own slots rewritten every step; the rest stay zero
        rec(2)

    step = step_staged if chunks == 1 else step_pipelined
    nev = 7 if chunks == 1 else 3

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local).start() if rank == 0 else None
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t1.record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    ms_total = t0.elapsed_time(t1)
    clk = clocks.stop() if clocks else None
    names = (["dwt_synthesis", "all_to_all_inverse", "fft_synthesis", "fft_analysis", "all_to_all_forward",
              "dwt_analysis"] if chunks == 1 else ["ifsoft_pipelined", "fsoft_pipelined"])
    stage_ms = {nm: statistics.mean(evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(args.steps))
                for i, nm in enumerate(names)}
    if dist is not None:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    # parity: gathered coefficients of the measured step == seeded input (round trip)
    full = sh.gather_coefficients(result["coeffs"].clone())

    # e2e through the sharded public API: every step moves this rank's input in from pinned host
    # memory (the coefficients) and its result back (its own coefficient slots, in a full-length
    # array); the beta slab stays on the device.  The variant that also moves the slab through host
    # memory is reported beside it ("slab_via_host").
    e2e = None
    if not args.no_e2e:
        h_c = torch.empty(C, dtype=torch.complex128, pin_memory=True)
        h_c.copy_(torch.from_numpy(host_c))
        h_slab = torch.empty(n * J * n, dtype=torch.complex128, pin_memory=True)
        h_out = torch.empty(C, dtype=torch.complex128, pin_memory=True)

        def e2e_step():
            c_dev = h_c.to(dev, non_blocking=True)
            h_out.copy_(sh.fsoft(sh.ifsoft(c_dev)), non_blocking=True)
            stream.synchronize()

        def slab_step():
            c_dev = h_c.to(dev, non_blocking=True)
            h_slab.copy_(sh.ifsoft(c_dev), non_blocking=True)
            s_dev = h_slab.to(dev, non_blocking=True)
            h_out.copy_(sh.fsoft(s_dev), non_blocking=True)
            stream.synchronize()

        def timed(fn):
            fn()
            torch.cuda.synchronize(dev)
            if dist is not None:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.e2e_steps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / args.e2e_steps
            if dist is not None:
                t = torch.tensor([ms], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            return ms

        e_ms = timed(e2e_step)
        s_ms = timed(slab_step)
        e2e = {"value": 2.0 * 1000.0 / e_ms, "unit": "transforms/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": 16 * C, "d2h_bytes_per_step": 16 * C, "steps": args.e2e_steps,
               "api": "pinned coefficients H2D -> ShardedSO3.ifsoft (device slab) -> ShardedSO3.fsoft -> own "
                      "coefficient slots D2H (per rank), synchronised per step",
               "slab_via_host": {"value": 2.0 * 1000.0 / s_ms, "unit": "transforms/s", "ms_per_step": s_ms,
                                 "h2d_bytes_per_step": 16 * (C + n * J * n),
                                 "d2h_bytes_per_step": 16 * (C + n * J * n),
                                 "api": "ShardedSO3.ifsoft(coefficients H2D) -> slab D2H; slab H2D -> "
                                        "ShardedSO3.fsoft -> own coefficient slots D2H (per rank, pinned)"}}
    got = full.cpu().numpy()
    diff = np.abs(got - host_c)
    if rank != 0:
        return
    peaks = measured_peaks()
    fl = dwt_flops(b) / world   # this rank's share of the DWT (cost-balanced)
    a2a_bytes = 16 * (m.layout_a_rows() - m.pairs[rank]) * J   # bytes this rank sends to peers, forward
    if chunks == 1:
        dom = max(("dwt_analysis", "dwt_synthesis"), key=lambda k: stage_ms[k])
        achieved = fl / (stage_ms[dom] * 1e-3) / 1e12
        roof = {"kernel": f"{dom} (rank 0, DMMA)", "bound": "tensor", "pipe": "fp64 DMMA (mma.sync f64)",
                "achieved": achieved,
                "peak": peaks["fp64_tflops"], "unit": "TFLOP/s", "frac": achieved / peaks["fp64_tflops"],
                "traffic": None, "algorithmic": "8*B*C(B)/world flop per rank and direction"}
        a2a = {"bytes_per_rank_per_direction": a2a_bytes,
               "GBps_forward": a2a_bytes / (stage_ms["all_to_all_forward"] * 1e-3) / 1e9,
               "GBps_inverse": a2a_bytes / (stage_ms["all_to_all_inverse"] * 1e-3) / 1e9}
    else:
        # stages overlap: the roofline is the whole direction's DWT work over its pipelined time
        dom = max(names, key=lambda k: stage_ms[k])
        achieved = fl / (stage_ms[dom] * 1e-3) / 1e12
        roof = {"kernel": f"{dom} (rank 0: FFT + chunked all_to_all overlapped with the DMMA DWT)",
                "bound": "tensor", "pipe": "fp64 DMMA (mma.sync f64)", "achieved": achieved,
                "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["fp64_tflops"], "traffic": None,
                "algorithmic": "8*B*C(B)/world flop per rank and direction, over the whole direction"}
        a2a = {"bytes_per_rank_per_direction": a2a_bytes, "chunks": chunks}
    line = {
        "metric": metric_name(b), "value": 2.0 * 1000.0 / ms_step, "unit": "transforms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(b, world), parallelism=f"sharded x{world}: beta slabs (J={J}) + "
                       f"cluster groups, all_to_all per direction in {chunks} chunk(s) overlapped with the DWT"),
        "stages_rank0_ms": stage_ms,
        "roofline": roof,
        "all_to_all": a2a,
        "cpu_baseline": None, "e2e": e2e, "gpu_launches": (4 + 2 * chunks) * args.steps,
        "clocks": clk,
        "parity": {"roundtrip_max_abs": float(diff.max()),
                   "roundtrip_max_rel_of_max": float(diff.max() / np.abs(host_c).max())},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-exec this command as N ranks (one
    process per GPU) through torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def launch_check(rank: int, world: int) -> None:
    """--launch-check: gloo rendezvous of all ranks (no GPU work); rank 0 prints who reported."""
    import torch
    import torch.distributed as tdist
    tdist.init_process_group("gloo")
    seen = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    tdist.all_gather(seen, torch.tensor([rank], dtype=torch.int64))
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks": [int(t.item()) for t in seen],
                          "backend": tdist.get_backend()}), flush=True)
    tdist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--bandwidth", "-B", type=int, default=DEFAULT_B)
    ap.add_argument("--batch", type=int, default=1, help="functions per step (BASELINE configs[1]: B=32, 64)")
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--chunks", type=int, default=0,
                    help="sharded mode: exchange chunks (0 = auto: 4 for B >= 128 on several GPUs)")
    ap.add_argument("--dwt-variant", choices=("mma", "simt"), default="mma")
    ap.add_argument("--mode", choices=("auto", "single", "sharded", "replicas"), default="auto",
                    help="auto: single GPU at N=1, sharded (one transform over N GPUs) at N>1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-stride", type=int, default=0,
                    help="CPU sample: every k-th beta slice and cluster per step (0 = auto: ~1/32 of a transform "
                         "pair at B=512, whole transforms at B <= 128)")
    ap.add_argument("--launch-check", action="store_true",
                    help="rendezvous only (gloo): every rank reports in, rank 0 prints the ranks it saw")
    args = ap.parse_args()
    if args.cpu_stride <= 0:
        args.cpu_stride = {512: 32, 256: 4}.get(args.bandwidth, 1)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the timing rules require >= 3 warm-up steps", file=sys.stderr)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
                 f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus")
    if args.launch_check:
        launch_check(rank, world)
        return
    dist = None
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    mode = args.mode if args.mode != "auto" else ("single" if world == 1 else "sharded")
    # under torchrun the sharded arm always goes through NCCL, also with one rank (self exchange)
    if world > 1 or (mode == "sharded" and "MASTER_ADDR" in os.environ):
        import torch
        import torch.distributed as tdist
        # communicator init lines (ranks, nRanks, NVLS/P2P transport) on stderr, so the driver can
        # see N ranks while stdout keeps the one JSON line
        for k, v in (("NCCL_DEBUG", "INFO"), ("NCCL_DEBUG_SUBSYS", "INIT"), ("NCCL_DEBUG_FILE", "/dev/stderr")):
            os.environ.setdefault(k, v)
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        tdist.init_process_group("nccl")
        dist = tdist
    if mode == "sharded":
        run_sharded_arm(args, rank, world, dist)
    else:
        run_gpu_arm(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
