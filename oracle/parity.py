"""Per-direction parity of the CUDA path against the oracle, with an extended-precision
attribution of the differences -- TEST INFRASTRUCTURE ONLY.

Imported by tests/test_gpu_parity_large.py and tools/parity_full.py (never by the product
package).  It follows SURVEY.md 8(d)'s protocol:

* inverse parity: the same seeded coefficients (seed = B) into the GPU iFSOFT and the oracle
  iFSOFT (bit-identical to the reference's ifsoft_parallel, soft.py:152-173);
* forward parity: the ORACLE's iFSOFT grid, bit for bit, into the GPU FSOFT and the oracle FSOFT
  (soft.py:124-149);
* round trips, GPU and oracle, as a third, separate check;

and splits each direction into its two stages, feeding the GPU stage the oracle's own input of
that stage (the oracle spectrum into the GPU DWT analysis and FFT synthesis), so a stage
difference cannot hide behind the other stage.  Every difference is then attributed: for
sampled beta slices and clusters (including the clusters of the worst per-slot coefficients)
oracle/extended.py gives long-double values, and the GPU's and the reference's fp64 errors
against them are reported side by side.

Metrics are the reference's error_metrics (bench.py:122-131): max |d| and the per-slot
max |d| / |ref|, plus max |d| / max |ref|.
"""

from __future__ import annotations

import time

import numpy as np

from . import extended as E
from . import so3_oracle as O


def _t_metrics(got, ref, chunk: int = 1 << 26) -> dict:
    """error_metrics on device tensors (ref != 0 for the per-slot form), in chunks so a 17 GB
    grid needs no full-size temporaries."""
    dmax = amax = pmax = 0.0
    for s in range(0, ref.numel(), chunk):
        g, r = got[s:s + chunk], ref[s:s + chunk]
        d = (g - r).abs()
        a = r.abs()
        dmax = max(dmax, float(d.max()))
        amax = max(amax, float(a.max()))
        nz = a > 0
        if bool(nz.any()):
            pmax = max(pmax, float((d[nz] / a[nz]).max()))
    return {"max_abs": dmax, "max_ref": amax, "rel_of_max": dmax / amax if amax else 0.0, "per_slot": pmax}


def _zero_nyquist(x, n: int, b: int) -> None:
    """Rows m' = B or m = B of a pair-major [m'][m][j] spectrum: never read by the DWT."""
    v = x.view(n, n, n)
    v[b].zero_()
    v[:, b].zero_()


def _slot_lmm(b: int, slots: np.ndarray) -> list[tuple[int, int, int]]:
    starts = np.array([l * (4 * l * l - 1) // 3 for l in range(b + 1)], dtype=np.int64)
    out = []
    for s in np.asarray(slots, dtype=np.int64):
        l = int(np.searchsorted(starts, s, side="right") - 1)
        r = int(s - starts[l])
        out.append((l, r // (2 * l + 1) - l, r % (2 * l + 1) - l))
    return out


def _breakdown(torch, b: int, got, ref, degree) -> dict:
    """Per-slot errors by degree band and by |ref| decade (coefficient vectors on the device)."""
    d = (got - ref).abs()
    a = ref.abs()
    per = d / a
    bands = []
    edges = sorted(set([0] + [int(round(b * k / 8)) for k in range(1, 8)] + [b]))
    for lo, hi in zip(edges[:-1], edges[1:]):
        sel = (degree >= lo) & (degree < hi)
        if int(sel.sum()) == 0:
            continue
        bands.append({"l": [lo, hi - 1], "slots": int(sel.sum()), "max_abs": float(d[sel].max()),
                      "rms_abs": float(d[sel].pow(2).mean().sqrt()), "per_slot": float(per[sel].max()),
                      "min_abs_ref": float(a[sel].min())})
    decades = []
    for e in range(-8, 2):
        sel = (a >= 10.0 ** e) & (a < 10.0 ** (e + 1))
        k = int(sel.sum())
        if k == 0:
            continue
        decades.append({"abs_ref": [10.0 ** e, 10.0 ** (e + 1)], "slots": k, "max_abs": float(d[sel].max()),
                        "per_slot": float(per[sel].max())})
    top = torch.topk(per, 5).indices.cpu().numpy()
    worst = [{"slot": int(s), "l": l, "m": m, "mp": mp, "abs_ref": float(a[int(s)]), "abs_diff": float(d[int(s)]),
              "per_slot": float(per[int(s)])} for s, (l, m, mp) in zip(top, _slot_lmm(b, top))]
    return {"by_degree": bands, "by_abs_ref": decades, "worst": worst}


def _to_pair_major(torch, spec_np: np.ndarray, n: int, w: np.ndarray | None, dev):
    """Oracle spectrum [m bin, j, m' bin] -> the GPU stage layout [m'][m][j] (times w_j: the
    reference's own w * s product, dwt.py:115), on the device."""
    s = torch.from_numpy(spec_np).to(dev)
    x = s.permute(2, 0, 1).contiguous()
    del s
    if w is not None:
        x *= torch.from_numpy(w).to(dev)
    return x.reshape(-1)


def run_parity(b: int, so3, torch, *, workers: int = 1, truth_slices=(0,), truth_clusters=((0, 0),),
               log=print) -> dict:
    """The whole protocol at bandwidth b on cuda:current.  Returns a JSON-ready dict."""
    n = 2 * b
    dev = torch.device("cuda", torch.cuda.current_device())
    res: dict = {"bandwidth": b, "workers": workers, "inputs": "coefficients N(0,1) re/im, seed = B"}
    rng = np.random.default_rng(b)
    C = O.n_coeffs(b)
    c = rng.standard_normal(C) + 1j * rng.standard_normal(C)
    plan = so3.make_plan(b, device=dev)
    cd = torch.from_numpy(c).to(dev)
    degree = torch.repeat_interleave(torch.arange(b, device=dev),
                                     torch.tensor([(2 * l + 1) ** 2 for l in range(b)], device=dev))
    w = O.beta_weights(b)
    times: dict = {}

    # ---------------- inverse: DWT synthesis stage (oracle vs GPU on the same coefficients)
    t0 = time.perf_counter()
    s_syn = O.dwt_synthesis_stage(c, b, workers)
    times["dwt_synthesis"] = time.perf_counter() - t0
    log(f"B={b}: oracle DWT synthesis {times['dwt_synthesis']:.1f} s")
    x_ref = _to_pair_major(torch, s_syn, n, None, dev)
    x_gpu = torch.zeros_like(x_ref)
    so3.dwt_synthesis(plan, cd, x_gpu)
    res["inverse_dwt_stage"] = _t_metrics(x_gpu, x_ref)   # both zero in the Nyquist rows
    truth = []
    for (bm, bmp) in truth_clusters:
        for (m, mp, col) in E.synthesis_cluster_ld(b, bm, bmp, c):
            tr = col.astype(np.clongdouble)
            g = x_gpu.view(n, n, n)[mp % n, m % n].cpu().numpy()
            r = s_syn[m % n, :, mp % n]
            scale = float(np.abs(tr).max())
            truth.append({"m": m, "mp": mp, "gpu_err": float(np.abs(g - tr).max()),
                          "ref_err": float(np.abs(r - tr).max()), "scale": scale})
    res["inverse_dwt_stage"]["truth"] = _summ_truth(truth)
    # ---------------- inverse: FFT synthesis stage (GPU fed the oracle spectrum)
    g_stage = torch.empty(n ** 3, dtype=torch.complex128, device=dev)
    so3.fft_synthesis(plan, x_ref, g_stage)
    del x_gpu
    t0 = time.perf_counter()
    g_ref = O.fft_synthesis_stage(s_syn, b, workers)
    times["fft_synthesis"] = time.perf_counter() - t0
    log(f"B={b}: oracle FFT synthesis {times['fft_synthesis']:.1f} s")
    g_ref_d = torch.from_numpy(g_ref).to(dev)
    res["inverse_fft_stage"] = _t_metrics(g_stage, g_ref_d)
    truth = []
    gs = g_stage.view(n, n, n)
    gr = g_ref.reshape(n, n, n)
    for j in truth_slices:
        tr = E.slice_dft_ld(s_syn[:, j, :], -1)
        truth.append({"j": j, "gpu_err": float(np.abs(gs[:, j, :].cpu().numpy() - tr).max()),
                      "ref_err": float(np.abs(gr[:, j, :] - tr).max()), "scale": float(np.abs(tr).max())})
    res["inverse_fft_stage"]["truth"] = _summ_truth(truth)
    del g_stage, gs, x_ref, s_syn
    # ---------------- inverse: whole transform
    g_gpu = so3.ifsoft_sequential(so3.So3Coefficients(b, cd), plan).data
    res["inverse"] = _t_metrics(g_gpu, g_ref_d)
    truth = []
    gg = g_gpu.view(n, n, n)
    for j in truth_slices:
        tr = E.inverse_slice_ld(c, b, j)
        truth.append({"j": j, "gpu_err": float(np.abs(gg[:, j, :].cpu().numpy() - tr).max()),
                      "ref_err": float(np.abs(gr[:, j, :] - tr).max()), "scale": float(np.abs(tr).max())})
    res["inverse"]["truth"] = _summ_truth(truth)
    log(f"B={b}: inverse {res['inverse']}")
    del gg

    # ---------------- forward: FFT analysis stage (the oracle grid into both)
    t0 = time.perf_counter()
    s_ana = O.fft_analysis_stage(g_ref, b, workers)
    times["fft_analysis"] = time.perf_counter() - t0
    log(f"B={b}: oracle FFT analysis {times['fft_analysis']:.1f} s")
    x_gpu = torch.empty(n ** 3, dtype=torch.complex128, device=dev)
    so3.fft_analysis(plan, g_ref_d, x_gpu)
    x_ref = _to_pair_major(torch, s_ana, n, w, dev)
    _zero_nyquist(x_gpu, n, b)
    _zero_nyquist(x_ref, n, b)
    res["forward_fft_stage"] = _t_metrics(x_gpu, x_ref)
    truth = []
    wl = E.weights_ld(b)
    xg = x_gpu.view(n, n, n)
    for j in truth_slices:
        tr = E.slice_dft_ld(gr[:, j, :], +1) * wl[j]                 # [m][m']
        got = xg[:, :, j].cpu().numpy().T                             # [m'][m] -> [m][m']
        ref = s_ana[:, j, :] * w[j]
        mask = np.ones((n, n), bool)
        mask[b, :] = mask[:, b] = False
        truth.append({"j": j, "gpu_err": float(np.abs(got - tr)[mask].max()),
                      "ref_err": float(np.abs(ref - tr)[mask].max()), "scale": float(np.abs(tr).max())})
    res["forward_fft_stage"]["truth"] = _summ_truth(truth)
    del x_gpu, xg
    # ---------------- forward: DWT analysis stage (GPU fed the oracle's weighted spectrum)
    f_stage = torch.empty(C, dtype=torch.complex128, device=dev)
    so3.dwt_analysis(plan, x_ref, f_stage)
    del x_ref
    t0 = time.perf_counter()
    f_ref = O.dwt_analysis_stage(s_ana, b, workers)
    times["dwt_analysis"] = time.perf_counter() - t0
    log(f"B={b}: oracle DWT analysis {times['dwt_analysis']:.1f} s")
    f_ref_d = torch.from_numpy(f_ref).to(dev)
    res["forward_dwt_stage"] = _t_metrics(f_stage, f_ref_d)
    stage_bd = _breakdown(torch, b, f_stage, f_ref_d, degree)
    extra = [(max(abs(x["m"]), abs(x["mp"])), min(abs(x["m"]), abs(x["mp"]))) for x in stage_bd["worst"]]
    clusters = list(dict.fromkeys([tuple(t) for t in truth_clusters] + extra))
    res["forward_dwt_stage"]["truth"] = _truth_analysis(b, clusters, s_ana, f_stage, f_ref, torch)
    res["forward_dwt_stage"]["breakdown"] = stage_bd
    # ---------------- forward: whole transform
    f_gpu = so3.fsoft_sequential(so3.So3SampleGrid(b, g_ref_d), plan).data
    res["forward"] = _t_metrics(f_gpu, f_ref_d)
    res["forward"]["breakdown"] = _breakdown(torch, b, f_gpu, f_ref_d, degree)
    log(f"B={b}: forward {res['forward']['rel_of_max']:.3e} rel-of-max, {res['forward']['per_slot']:.3e} per slot")
    del f_stage, s_ana
    # ---------------- round trips (truth = the input coefficients)
    f_rt = so3.fsoft_sequential(so3.So3SampleGrid(b, g_gpu), plan).data
    res["round_trip_gpu"] = _t_metrics(f_rt, cd)
    res["round_trip_gpu"]["breakdown"] = _breakdown(torch, b, f_rt, cd, degree)
    res["round_trip_reference"] = _t_metrics(f_ref_d, cd)
    res["round_trip_reference"]["breakdown"] = _breakdown(torch, b, f_ref_d, cd, degree)
    # the same slots compared: where the GPU's per-slot error exceeds the reference's
    dg = (f_rt - cd).abs()
    dr = (f_ref_d - cd).abs()
    res["round_trip_compare"] = {
        "gpu_rms_abs": float(dg.pow(2).mean().sqrt()), "reference_rms_abs": float(dr.pow(2).mean().sqrt()),
        "slots_gpu_worse": float((dg > dr).double().mean()),
        "gpu_per_slot_at_reference_worst": float(dg[int(torch.argmax(dr / cd.abs()))] /
                                                 cd.abs()[int(torch.argmax(dr / cd.abs()))]),
        "reference_per_slot_at_gpu_worst": float(dr[int(torch.argmax(dg / cd.abs()))] /
                                                 cd.abs()[int(torch.argmax(dg / cd.abs()))]),
        "min_abs_coefficient": float(cd.abs().min()),
    }
    # the per-slot distribution, not only its single largest entry (which sits at the smallest
    # |c| of the draw for both implementations)
    ca = cd.abs()
    for name, d in (("gpu", dg), ("reference", dr)):
        per = torch.sort(d / ca).values
        k = per.numel()
        res["round_trip_compare"][f"{name}_per_slot_quantiles"] = {
            q: float(per[min(k - 1, int(float(q) * k))]) for q in ("0.5", "0.99", "0.999", "0.9999", "0.99999")}
        res["round_trip_compare"][f"{name}_slots_over_1e-10"] = int((per > 1e-10).sum())
        del per
    del ca
    # ---------------- the fp64 floor of the round trip: the grid itself is fp64
    # g_gpu holds the band-limited function rounded to fp64.  Moving every component by one
    # ulp in a random direction (a perturbation of the size of that rounding; uniform rounding
    # error has rms ulp/sqrt(12)) and transforming again shows the coefficient error that no
    # fp64-grid implementation can avoid, slot by slot.
    gen = torch.Generator(device=dev).manual_seed(1234)
    gv = torch.view_as_real(g_gpu).reshape(-1)
    pert = torch.empty_like(gv)
    inf = torch.tensor(float("inf"), dtype=torch.float64, device=dev)
    for s0 in range(0, gv.numel(), 1 << 27):
        x = gv[s0:s0 + (1 << 27)]
        up = torch.rand(x.shape, generator=gen, device=dev, dtype=torch.float64) < 0.5
        pert[s0:s0 + (1 << 27)] = torch.where(up, torch.nextafter(x, inf), torch.nextafter(x, -inf))
    del up, x
    pert = pert.view(-1, 2)
    f_pert = so3.fsoft_sequential(so3.So3SampleGrid(b, torch.view_as_complex(pert)), plan).data
    del pert
    dp = (f_pert - f_rt).abs()
    ca = cd.abs()
    imin = int(torch.argmin(ca))
    res["grid_ulp_floor"] = {
        "what": "coefficients of fsoft(grid moved by 1 ulp per component, random sign) - fsoft(grid)",
        "max_abs": float(dp.max()), "rms_abs": float(dp.pow(2).mean().sqrt()),
        "per_slot": float((dp / ca).max()),
        "per_slot_at_min_abs_coefficient": float(dp[imin] / ca[imin]),
        "rounding_scale": 1.0 / 12 ** 0.5,
        "expected_rounding_per_slot_at_min_abs_coefficient": float(dp[imin] / ca[imin]) / 12 ** 0.5,
        "expected_rounding_rms_abs": float(dp.pow(2).mean().sqrt()) / 12 ** 0.5,
    }
    del f_pert, dp
    res["oracle_seconds"] = times
    res["oracle_inverse_s"] = times["dwt_synthesis"] + times["fft_synthesis"]
    res["oracle_forward_s"] = times["fft_analysis"] + times["dwt_analysis"]
    plan.release()
    return res


def _summ_truth(rows: list[dict]) -> dict:
    """Long-double attribution: max fp64 error of the GPU and of the reference arithmetic
    against the extended-precision values, on the same samples."""
    if not rows:
        return {}
    return {"samples": len(rows), "gpu_max_err": max(r["gpu_err"] for r in rows),
            "reference_max_err": max(r["ref_err"] for r in rows), "scale": max(r["scale"] for r in rows),
            "rows": rows}


def _truth_analysis(b, clusters, s_ana, f_stage, f_ref, torch) -> dict:
    rows = []
    for (bm, bmp) in clusters:
        for (m, mp, col) in E.analysis_cluster_ld(b, bm, bmp, s_ana):
            sl = O.pair_slots(m, mp, b)
            g = f_stage[torch.from_numpy(sl).to(f_stage.device)].cpu().numpy()
            r = f_ref[sl]
            a = np.abs(col).astype(np.float64)
            nz = a > 0
            rows.append({"m": m, "mp": mp, "gpu_err": float(np.abs(g - col).max()),
                         "ref_err": float(np.abs(r - col).max()), "scale": float(a.max()),
                         "gpu_per_slot": float((np.abs(g - col)[nz] / a[nz]).max()),
                         "ref_per_slot": float((np.abs(r - col)[nz] / a[nz]).max())})
    out = _summ_truth(rows)
    out["gpu_max_per_slot"] = max(r["gpu_per_slot"] for r in rows)
    out["reference_max_per_slot"] = max(r["ref_per_slot"] for r in rows)
    return out
