"""Segment-parallel DWT kernels (csrc/dwt_seg.cuh) against the dwt_mma.cuh kernels and the oracle.

The segment-parallel kernels start every degree segment from a checkpoint the plan wrote with the
same fma sequence, so each Wigner value is the one an uninterrupted recurrence gives; only the
order of the beta (analysis) / degree (synthesis) sums differs from the dwt_mma.cuh kernels:
agreement to a few ulps of the largest value (1e-14 relative to max), and the oracle bounds of
test_gpu_parity.py hold for either.  Knob dwt_seg: bit 1 synthesis (default for B % 64 == 0),
bit 2 analysis (one CTA per cluster part), bit 4 persistent analysis.
"""
import numpy as np
import pytest

from oracle import so3_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
so3 = pytest.importorskip("paper_1808_00896_b200")


def seeded(b, seed=None):
    rng = np.random.default_rng(b if seed is None else seed)
    C = O.n_coeffs(b)
    return rng.standard_normal(C) + 1j * rng.standard_normal(C)


@pytest.mark.parametrize("b", [64, 128, 192, 320])
def test_seg_synthesis_matches_mma_synthesis(b):
    """Default synthesis (segments) vs dwt_synthesis_mma_kernel on the same coefficients; B = 192
    and 320 take the 2-warp CTA shape (2B / 64 not a multiple of 4)."""
    plan = so3.make_plan(b)
    c = torch.from_numpy(seeded(b)).cuda()
    n = 2 * b
    spec = []
    for seg in (0, 1, 1):
        plan.set_knob("dwt_seg", seg)
        s = torch.zeros(n ** 3, dtype=torch.complex128, device="cuda")
        so3.dwt_synthesis(plan, c, s)
        spec.append(s)
    torch.cuda.synchronize()
    assert (spec[1] - spec[0]).abs().max().item() <= 1e-14 * spec[0].abs().max().item()
    assert torch.equal(spec[1], spec[2])                    # deterministic
    assert torch.equal(spec[1] != 0, spec[0] != 0)          # the same order pairs written (Nyquist rows untouched)


@pytest.mark.parametrize("b,knobs", [(64, {"dwt_seg": 2}), (128, {"dwt_seg": 2}), (128, {"dwt_seg": 4}),
                                     (128, {"dwt_seg": 4, "seg_ana_w": 4}), (192, {"dwt_seg": 4}),
                                     (320, {"dwt_seg": 2}), (320, {"dwt_seg": 4}),
                                     (256, {"dwt_seg": 4, "seg_ana_w": 4})])
def test_seg_analysis_variants_match_mma_analysis(b, knobs):
    """One-CTA-per-part (bit 2) and persistent (bit 4) segment analysis vs dwt_analysis_mma_cta_kernel
    on the same spectrum: split clusters (B = 320: two parts; seg_ana_w = 4 at B = 256: two passes
    accumulated through the plan scratch), both table halves in one CTA (B <= 256)."""
    plan = so3.make_plan(b)
    plan.set_knob("dwt_seg", 0)
    c = torch.from_numpy(seeded(b)).cuda()
    spec = torch.zeros((2 * b) ** 3, dtype=torch.complex128, device="cuda")
    so3.dwt_synthesis(plan, c, spec)
    ref = torch.zeros_like(c)
    so3.dwt_analysis(plan, spec, ref)
    for k, v in knobs.items():
        plan.set_knob(k, v)
    outs = []
    for _ in range(2):
        o = torch.zeros_like(c)
        so3.dwt_analysis(plan, spec, o)
        outs.append(o)
    torch.cuda.synchronize()
    assert (outs[0] - ref).abs().max().item() <= 1e-14 * ref.abs().max().item()
    assert torch.equal(outs[0], outs[1])
    assert torch.isfinite(torch.view_as_real(outs[0])).all()


@pytest.mark.parametrize("seg", [1, 3, 5])
def test_seg_whole_transform_against_oracle_b64(seg):
    """iFSOFT and FSOFT at B = 64 with the segment kernels, each direction against the oracle
    (the bounds of test_gpu_parity.py: 1e-12 of max, per-slot 1e-10)."""
    b = 64
    plan = so3.make_plan(b)
    plan.set_knob("dwt_seg", seg)
    c = seeded(b)
    g_ref = O.ifsoft(c, b)
    f_ref = O.fsoft(g_ref, b)
    g = so3.ifsoft_sequential(so3.So3Coefficients(b, c), plan).data
    f = so3.fsoft_sequential(so3.So3SampleGrid(b, g_ref), plan).data
    assert np.abs(g - g_ref).max() <= 1e-12 * np.abs(g_ref).max()
    assert np.abs(f - f_ref).max() <= 1e-12 * np.abs(f_ref).max()
    assert O.error_metrics(f_ref, f)[1] <= 1e-10


def test_seg_knob_off_without_checkpoints_and_ineligible_bandwidths():
    """B not a multiple of 64 keeps the dwt_mma.cuh kernels whatever the knob says (no checkpoint
    table is built), and results do not depend on the knob."""
    b = 48
    plan = so3.make_plan(b)
    before = plan.device_bytes
    c = torch.from_numpy(seeded(b)).cuda()
    outs = []
    for seg in (0, 7):
        plan.set_knob("dwt_seg", seg)
        s = torch.zeros((2 * b) ** 3, dtype=torch.complex128, device="cuda")
        so3.dwt_synthesis(plan, c, s)
        outs.append(s)
    assert torch.equal(outs[0], outs[1])
    assert plan.device_bytes == before
    # eligible: the table is 8 x 2B x 16 bytes per cluster
    b = 64
    plan = so3.make_plan(b)
    assert plan.device_bytes >= (b * (b + 1) // 2) * 8 * 2 * b * 16


def test_seg_synthesis_batched_plan_matches_single_function_plans():
    """A batched plan at B = 64 (beyond the dense-contraction kernels' 2B <= 64) runs the segment
    synthesis once per function (grid.y): bit-identical to one-function plans."""
    b, f = 64, 3
    n, C = 2 * b, O.n_coeffs(b)
    rng = np.random.default_rng(7)
    c = rng.standard_normal(f * C) + 1j * rng.standard_normal(f * C)
    pb = so3.make_plan(b, batch=f)
    spec_b = torch.zeros(f * n ** 3, dtype=torch.complex128, device="cuda")
    so3.dwt_synthesis(pb, torch.from_numpy(c).cuda(), spec_b)
    p1 = so3.make_plan(b)
    for i in range(f):
        s1 = torch.zeros(n ** 3, dtype=torch.complex128, device="cuda")
        so3.dwt_synthesis(p1, torch.from_numpy(c[i * C:(i + 1) * C].copy()).cuda(), s1)
        assert torch.equal(s1, spec_b[i * n ** 3:(i + 1) * n ** 3])
    g = so3.ifsoft_batch(c, pb)
    back = so3.fsoft_batch(g, pb)
    assert np.abs(np.asarray(back).reshape(-1) - c).max() < 1e-11


def test_default_analysis_at_b320_is_the_persistent_segment_kernel():
    """B = 320 (2B / 64 = 10 warps): the plan's default analysis is the persistent segment kernel
    (two passes per cluster through the plan scratch): equal to the knob-selected kernel, within
    rounding of the dwt_mma.cuh analysis, and the whole round trip recovers the coefficients."""
    b = 320
    plan = so3.make_plan(b)
    c = seeded(b)
    cd = torch.from_numpy(c).cuda()
    spec = torch.zeros((2 * b) ** 3, dtype=torch.complex128, device="cuda")
    so3.dwt_synthesis(plan, cd, spec)
    out_default = torch.zeros_like(cd)
    so3.dwt_analysis(plan, spec, out_default)
    plan.set_knob("dwt_seg", 1)                      # dwt_mma.cuh analysis
    out_mma = torch.zeros_like(cd)
    so3.dwt_analysis(plan, spec, out_mma)
    plan.set_knob("dwt_seg", 5)
    out_p = torch.zeros_like(cd)
    so3.dwt_analysis(plan, spec, out_p)
    assert torch.equal(out_default, out_p)          # the default IS the persistent kernel
    assert (out_p - out_mma).abs().max().item() <= 1e-14 * out_mma.abs().max().item()
    g = so3.ifsoft_sequential(so3.So3Coefficients(b, cd), plan)
    back = so3.fsoft_sequential(g, plan).data
    assert (back - cd).abs().max().item() < 1e-11
