"""Per-direction parity at BASELINE sizes B=128 and B=256 (SURVEY.md 8(d) protocol, oracle/parity.py):

* inverse: the same seeded coefficients (seed = B) into the GPU iFSOFT and the oracle iFSOFT
  (bit-identical to the reference's ifsoft_parallel, soft.py:152-173);
* forward: the oracle's grid, bit for bit, into the GPU FSOFT and the oracle FSOFT (soft.py:124-149);
* each stage fed the oracle's own stage input, and every difference attributed against
  long-double values (oracle/extended.py) on sampled slices and clusters.

Bounds (north_star: max relative coefficient error <= 1e-10, fp64):
  * coefficients: per-slot max |d| / |ref| <= 1e-10 (reference error_metrics, bench.py:122-131)
    and max |d| / max |ref| <= 1e-12, in the forward direction against the reference arithmetic;
  * grids: max |d| / max |ref| <= 1e-12 (grid values cross zero, so a per-point ratio is not a
    coefficient error);
  * every stage: the GPU's error against the long-double values at most 1.5x the reference's;
  * round trip: per-slot <= 1e-10 at B=128; at B=256 the per-slot error distribution at or
    below the reference's own arithmetic at every quantile, and smaller max / rms abs error.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
so3 = pytest.importorskip("paper_1808_00896_b200")

from oracle import so3_oracle as O  # noqa: E402
from oracle.parity import run_parity  # noqa: E402

_CACHE = {}


def parity(b):
    if b not in _CACHE:
        slices = sorted({0, b // 3, b - 1, 2 * b - 1})
        clusters = [(0, 0), (1, 0), (b // 2, 0), (b - 1, 0), (b // 3, b // 3), (b - 1, b - 1), (b // 2, b // 5),
                    (b - 1, b - 2)]
        _CACHE[b] = run_parity(b, so3, torch, workers=O.default_workers(), truth_slices=slices,
                               truth_clusters=clusters, log=lambda s: None)
    return _CACHE[b]


@pytest.mark.parametrize("b", [128, pytest.param(256, marks=pytest.mark.slow)])
def test_inverse_matches_reference_arithmetic(b):
    r = parity(b)
    assert r["inverse"]["rel_of_max"] < 1e-12
    assert r["inverse_dwt_stage"]["rel_of_max"] < 1e-12
    assert r["inverse_fft_stage"]["rel_of_max"] < 1e-14


@pytest.mark.parametrize("b", [128, pytest.param(256, marks=pytest.mark.slow)])
def test_forward_matches_reference_arithmetic(b):
    r = parity(b)
    assert r["forward"]["per_slot"] < 1e-10
    assert r["forward"]["rel_of_max"] < 1e-12
    assert r["forward_dwt_stage"]["per_slot"] < 1e-10
    assert r["forward_fft_stage"]["rel_of_max"] < 1e-13


@pytest.mark.parametrize("b", [128, pytest.param(256, marks=pytest.mark.slow)])
def test_stage_errors_attributed_against_long_double(b):
    r = parity(b)
    for stage in ("inverse_dwt_stage", "inverse_fft_stage", "inverse", "forward_fft_stage", "forward_dwt_stage"):
        t = r[stage]["truth"]
        assert t["gpu_max_err"] <= 1.5 * t["reference_max_err"], (stage, t["gpu_max_err"], t["reference_max_err"])


@pytest.mark.parametrize("b", [128, pytest.param(256, marks=pytest.mark.slow)])
def test_round_trip_at_or_below_the_reference_floor(b):
    """Round trip iFSOFT -> FSOFT against the input coefficients.  Below 1e-10 per slot at B=128.
    At B=256 the single worst slot is the smallest |c| of the draw (1.0e-4) for the GPU and the
    reference alike; the per-slot error DISTRIBUTION is compared on the same slots instead: the
    GPU must be at or below the reference's own arithmetic at every reported quantile (median to
    1 - 1e-5), and in max and rms abs error."""
    r = parity(b)
    gpu, ref, cmp = r["round_trip_gpu"], r["round_trip_reference"], r["round_trip_compare"]
    assert gpu["max_abs"] < ref["max_abs"]
    assert cmp["gpu_rms_abs"] < cmp["reference_rms_abs"]
    for q, v in cmp["gpu_per_slot_quantiles"].items():
        assert v <= cmp["reference_per_slot_quantiles"][q], q
    if b <= 128:
        assert gpu["per_slot"] < 1e-10
