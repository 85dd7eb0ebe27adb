"""The CPU oracle (oracle/so3_oracle.py) against the reference's golden vectors and
known answers.  Golden vectors were produced by importing the reference itself
(oracle/gen_golden.py); the oracle must reproduce them bit for bit."""
import math

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

from oracle import so3_oracle as O

SOFT_B = [1, 2, 3, 4, 5, 6, 8, 16]


@pytest.mark.parametrize("b", SOFT_B)
def test_oracle_inverse_matches_reference_bitwise(golden, b):
    g = golden(f"soft_b{b}.npz")
    assert_array_equal(O.ifsoft(g["coeffs"], b), g["inverse"])


@pytest.mark.parametrize("b", SOFT_B)
def test_oracle_forward_matches_reference_bitwise(golden, b):
    g = golden(f"soft_b{b}.npz")
    assert_array_equal(O.fsoft(g["inverse"], b), g["roundtrip"])
    assert_array_equal(O.fsoft(g["raw_grid"], b), g["forward_raw"])


@pytest.mark.parametrize("b", SOFT_B)
def test_oracle_tables_match_reference(golden, b):
    g = golden(f"soft_b{b}.npz")
    assert_array_equal(O.beta_weights(b), g["weights"])
    assert_array_equal(O.beta_nodes(b), g["betas"])


@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_oracle_direct_route_matches_reference(golden, b):
    g = golden(f"soft_b{b}.npz")
    assert_allclose(O.ifsoft_direct(g["coeffs"], b), g["direct_inverse"], rtol=0, atol=1e-14)
    assert_allclose(O.fsoft_direct(g["raw_grid"], b), g["direct_forward"], rtol=0, atol=1e-14)
    # fast vs direct (reference test_soft.py:30-45)
    assert_allclose(O.ifsoft(g["coeffs"], b), g["direct_inverse"], atol=1e-12)


def test_oracle_slice_dfts_match_reference(golden):
    g = golden("slices.npz")
    for n in (1, 2, 4, 6, 8, 10, 16, 32, 64):
        assert_array_equal(O.slice_dft(g[f"in_{n}"], +1), g[f"plus_{n}"])
        assert_array_equal(O.slice_dft(g[f"in_{n}"], -1), g[f"minus_{n}"])


def test_oracle_wigner_rows_and_columns_match_reference(golden):
    g = golden("wigner.npz")
    for b in (16, 64):
        betas = O.beta_nodes(b)
        w = O.beta_weights(b)
        v = (2.0 * np.arange(b) + 1.0) / (8.0 * math.pi * b)
        for (m, mp) in [(0, 0), (1, 0), (3, 3), (5, 2), (b - 1, 0), (b - 1, b - 2), (b // 2, b // 3)]:
            rows = O.recurrence_rows(m, mp, betas, b)
            assert_array_equal(rows, g[f"rows_b{b}_{m}_{mp}"])
            for (pm, pmp, tag) in O.cluster_members(m, mp):
                mat = O.member_matrix(rows, tag, m, mp, b)
                tagk = f"b{b}_{pm}_{pmp}"
                assert_array_equal(O.analysis_column(mat, v[m:], w, g[f"dwt_in_{tagk}"]), g[f"dwt_out_{tagk}"])
                assert_array_equal(O.synthesis_column(mat, g[f"idwt_in_{tagk}"]), g[f"idwt_out_{tagk}"])


def test_oracle_schedule_matches_reference(golden):
    g = golden("schedule.npz")
    for b in (1, 2, 3, 4, 7, 8, 16, 33):
        assert [tuple(x) for x in g[f"bases_b{b}"]] == O.base_pairs(b)


# ---- known answers frozen in the reference's tests

def test_known_answers():
    assert O.n_coeffs(1) == 1 and O.n_coeffs(2) == 10 and O.n_coeffs(32) == 43680   # test_core.py:11-14
    assert O.slot(2, 0, 1) == 23                                                     # test_core.py:22-23
    assert_allclose(O.beta_weights(1), [math.pi, math.pi], atol=1e-15)               # test_quadrature.py:30-32
    w2 = O.beta_weights(2)                                                           # test_quadrature.py:35-42
    assert w2[0] == pytest.approx(0.41515792, abs=1e-8)
    assert w2[1] == pytest.approx(1.15563841, abs=1e-8)
    col = O.recurrence_rows(0, 0, np.array([math.pi / 3]), 3)[:, 0]                  # test_wigner.py:103-107
    assert_allclose(col, [1.0, 0.5, -0.125], atol=1e-15)
    col = O.recurrence_rows(0, 0, np.array([math.pi / 2]), 3)[:, 0]
    assert_allclose(col, [1.0, 0.0, -0.5], atol=1e-15)
    betas = np.linspace(0.05, math.pi - 0.05, 9)                                     # test_wigner.py:56-61
    assert_allclose(O.closed_form_d(1, 1, 0, betas), np.sin(betas) / math.sqrt(2), atol=1e-15)
    assert_allclose(O.closed_form_d(1, 0, 1, betas), -np.sin(betas) / math.sqrt(2), atol=1e-15)


def test_dft_delta_frozen():
    x = np.zeros(4, dtype=np.complex128)                                             # test_fft.py:13-17
    x[1] = 1.0
    assert_allclose(O.dft_lastaxis(x, -1), [1.0, -1.0j, -1.0, 1.0j], atol=1e-15)
    assert_allclose(O.dft_lastaxis(x, +1), [1.0, 1.0j, -1.0, -1.0j], atol=1e-15)


@pytest.mark.parametrize("b", [2, 4, 8])
def test_dwt_exactness_every_pair(b):
    """v T W T^t = I/(2B)^2 for every order pair (reference test_dwt.py:95-114)."""
    w = O.beta_weights(b)
    v = (2.0 * np.arange(b) + 1.0) / (8.0 * math.pi * b)
    betas = O.beta_nodes(b)
    rng = np.random.default_rng(b)
    for bm, bmp in O.base_pairs(b):
        rows = O.recurrence_rows(bm, bmp, betas, b)
        for (m, mp, tag) in O.cluster_members(bm, bmp):
            mat = O.member_matrix(rows, tag, bm, bmp, b)
            c = rng.standard_normal(mat.shape[0]) + 1j * rng.standard_normal(mat.shape[0])
            back = O.analysis_column(mat, v[bm:], w, O.synthesis_column(mat, c))
            assert_allclose(back, c / (2 * b) ** 2, atol=1e-12)


def test_oracle_round_trip_and_constant():
    b = 8
    rng = np.random.default_rng(3)
    c = rng.standard_normal(O.n_coeffs(b)) + 1j * rng.standard_normal(O.n_coeffs(b))
    assert_allclose(O.fsoft(O.ifsoft(c, b), b), c, atol=1e-11)
    f = O.fsoft(np.ones((2 * b) ** 3, dtype=np.complex128), 4 if False else b)
    e = np.zeros_like(f)
    e[0] = 1.0
    assert_allclose(f, e, atol=1e-12)                                                # test_soft.py:73-84


def test_oracle_members_cover_order_square():
    for b in (1, 2, 5, 9):
        pairs = [(m, mp) for bm, bmp in O.base_pairs(b) for (m, mp, _) in O.cluster_members(bm, bmp)]
        assert len(pairs) == (2 * b - 1) ** 2
        assert set(pairs) == {(m, mp) for m in range(-b + 1, b) for mp in range(-b + 1, b)}
