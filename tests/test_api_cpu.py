"""Host-side API: containers, validation and SOFC/SOFG persistence (reference core.py,
soft.py argument checks) -- no GPU needed."""
import numpy as np
import pytest
from numpy.testing import assert_array_equal

import paper_1808_00896_b200 as so3


def test_validate_bandwidth():
    assert so3.validate_bandwidth(3) == 3
    for bad in (0, -1, 2.5, "4", True):
        with pytest.raises(ValueError):
            so3.validate_bandwidth(bad)


def test_containers_validate_lengths():
    with pytest.raises(ValueError):
        so3.So3Coefficients(4, np.zeros(10))
    with pytest.raises(ValueError):
        so3.So3SampleGrid(2, np.zeros(63))
    c = so3.So3Coefficients(2, np.arange(10))
    assert c.data.dtype == np.complex128 and c.slot(1, -1, 1) == 3
    g = so3.So3SampleGrid.zeros(2)
    assert g.as_3d().shape == (4, 4, 4)
    with pytest.raises(ValueError):
        so3.So3SampleGrid.from_3d(2, np.zeros((4, 4, 3)))


def test_order_pair_slots_matches_coeff_index():
    b = 6
    for m in range(-b + 1, b):
        for mp in range(-b + 1, b):
            lo = max(abs(m), abs(mp))
            assert so3.order_pair_slots(m, mp, b).tolist() == [so3.coeff_index(l, m, mp, b) for l in range(lo, b)]
    with pytest.raises(ValueError):
        so3.coeff_index(4, 0, 0, 4)


def test_degree_of_slots():
    d = so3.degree_of_slots(5)
    assert d.shape == (so3.coeff_count(5),)
    assert d[so3.coeff_index(3, -2, 1, 5)] == 3


def test_make_plan_validation_before_any_device_work():
    with pytest.raises(ValueError):
        so3.make_plan(4, matrix_policy="lazy")
    with pytest.raises(ValueError):
        so3.make_plan(4, partitioner="spiral")
    with pytest.raises(ValueError):
        so3.make_plan(0)
    with pytest.raises(ValueError):
        so3.make_plan(4, batch=0)


def test_threads_validated_like_reference():
    g = so3.So3SampleGrid.zeros(2)
    for bad in (0, -2, 1.5, True):
        with pytest.raises(ValueError):
            so3.fsoft_parallel(g, None, bad)
        with pytest.raises(ValueError):
            so3.ifsoft_parallel(so3.So3Coefficients.zeros(2), None, bad)


def test_binary_round_trips_are_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    c = so3.So3Coefficients(3, rng.standard_normal(35) + 1j * rng.standard_normal(35))
    so3.write_coefficients(str(tmp_path / "c.sofc"), c)
    assert_array_equal(so3.read_coefficients(str(tmp_path / "c.sofc")).data, c.data)
    g = so3.So3SampleGrid(2, rng.standard_normal(64) + 1j * rng.standard_normal(64))
    so3.write_samples(str(tmp_path / "g.sofg"), g)
    back = so3.read_samples(str(tmp_path / "g.sofg"))
    assert back.bandwidth == 2
    assert_array_equal(back.data, g.data)


def test_binary_header_and_rejections(tmp_path):
    c = so3.So3Coefficients.zeros(2)
    p = tmp_path / "c.sofc"
    so3.write_coefficients(str(p), c)
    blob = p.read_bytes()
    assert blob[:4] == so3.SOFC_MAGIC
    assert np.frombuffer(blob[4:12], dtype="<u4").tolist() == [so3.FORMAT_VERSION, 2]
    assert len(blob) == 12 + 16 * 10
    with pytest.raises(ValueError):
        so3.read_samples(str(p))                       # wrong magic
    (tmp_path / "bad.sofc").write_bytes(blob[:4] + np.asarray([9, 2], "<u4").tobytes() + blob[12:])
    with pytest.raises(ValueError):
        so3.read_coefficients(str(tmp_path / "bad.sofc"))   # version
    (tmp_path / "short.sofc").write_bytes(blob[:-16])
    with pytest.raises(ValueError):
        so3.read_coefficients(str(tmp_path / "short.sofc"))  # length
    bad = so3.So3Coefficients.zeros(2)
    bad.data[3] = np.nan
    with pytest.raises(ValueError):
        so3.write_coefficients(str(tmp_path / "nan.sofc"), bad)


def test_work_index_maps_follow_the_reference(golden):
    """sigma / kappa maps (reference schedule.py:40-90): the kappa part of the golden
    cluster order (after origin, axes, diagonals) is kappa_to_orders(0..), and both maps
    cover their triangles exactly once."""
    g = golden("schedule.npz")
    for b in (3, 4, 7, 8, 16, 33):
        kap = [tuple(x) for x in g[f"bases_b{b}"]][1 + 2 * (b - 1):]
        assert [tuple(so3.kappa_to_orders(k, b)) for k in range(so3.kappa_count(b))] == kap
        assert {tuple(so3.kappa_to_orders(k, b)) for k in range(so3.kappa_count(b))} == \
            {(m, mp) for m in range(2, b) for mp in range(1, m)}
    for s in range(500):
        m, mp = so3.sigma_inverse(s)
        assert so3.sigma_index(m, mp) == s and 0 <= mp <= m
    assert so3.kappa_split(0, 8) == (1, 1) and so3.kappa_split(so3.kappa_count(8) - 1, 8) == (3, 7)
    assert so3.kappa_count(1) == 0 and so3.kappa_count(2) == 0


@pytest.mark.parametrize("call", [
    lambda: so3.sigma_index(2, 3), lambda: so3.sigma_index(3, -1), lambda: so3.sigma_inverse(-1),
    lambda: so3.kappa_split(so3.kappa_count(6), 6), lambda: so3.kappa_split(-1, 6),
    lambda: so3.rect_to_orders(0, 1, 8), lambda: so3.rect_to_orders(4, 1, 8), lambda: so3.rect_to_orders(1, 8, 8),
    lambda: so3.rect_to_orders(3, 4, 7),   # beyond the half row of odd B
    lambda: so3.kappa_count(0),
])
def test_work_index_maps_reject_like_the_reference(call):
    with pytest.raises(ValueError):
        call()
