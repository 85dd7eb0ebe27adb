"""The C-ABI library without a GPU: it loads, exports every symbol include/*.h declares,
and its host-side plan logic (weights, angles, layouts, cluster schedule) matches the oracle."""
import glob
import os
import re

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

import paper_1808_00896_b200 as so3
from paper_1808_00896_b200 import _native
from oracle import so3_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(hdr).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(so3_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for name in sorted(names):
        assert hasattr(lib, name), name
    assert names == set(_native.SIGNATURES), "ctypes signatures must cover exactly the header"


def test_layout_helpers_match_oracle():
    lib = _native.lib()
    for b in (1, 2, 3, 8, 17, 64, 512):
        assert lib.so3_coeff_count(b) == O.n_coeffs(b) == so3.coeff_count(b)
        assert lib.so3_grid_count(b) == (2 * b) ** 3
    for b in (1, 2, 5, 8):
        seen = [lib.so3_coeff_index(l, m, mp, b) for l in range(b) for m in range(-l, l + 1) for mp in range(-l, l + 1)]
        assert seen == list(range(O.n_coeffs(b)))
    assert lib.so3_coeff_index(2, 0, 1, 4) == 23
    assert lib.so3_coeff_index(4, 0, 0, 4) == -1 and lib.so3_coeff_index(2, 3, 0, 4) == -1
    assert lib.so3_coeff_count(0) == 0


@pytest.mark.parametrize("b", [1, 2, 3, 4, 8, 16, 33, 64, 128, 512])
def test_quadrature_weights_match_oracle(b):
    w = so3.quadrature_weights(b).values
    ref = O.beta_weights(b)
    # long double host evaluation vs the reference's double numpy expression
    assert_allclose(w, ref, rtol=0, atol=max(4e-15, 3e-17 * b) * ref.max())   # numpy's error grows ~B ulp
    assert np.all(w > 0)
    assert_allclose(w[::-1], w, rtol=1e-14)
    assert abs(w.sum() - 2 * np.pi / b) < 1e-13


@pytest.mark.parametrize("b", [1, 2, 7, 64])
def test_sample_angles_match_oracle_exactly(b):
    a = so3.sample_angles(b)
    assert_array_equal(a.betas, O.beta_nodes(b))
    assert_array_equal(a.alphas, O.angle_nodes(b))
    assert_array_equal(a.gammas, a.alphas)


@pytest.mark.parametrize("b", [1, 2, 3, 8, 33, 128])
def test_cluster_schedule_is_a_cost_sorted_permutation(b):
    bases, mem = so3.cluster_schedule(b)
    assert len(bases) == b * (b + 1) // 2
    assert sorted(map(tuple, bases.tolist())) == sorted(O.base_pairs(b))
    for (m, mp), k in zip(bases.tolist(), mem.tolist()):
        assert k == len(O.cluster_members(m, mp))
    cost = mem * (b - bases[:, 0])
    assert np.all(np.diff(cost) <= 0), "longest clusters first"


def test_enumerate_clusters_matches_reference_order(golden):
    g = golden("schedule.npz")
    for b in (1, 2, 3, 4, 7, 8, 16, 33):
        assert [tuple(c.base) for c in so3.enumerate_clusters(b)] == [tuple(x) for x in g[f"bases_b{b}"]]
        assert sorted(tuple(c.base) for c in so3.enumerate_clusters(b, "sigma")) == sorted(O.base_pairs(b))
    with pytest.raises(ValueError):
        so3.enumerate_clusters(4, "spiral")


def test_cluster_members_match_oracle():
    for b in (2, 6, 11):
        for (m, mp) in O.base_pairs(b):
            ours = [(p.m, p.mp, rel.tag) for p, rel in so3.cluster_for_base(m, mp).members]
            assert ours == O.cluster_members(m, mp)


def test_invalid_bandwidth_maps_to_valueerror():
    with pytest.raises(ValueError):
        so3.quadrature_weights(0)
    lib = _native.lib()
    out = np.empty(8)
    assert lib.so3_quadrature_weights(0, out.ctypes.data_as(_native._dp)) == _native.SO3_ERR_INVALID
    assert b"bandwidth" in lib.so3_last_error()
