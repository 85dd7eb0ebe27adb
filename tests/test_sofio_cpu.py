"""SOFC / SOFG containers through the C library's streaming reader / writer (csrc/sofio.cuh),
host buffers (no GPU): byte-exact against files the reference itself wrote
(oracle/gen_sof_golden.py), beta-slab reads and sharded writes, and the reference's errors
(core.py:179-225)."""
import os

import numpy as np
import pytest

import paper_1808_00896_b200 as so3

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
B, N = 4, 8


def _payloads():
    g = np.random.default_rng(4)
    grid = g.standard_normal(N ** 3) + 1j * g.standard_normal(N ** 3)
    c = np.random.default_rng(5)
    coeffs = c.standard_normal(so3.coeff_count(B)) + 1j * c.standard_normal(so3.coeff_count(B))
    return grid, coeffs


def test_reads_reference_written_files_exactly():
    grid, coeffs = _payloads()
    assert so3.container_info(os.path.join(GOLD, "ref_b4.sofg")) == ("SOFG", B)
    assert np.array_equal(so3.read_samples(os.path.join(GOLD, "ref_b4.sofg")).data, grid)
    assert np.array_equal(so3.read_coefficients(os.path.join(GOLD, "ref_b4.sofc")).data, coeffs)


def test_writes_the_reference_bytes(tmp_path):
    grid, coeffs = _payloads()
    so3.write_samples(str(tmp_path / "g.sofg"), so3.So3SampleGrid(B, grid))
    so3.write_coefficients(str(tmp_path / "c.sofc"), so3.So3Coefficients(B, coeffs))
    assert (tmp_path / "g.sofg").read_bytes() == open(os.path.join(GOLD, "ref_b4.sofg"), "rb").read()
    assert (tmp_path / "c.sofc").read_bytes() == open(os.path.join(GOLD, "ref_b4.sofc"), "rb").read()


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_beta_slabs_read_and_written_per_rank(tmp_path, world):
    grid, _ = _payloads()
    cube = grid.reshape(N, N, N)
    J = N // world
    path = str(tmp_path / "s.sofg")
    for r in range(world):   # rank 0 creates the file, the others add their slabs
        so3.write_samples_slab(path, B, np.ascontiguousarray(cube[:, r * J:(r + 1) * J, :]).reshape(-1), r * J, J,
                               create=(r == 0))
    assert open(path, "rb").read() == open(os.path.join(GOLD, "ref_b4.sofg"), "rb").read()
    for r in range(world):
        sl = so3.read_samples_slab(os.path.join(GOLD, "ref_b4.sofg"), r * J, J)
        assert np.array_equal(sl.reshape(N, J, N), cube[:, r * J:(r + 1) * J, :])


def test_reference_errors(tmp_path):
    gold = open(os.path.join(GOLD, "ref_b4.sofg"), "rb").read()
    with pytest.raises(ValueError, match="not a SOFC container"):
        so3.read_coefficients(os.path.join(GOLD, "ref_b4.sofg"))
    (tmp_path / "v.sofg").write_bytes(gold[:4] + (2).to_bytes(4, "little") + gold[8:])
    with pytest.raises(ValueError, match="unsupported format version 2"):
        so3.read_samples(str(tmp_path / "v.sofg"))
    (tmp_path / "t.sofg").write_bytes(gold[:-8])
    with pytest.raises(ValueError, match="truncated"):
        so3.read_samples(str(tmp_path / "t.sofg"))
    (tmp_path / "l.sofg").write_bytes(gold[:-16])
    with pytest.raises(ValueError, match="does not match bandwidth"):
        so3.read_samples(str(tmp_path / "l.sofg"))
    nan = bytearray(gold)
    nan[12 + 16 * 7:12 + 16 * 7 + 8] = np.array([np.nan]).tobytes()
    (tmp_path / "n.sofg").write_bytes(bytes(nan))
    with pytest.raises(ValueError, match="non-finite"):
        so3.read_samples(str(tmp_path / "n.sofg"))
    with pytest.raises(ValueError, match="refusing to persist non-finite"):
        so3.write_samples(str(tmp_path / "w.sofg"), so3.So3SampleGrid(B, np.full(N ** 3, np.inf + 0j)))
    assert not (tmp_path / "w.sofg").exists()
    with pytest.raises(ValueError):
        so3.read_samples_slab(os.path.join(GOLD, "ref_b4.sofg"), 6, 4)
