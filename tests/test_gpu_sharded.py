"""CUDA sharded kernels (so3_shard_*), G ranks emulated sequentially in one process on one
GPU: each rank's FFT stage, the all-to-all done by device copies, each rank's DWT.  The
gathered result must be bit-identical to the single-GPU transform (same per-row FFTs and
per-cluster reductions whatever the split)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
so3 = pytest.importorskip("paper_1808_00896_b200")
from paper_1808_00896_b200.distributed import NativeShardBackend, ShardMap  # noqa: E402


def emulate(b, world, grid, coeffs):
    n = 2 * b
    m = ShardMap(b, world)
    J = m.J
    pref = np.concatenate([[0], np.cumsum(m.pairs)])
    be = [NativeShardBackend(b, world, r) for r in range(world)]
    cube = grid.reshape(n, n, n)
    # forward
    sends = []
    for r in range(world):
        slab = cube[:, r * J:(r + 1) * J, :].contiguous().reshape(-1)
        s = be[r].empty(m.layout_a_rows() * J)
        be[r].fft_analysis(slab, s)
        sends.append(s)
    out = torch.zeros_like(coeffs)
    for g in range(world):
        recv = torch.cat([sends[h][pref[g] * J:pref[g + 1] * J] for h in range(world)])
        c = be[g].zeros(out.numel())
        be[g].dwt_analysis(recv, c)
        out += c
    # inverse
    sends = []
    for g in range(world):
        s = be[g].empty(m.layout_b_rows(g) * J)
        be[g].dwt_synthesis(coeffs, s)
        sends.append(s)
    slabs = []
    for h in range(world):
        recv = torch.cat([sends[g][h * m.pairs[g] * J:(h + 1) * m.pairs[g] * J] for g in range(world)])
        slab = be[h].empty(n * J * n)
        be[h].fft_synthesis(recv, slab)
        slabs.append(slab.reshape(n, J, n))
    back = torch.cat(slabs, dim=1).reshape(-1)
    torch.cuda.synchronize()
    for x in be:
        x.release()
    return out, back


@pytest.mark.parametrize("b,world", [(8, 2), (16, 4), (33, 2), (64, 8), (128, 4)])
def test_sharded_equals_single_gpu_bitwise(b, world):
    n = 2 * b
    rng = np.random.default_rng(b + world)
    grid = torch.from_numpy(rng.standard_normal(n ** 3) + 1j * rng.standard_normal(n ** 3)).cuda()
    C = so3.coeff_count(b)
    coeffs = torch.from_numpy(rng.standard_normal(C) + 1j * rng.standard_normal(C)).cuda()
    plan = so3.make_plan(b)
    ref_f = so3.fsoft_sequential(so3.So3SampleGrid(b, grid), plan).data
    ref_i = so3.ifsoft_sequential(so3.So3Coefficients(b, coeffs), plan).data
    got_f, got_i = emulate(b, world, grid, coeffs)
    assert torch.equal(got_f, ref_f)
    assert torch.equal(got_i, ref_i)
