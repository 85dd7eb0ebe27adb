"""Sharded pipeline host logic on CPU: the C shard map and the all-to-all orchestration of
paper_1808_00896_b200.distributed, run with world_size 2 (and 4) over gloo, with numpy
stand-ins for the stage kernels; the gathered result must equal the single-process oracle."""
import multiprocessing as mp
import os
import socket
import traceback

import numpy as np
import pytest

from oracle import so3_oracle as O
from paper_1808_00896_b200.distributed import ShardedSO3, ShardMap


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, b, port, q, chunks=1):
    try:
        import torch
        import torch.distributed as dist
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from dist_helpers import NumpyShardBackend
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n = 2 * b
        rng = np.random.default_rng(b)
        grid = rng.standard_normal(n ** 3) + 1j * rng.standard_normal(n ** 3)
        sh = ShardedSO3(b, rank, world, NumpyShardBackend(b, world, rank, chunks))
        J = n // world
        slab = np.ascontiguousarray(grid.reshape(n, n, n)[:, rank * J:(rank + 1) * J, :]).reshape(-1)
        coeffs = sh.gather_coefficients(sh.fsoft(torch.from_numpy(slab.copy())))
        ref = O.fsoft(grid, b)
        err_f = float(np.abs(coeffs.numpy() - ref).max())
        back = sh.ifsoft(torch.from_numpy(ref.copy())).numpy()
        ref_g = O.ifsoft(ref, b).reshape(n, n, n)[:, rank * J:(rank + 1) * J, :].reshape(-1)
        err_i = float(np.abs(back - ref_g).max())
        dist.destroy_process_group()
        q.put((rank, err_f, err_i, None))
    except Exception:
        q.put((rank, None, None, traceback.format_exc()))


def _run(world, b, chunks=1):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, b, port, q, chunks)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ef, ei, tb in res:
        assert tb is None, tb
        assert ef < 1e-13 and ei < 1e-13, (rank, ef, ei)


@pytest.mark.parametrize("world,b", [(2, 4), (2, 6), (4, 8)])
def test_sharded_pipeline_matches_single_process(world, b):
    _run(world, b)


@pytest.mark.parametrize("world,b,chunks", [(2, 6, 2), (2, 8, 3), (4, 8, 4), (2, 3, 5), (1, 6, 1), (1, 8, 3)])
def test_chunked_exchange_pipeline_matches_single_process(world, b, chunks):
    """Exchange split into K chunks (async all_to_all per chunk, DWT per chunk), including
    chunks that are empty on some ranks (B=3, K=5)."""
    _run(world, b, chunks)


@pytest.mark.parametrize("b,world,chunks", [(8, 2, 3), (64, 8, 4), (512, 8, 8), (5, 2, 7)])
def test_chunk_map_is_a_partition_in_layout_order(b, world, chunks):
    m = ShardMap(b, world, chunks)
    assert sum(sum(r) for r in m.chunk_pairs) == (2 * b - 1) ** 2
    # chunk ranges tile layouts A and B exactly, in order
    ends_a = [m.chunk_a(q) for q in range(chunks)]
    assert ends_a[0][0] == 0 and ends_a[-1][1] == m.layout_a_rows() * m.J
    assert all(ends_a[q][1] == ends_a[q + 1][0] for q in range(chunks - 1))
    for r in range(world):
        ends_b = [m.chunk_b(r, q) for q in range(chunks)]
        assert ends_b[0][0] == 0 and ends_b[-1][1] == m.layout_b_rows(r) * m.J
        assert all(ends_b[q][1] == ends_b[q + 1][0] for q in range(chunks - 1))
        for q in range(chunks):
            assert sum(m.forward_send_splits(r, q)) == ends_a[q][1] - ends_a[q][0]
            assert sum(m.forward_recv_splits(r, q)) == ends_b[q][1] - ends_b[q][0]
    if b >= 64:   # chunks of one rank carry comparable DWT work (cost-balanced runs)
        from paper_1808_00896_b200 import cluster_schedule
        bases, mem = cluster_schedule(b)
        owner = m.cluster_owner()
        cost = mem.astype(np.int64) * (b - bases[:, 0]) + 1
        own0 = np.where(owner == 0)[0]
        cum = np.cumsum(cost[own0])
        q_of = np.minimum(chunks - 1, (np.concatenate([[0], cum[:-1]]) * chunks) // cum[-1])
        per = np.bincount(q_of, weights=cost[own0], minlength=chunks)
        assert per.max() / per.mean() < 1.25


@pytest.mark.parametrize("b,world", [(4, 1), (8, 2), (16, 4), (64, 8), (512, 8)])
def test_shard_map_partitions_pairs_and_balances(b, world):
    m = ShardMap(b, world)
    assert m.J * world == 2 * b
    pairs = [tuple(p) for r in range(world) for p in m.pair_list(r).tolist()]
    assert len(pairs) == len(set(pairs)) == (2 * b - 1) ** 2
    assert set(pairs) == {(x, y) for x in range(-b + 1, b) for y in range(-b + 1, b)}
    owner = m.cluster_owner()
    assert set(owner.tolist()) <= set(range(world))
    # cost balance of the LPT split (members * (B - m) per cluster)
    from paper_1808_00896_b200 import cluster_schedule
    bases, mem = cluster_schedule(b)
    cost = mem.astype(np.int64) * (b - bases[:, 0])
    load = np.bincount(owner, weights=cost, minlength=world)
    if b >= 64:
        assert load.max() / load.mean() < 1.01
    assert sum(m.forward_send_splits(0)) == (2 * b - 1) ** 2 * m.J
    for r in range(world):
        assert sum(m.forward_recv_splits(r)) == world * m.pairs[r] * m.J


def test_shard_map_rejects_indivisible_slabs():
    with pytest.raises(ValueError):
        ShardMap(3, 4)
