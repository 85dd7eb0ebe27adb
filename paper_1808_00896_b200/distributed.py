"""Sharded FSOFT / iFSOFT: one process per GPU, one all-to-all per direction.

The reference parallelises inside one host with a fork pool (schedule.py:200-257) and joins
its two stages with an in-memory transpose of the spectrum (soft.py:131-132, 142, 167).  Here
G ranks split

  * the torus FFT by beta slab  [rank*J, (rank+1)*J),  J = 2B / G  (the input/output samples
    of a rank are grid[:, slab, :], laid out [i][jj][k]);
  * the DWT by cost-balanced symmetry-cluster groups (LPT greedy over the launch schedule,
    computed by the C library: so3_shard_*);

and the transpose becomes ``torch.distributed.all_to_all_single`` (NCCL over NVLink on a
B200 box, gloo in the CPU tests), split into K chunks of clusters so the exchange overlaps
the DWT: forward, the all-to-alls of all chunks are queued behind the FFT and the DWT of
chunk q starts as soon as chunk q has arrived; inverse, chunk q is sent while chunk q+1 is
synthesised.  Pack and unpack are fused into the FFT kernels through a pair -> row table,
so the exchange moves the FFT output / DWT output buffers directly.  One exchange buffer per
direction holds both layouts:

  layout A  rows [chunk q][rank g][pairs_{g,q}][J]      forward send, inverse recv
  layout B  rows [chunk q][rank h][pairs_{rank,q}][J]   forward recv, inverse send

and the rank's own block exists in layout B only (the FFT writes / reads the own pairs there),
so the all-to-all carries the other ranks' blocks and no self copy.

Results are bit-identical for every G and K (the same per-row FFTs and per-cluster
reductions run whatever the split).  Coefficients stay sharded: a rank writes / reads only the slots of its
clusters in a full-length array; ``gather_coefficients`` all-reduces them (each slot has one
writer and zeros elsewhere, so the sum is exact).

The stage kernels are supplied by a backend; ``NativeShardBackend`` calls the CUDA library.
"""

from __future__ import annotations

import ctypes
from typing import Protocol

import numpy as np

from . import _native
from .core import coeff_count, grid_size, validate_bandwidth


class ShardMap:
    """Host-side shard map of G ranks and K exchange chunks (no GPU needed): pairs per
    (chunk, rank), slab width, all-to-all splits and buffer offsets."""

    def __init__(self, bandwidth: int, world: int, chunks: int = 1):
        self.bandwidth = validate_bandwidth(bandwidth)
        n = grid_size(self.bandwidth)
        if world < 1 or n % world:
            raise ValueError(f"2B={n} must be divisible by the number of ranks {world}")
        if not 1 <= chunks <= 64:
            raise ValueError(f"chunks must be in [1, 64], got {chunks}")
        self.world = world
        self.chunks = chunks
        self.n = n
        self.J = n // world
        counts = (ctypes.c_int64 * world)()
        _native.check(_native.lib().so3_shard_pair_counts(self.bandwidth, world, counts), "shard_pair_counts")
        self.pairs = [int(v) for v in counts]
        assert sum(self.pairs) == (n - 1) ** 2
        cp = (ctypes.c_int64 * (chunks * world))()
        _native.check(_native.lib().so3_shard_chunk_pairs(self.bandwidth, world, chunks, cp), "shard_chunk_pairs")
        # chunk_pairs[q][g]: pairs of rank g in chunk q
        self.chunk_pairs = [[int(cp[q * world + g]) for g in range(world)] for q in range(chunks)]
        assert [sum(self.chunk_pairs[q][g] for q in range(chunks)) for g in range(world)] == self.pairs

    def pair_list(self, rank: int) -> np.ndarray:
        out = np.empty((self.pairs[rank], 2), dtype=np.int32)
        _native.check(_native.lib().so3_shard_pair_list(
            self.bandwidth, self.world, rank, out.ctypes.data_as(_native._i32p)), "shard_pair_list")
        return out

    def cluster_owner(self) -> np.ndarray:
        k = int(_native.lib().so3_cluster_count(self.bandwidth))
        out = np.empty(k, dtype=np.int32)
        _native.check(_native.lib().so3_shard_cluster_owner(
            self.bandwidth, self.world, out.ctypes.data_as(_native._i32p)), "shard_cluster_owner")
        return out

    def layout_a_rows(self) -> int:
        return sum(self.pairs)

    def layout_b_rows(self, rank: int) -> int:
        return self.world * self.pairs[rank]

    # element ranges of chunk q (complex128 units)
    def chunk_a(self, q: int) -> tuple[int, int]:
        start = sum(sum(self.chunk_pairs[p]) for p in range(q)) * self.J
        return start, start + sum(self.chunk_pairs[q]) * self.J

    def chunk_b(self, rank: int, q: int) -> tuple[int, int]:
        start = self.world * sum(self.chunk_pairs[p][rank] for p in range(q)) * self.J
        return start, start + self.world * self.chunk_pairs[q][rank] * self.J

    # the exchange buffer of `rank`: layout A rows, then layout B rows (own block in B only)
    def exchange_rows(self, rank: int) -> int:
        return self.layout_a_rows() + self.layout_b_rows(rank)

    def a_block(self, q: int, g: int) -> tuple[int, int]:
        """element range of layout A block (chunk q, rank g) in the exchange buffer"""
        start = sum(sum(self.chunk_pairs[p]) for p in range(q)) + sum(self.chunk_pairs[q][:g])
        return start * self.J, (start + self.chunk_pairs[q][g]) * self.J

    def b_block(self, rank: int, q: int, h: int) -> tuple[int, int]:
        """element range of layout B block (chunk q, source slab h) in `rank`'s exchange buffer"""
        start = self.layout_a_rows() + self.world * sum(self.chunk_pairs[p][rank] for p in range(q)) \
            + h * self.chunk_pairs[q][rank]
        return start * self.J, (start + self.chunk_pairs[q][rank]) * self.J

    def b_chunk(self, rank: int, q: int) -> tuple[int, int]:
        """element range of layout B chunk q (all source slabs) in `rank`'s exchange buffer"""
        a0 = self.b_block(rank, q, 0)[0]
        return a0, a0 + self.world * self.chunk_pairs[q][rank] * self.J

    # all_to_all_single split sizes of chunk q, in complex128 elements
    def forward_send_splits(self, rank: int, q: int = 0) -> list[int]:
        if self.chunks == 1:
            return [p * self.J for p in self.pairs]
        return [p * self.J for p in self.chunk_pairs[q]]

    def forward_recv_splits(self, rank: int, q: int = 0) -> list[int]:
        own = self.pairs[rank] if self.chunks == 1 else self.chunk_pairs[q][rank]
        return [own * self.J] * self.world

    def inverse_send_splits(self, rank: int, q: int = 0) -> list[int]:
        return self.forward_recv_splits(rank, q)

    def inverse_recv_splits(self, rank: int, q: int = 0) -> list[int]:
        return self.forward_send_splits(rank, q)


class ShardBackend(Protocol):
    """The four stage kernels of one rank (buffer layouts above)."""

    def fft_analysis(self, slab, send_a) -> None: ...
    def dwt_analysis_chunk(self, q, recv_b_chunk, coeffs) -> None: ...
    def dwt_synthesis_chunk(self, q, coeffs, send_b_chunk) -> None: ...
    def fft_synthesis(self, recv_a, slab) -> None: ...
    def empty(self, count: int): ...
    def zeros(self, count: int): ...


class NativeShardBackend:
    """CUDA kernels of libso3fft_b200.so on the current device (torch complex128 tensors)."""

    def __init__(self, bandwidth: int, world: int, rank: int, device=None, chunks: int = 1):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            torch.empty(1, device=self.device)
            _native.check(_native.lib().so3_shard_plan_create_chunked(bandwidth, world, rank, chunks,
                                                                      ctypes.byref(handle)), "shard_plan_create")
        self.handle = handle
        self.chunks = chunks

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr())

    def fft_analysis(self, slab, send_a):
        _native.check(_native.lib().so3_shard_fft_analysis(self.handle, self._p(slab), self._p(send_a), self._stream()),
                      "shard_fft_analysis")

    def dwt_analysis(self, recv_b, coeffs):
        _native.check(_native.lib().so3_shard_dwt_analysis(self.handle, self._p(recv_b), self._p(coeffs), self._stream()),
                      "shard_dwt_analysis")

    def dwt_synthesis(self, coeffs, send_b):
        _native.check(_native.lib().so3_shard_dwt_synthesis(self.handle, self._p(coeffs), self._p(send_b), self._stream()),
                      "shard_dwt_synthesis")

    def dwt_analysis_chunk(self, q, recv_chunk, coeffs):
        _native.check(_native.lib().so3_shard_dwt_analysis_chunk(self.handle, q, self._p(recv_chunk), self._p(coeffs),
                                                                  self._stream()), "shard_dwt_analysis_chunk")

    def dwt_synthesis_chunk(self, q, coeffs, send_chunk):
        _native.check(_native.lib().so3_shard_dwt_synthesis_chunk(self.handle, q, self._p(coeffs), self._p(send_chunk),
                                                                   self._stream()), "shard_dwt_synthesis_chunk")

    def fft_synthesis(self, recv_a, slab):
        _native.check(_native.lib().so3_shard_fft_synthesis(self.handle, self._p(recv_a), self._p(slab), self._stream()),
                      "shard_fft_synthesis")

    def empty(self, count):
        return self.torch.empty(count, dtype=self.torch.complex128, device=self.device)

    def zeros(self, count):
        return self.torch.zeros(count, dtype=self.torch.complex128, device=self.device)

    def release(self):
        if self.handle is not None:
            _native.lib().so3_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.release()
        except Exception:
            pass


def _as_real(t):
    import torch
    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t


class ShardedSO3:
    """One rank of the sharded transform pair.  The backend's chunk count K (default 1) sets
    the pipelining of the exchange (see the module docstring)."""

    def __init__(self, bandwidth: int, rank: int, world: int, backend: ShardBackend, group=None, chunks=None):
        chunks = getattr(backend, "chunks", 1) if chunks is None else chunks
        self.map = ShardMap(bandwidth, world, chunks)
        self.bandwidth = self.map.bandwidth
        self.rank, self.world, self.chunks = rank, world, chunks
        self.backend = backend
        self.group = group
        self.coeff_count = coeff_count(self.bandwidth)
        self.slab_count = self.map.n * self.map.J * self.map.n

    def _exchange(self, ex, q: int, forward: bool):
        """One chunk of the all-to-all on the exchange buffer, the other ranks' blocks only
        (the own block already sits in layout B): forward sends layout A blocks (q, g) and
        receives layout B blocks (q, h); the inverse the reverse.  Grouped point-to-point
        operations (one NCCL group per chunk; gloo in the CPU tests), since a collective over
        all ranks would carry the self block.  Returns the pending works."""
        import torch.distributed as dist
        if self.world == 1:
            return []
        m, r = self.map, self.rank
        ops = []
        for peer in range(self.world):
            if peer == r:
                continue
            a = _as_real(ex[slice(*m.a_block(q, peer))])       # pairs of `peer`, this rank's slab
            b = _as_real(ex[slice(*m.b_block(r, q, peer))])    # this rank's pairs, slab of `peer`
            if forward:
                ops += [dist.P2POp(dist.isend, a, peer, self.group), dist.P2POp(dist.irecv, b, peer, self.group)]
            else:
                ops += [dist.P2POp(dist.isend, b, peer, self.group), dist.P2POp(dist.irecv, a, peer, self.group)]
        return dist.batch_isend_irecv(ops)

    def fsoft(self, slab, out=None):
        """This rank's beta slab [i][jj][k] -> coefficients: this rank's slots are written, the
        others are zero (a fresh array) or left as they are in ``out`` (reuse a buffer zeroed
        once to skip a full-length memset per call).
        All chunk exchanges are queued behind the FFT; the DWT of chunk q waits for chunk q
        only (on the device stream for NCCL), so it overlaps the exchange of chunks > q."""
        m, r = self.map, self.rank
        ex = self.backend.empty(m.exchange_rows(r) * m.J)
        self.backend.fft_analysis(slab, ex)
        works = [self._exchange(ex, q, forward=True) for q in range(self.chunks)]
        coeffs = self.backend.zeros(self.coeff_count) if out is None else out
        for q in range(self.chunks):
            for w in works[q]:
                w.wait()
            self.backend.dwt_analysis_chunk(q, ex[slice(*m.b_chunk(r, q))], coeffs)
        return coeffs

    def ifsoft(self, coeffs):
        """Coefficients (this rank's slots are read) -> this rank's beta slab [i][jj][k].
        Chunk q is exchanged while chunk q+1 is synthesised."""
        m, r = self.map, self.rank
        ex = self.backend.empty(m.exchange_rows(r) * m.J)
        works = []
        for q in range(self.chunks):
            self.backend.dwt_synthesis_chunk(q, coeffs, ex[slice(*m.b_chunk(r, q))])
            works.append(self._exchange(ex, q, forward=False))
        for ws in works:
            for w in ws:
                w.wait()
        slab = self.backend.empty(self.slab_count)
        self.backend.fft_synthesis(ex, slab)
        return slab

    def gather_coefficients(self, coeffs):
        """Full coefficient array on every rank (exact: one writer per slot)."""
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(_as_real(coeffs), group=self.group)
        return coeffs
