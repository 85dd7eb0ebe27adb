"""Numpy stand-in for the four sharded stage kernels (test infrastructure: lets the gloo
tests run the real shard map + exchange orchestration of paper_1808_00896_b200.distributed
on CPU).  Layouts follow include/so3fft_b200.h: slab [i][jj][k], layout A rows
[g][pairs_g][J], layout B rows [h][pairs_rank][J]."""
import math

import numpy as np
import torch

from oracle import so3_oracle as O
from paper_1808_00896_b200 import cluster_schedule
from paper_1808_00896_b200.distributed import ShardMap


class NumpyShardBackend:
    def __init__(self, b: int, world: int, rank: int):
        self.b, self.world, self.rank = b, world, rank
        self.map = ShardMap(b, world)
        self.n, self.J = self.map.n, self.map.J
        self.jbase = rank * self.J
        lists = [self.map.pair_list(g) for g in range(world)]
        self.glob = {}
        off = 0
        for g in range(world):
            for p, (pm, pmp) in enumerate(lists[g].tolist()):
                self.glob[(pm, pmp)] = off + p
            off += len(lists[g])
        self.local = {tuple(x): p for p, x in enumerate(lists[rank].tolist())}
        bases, _ = cluster_schedule(b)
        owner = self.map.cluster_owner()
        self.clusters = [tuple(bases[i].tolist()) for i in range(len(bases)) if owner[i] == rank]
        self.betas = O.beta_nodes(b)
        self.w = O.beta_weights(b)
        self.v = (2.0 * np.arange(b) + 1.0) / (8.0 * math.pi * b)

    def empty(self, count):
        return torch.empty(count, dtype=torch.complex128)

    def zeros(self, count):
        return torch.zeros(count, dtype=torch.complex128)

    def fft_analysis(self, slab, send):
        n, J = self.n, self.J
        s = slab.numpy().reshape(n, J, n)
        out = send.numpy()
        for jj in range(J):
            S = O.slice_dft(s[:, jj, :], +1) * self.w[self.jbase + jj]
            for (pm, pmp), R in self.glob.items():
                out[R * J + jj] = S[pm % n, pmp % n]

    def fft_synthesis(self, recv, slab):
        n, J = self.n, self.J
        a = recv.numpy()
        s = slab.numpy().reshape(n, J, n)
        for jj in range(J):
            S = np.zeros((n, n), dtype=np.complex128)
            for (pm, pmp), R in self.glob.items():
                S[pm % n, pmp % n] = a[R * J + jj]
            s[:, jj, :] = O.slice_dft(S, -1)

    def dwt_analysis(self, recv, coeffs):
        P = len(self.local)
        r = recv.numpy().reshape(self.world, P, self.J)
        c = coeffs.numpy()
        ones = np.ones(self.n)
        for (bm, bmp) in self.clusters:
            rows = O.recurrence_rows(bm, bmp, self.betas, self.b)
            for (pm, pmp, tag) in O.cluster_members(bm, bmp):
                col = r[:, self.local[(pm, pmp)], :].reshape(-1)
                mat = O.member_matrix(rows, tag, bm, bmp, self.b)
                c[O.pair_slots(pm, pmp, self.b)] = O.analysis_column(mat, self.v[bm:], ones, col)

    def dwt_synthesis(self, coeffs, send):
        P = len(self.local)
        out = send.numpy().reshape(self.world, P, self.J)
        c = coeffs.numpy()
        for (bm, bmp) in self.clusters:
            rows = O.recurrence_rows(bm, bmp, self.betas, self.b)
            for (pm, pmp, tag) in O.cluster_members(bm, bmp):
                g = O.synthesis_column(O.member_matrix(rows, tag, bm, bmp, self.b), c[O.pair_slots(pm, pmp, self.b)])
                out[:, self.local[(pm, pmp)], :] = g.reshape(self.world, self.J)
