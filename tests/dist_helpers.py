"""Numpy stand-in for the four sharded stage kernels (test infrastructure: lets the gloo
tests run the real shard map + exchange orchestration of paper_1808_00896_b200.distributed
on CPU).  Layouts follow include/so3fft_b200.h: slab [i][jj][k], layout A rows
[q][g][pairs_{g,q}][J], layout B rows [q][h][pairs_{rank,q}][J] (chunk-major), both in one
exchange buffer (A first) with the rank's own pairs in layout B only."""
import math

import numpy as np
import torch

from oracle import so3_oracle as O
from paper_1808_00896_b200 import cluster_schedule
from paper_1808_00896_b200.distributed import ShardMap


class NumpyShardBackend:
    def __init__(self, b: int, world: int, rank: int, chunks: int = 1):
        self.b, self.world, self.rank, self.chunks = b, world, rank, chunks
        self.map = ShardMap(b, world, chunks)
        self.n, self.J = self.map.n, self.map.J
        self.jbase = rank * self.J
        cp = self.map.chunk_pairs
        lists = [self.map.pair_list(g).tolist() for g in range(world)]   # layout order, chunk by chunk
        # layout A row of every pair: rows [q][g][pairs_{g,q}]
        self.glob, self.local = {}, {}
        row = 0
        off = [0] * world
        for q in range(chunks):
            for g in range(world):
                for i in range(cp[q][g]):
                    pair = tuple(lists[g][off[g] + i])
                    self.glob[pair] = row
                    row += 1
                    if g == rank:
                        self.local[pair] = (q, i)
                off[g] += cp[q][g]
        # exchange buffer = layout A then layout B: the own pairs live in layout B only
        for pair, (q, i) in self.local.items():
            self.glob[pair] = self.map.b_block(rank, q, rank)[0] // self.J + i
        bases, _ = cluster_schedule(b)
        owner = self.map.cluster_owner()
        self.clusters = [[] for _ in range(chunks)]
        for i in range(len(bases)):
            if owner[i] == rank:
                base = tuple(bases[i].tolist())
                self.clusters[self.local[base][0]].append(base)
        self.betas = O.beta_nodes(b)
        self.w = O.beta_weights(b)
        self.v = (2.0 * np.arange(b) + 1.0) / (8.0 * math.pi * b)

    def empty(self, count):
        return torch.empty(count, dtype=torch.complex128)

    def zeros(self, count):
        return torch.zeros(count, dtype=torch.complex128)

    def fft_analysis(self, slab, send):   # send: the exchange buffer
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

    def dwt_analysis_chunk(self, q, recv_chunk, coeffs):
        P = self.map.chunk_pairs[q][self.rank]
        r = recv_chunk.numpy().reshape(self.world, P, self.J)
        c = coeffs.numpy()
        ones = np.ones(self.n)
        for (bm, bmp) in self.clusters[q]:
            rows = O.recurrence_rows(bm, bmp, self.betas, self.b)
            for (pm, pmp, tag) in O.cluster_members(bm, bmp):
                col = r[:, self.local[(pm, pmp)][1], :].reshape(-1)
                mat = O.member_matrix(rows, tag, bm, bmp, self.b)
                c[O.pair_slots(pm, pmp, self.b)] = O.analysis_column(mat, self.v[bm:], ones, col)

    def dwt_synthesis_chunk(self, q, coeffs, send_chunk):
        P = self.map.chunk_pairs[q][self.rank]
        out = send_chunk.numpy().reshape(self.world, P, self.J)
        c = coeffs.numpy()
        for (bm, bmp) in self.clusters[q]:
            rows = O.recurrence_rows(bm, bmp, self.betas, self.b)
            for (pm, pmp, tag) in O.cluster_members(bm, bmp):
                g = O.synthesis_column(O.member_matrix(rows, tag, bm, bmp, self.b), c[O.pair_slots(pm, pmp, self.b)])
                out[:, self.local[(pm, pmp)][1], :] = g.reshape(self.world, self.J)
