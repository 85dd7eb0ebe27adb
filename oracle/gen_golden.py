"""Generate the golden fixtures in tests/golden/ by importing the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the read-only
reference is mounted:

    OMP_NUM_THREADS=1 python oracle/gen_golden.py

It imports ``so3fft`` from /root/reference/pkg/src (the Python reference, not
our oracle) and stores its outputs on seeded inputs.  The fixtures travel with
the repo; /root/reference does not exist on the GPU box.

Inputs follow BASELINE.json / SURVEY.md 8(d): complex128 coefficients with real
and imaginary parts i.i.d. N(0,1) from ``np.random.default_rng(seed)``
(``standard_normal(C)`` for the real part, then for the imaginary part).
"""

from __future__ import annotations

import os
import sys

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def seeded_coeffs(count: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal(count) + 1j * rng.standard_normal(count)


def main() -> None:
    sys.path.insert(0, REF)
    import so3fft as sf
    from so3fft.fft import transform_slice

    os.makedirs(OUT, exist_ok=True)
    # end-to-end: B in {1..5, 8 (configs[0]), 16}
    for b in (1, 2, 3, 4, 5, 6, 8, 16):
        plan = sf.make_plan(b)
        c = seeded_coeffs(sf.coeff_count(b), b)
        grid = sf.ifsoft_sequential(sf.So3Coefficients(b, c), plan).data
        back = sf.fsoft_sequential(sf.So3SampleGrid(b, grid), plan).data
        rng = np.random.default_rng(1000 + b)
        n = sf.grid_size(b) ** 3
        raw = rng.standard_normal(n) + 1j * rng.standard_normal(n)   # not band-limited
        fraw = sf.fsoft_sequential(sf.So3SampleGrid(b, raw), plan).data
        extra = {}
        if b <= 4:   # the reference's O(B^6) direct route (soft.py:212-256)
            extra["direct_inverse"] = sf.ifsoft_direct(sf.So3Coefficients(b, c)).data
            extra["direct_forward"] = sf.fsoft_direct(sf.So3SampleGrid(b, raw)).data
        np.savez_compressed(
            os.path.join(OUT, f"soft_b{b}.npz"),
            bandwidth=b, coeffs=c, inverse=grid, roundtrip=back, raw_grid=raw, forward_raw=fraw,
            weights=sf.quadrature_weights(b).values, betas=sf.sample_angles(b).betas, **extra,
        )
    # stage goldens: slice DFTs (fft.py:72-76), including non power-of-two lengths
    slices = {}
    for n in (1, 2, 4, 6, 8, 10, 16, 32, 64):
        rng = np.random.default_rng(50 + n)
        plane = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        slices[f"in_{n}"] = plane
        slices[f"plus_{n}"] = transform_slice(plane, +1)
        slices[f"minus_{n}"] = transform_slice(plane, -1)
    np.savez_compressed(os.path.join(OUT, "slices.npz"), **slices)
    # stage goldens: Wigner rows (wigner.py:139-178) and DWT columns (dwt.py:109-125)
    rows = {}
    for b in (16, 64):
        betas = sf.sample_angles(b).betas
        w = sf.quadrature_weights(b)
        for (m, mp) in [(0, 0), (1, 0), (3, 3), (5, 2), (b - 1, 0), (b - 1, b - 2), (b // 2, b // 3)]:
            base = sf.build_wigner_matrix(m, mp, b, betas)
            rows[f"rows_b{b}_{m}_{mp}"] = base.values
            cluster = sf.cluster_for_base(m, mp)
            mats = sf.derive_cluster_matrices(base, cluster)
            rng = np.random.default_rng(7 * b + m + 3 * mp)
            for pair, _ in cluster.members:
                s = rng.standard_normal(2 * b) + 1j * rng.standard_normal(2 * b)
                k = mats[pair].values.shape[0]
                cf = rng.standard_normal(k) + 1j * rng.standard_normal(k)
                sc = sf.make_scalers(pair.m, pair.mp, b, w)
                tag = f"b{b}_{pair.m}_{pair.mp}"
                rows[f"dwt_in_{tag}"] = s
                rows[f"dwt_out_{tag}"] = sf.dwt_apply(mats[pair], sc, s)
                rows[f"idwt_in_{tag}"] = cf
                rows[f"idwt_out_{tag}"] = sf.idwt_apply(mats[pair], cf)
    np.savez_compressed(os.path.join(OUT, "wigner.npz"), **rows)
    # schedule: kappa cluster order (schedule.py:136-153)
    sched = {}
    for b in (1, 2, 3, 4, 7, 8, 16, 33):
        sched[f"bases_b{b}"] = np.array([tuple(c.base) for c in sf.enumerate_clusters(b)], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "schedule.npz"), **sched)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
