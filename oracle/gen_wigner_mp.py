"""High-precision Wigner-d golden values at B = 512 (test infrastructure).

The fp64 oracle restates the reference's three-term recurrence, so it cannot tell how
accurate that recurrence is at large degree.  This script evaluates d^l_{m,m'}(beta_j) on the
B = 512 quadrature nodes with mpmath at 50 significant digits, through the same
canonicalisation and Jacobi closed form as the reference's direct route (wigner.py:78-114,
oracle.closed_form_d), so the sign convention is the reference's (d^1_{1,0} = +sin(beta)/sqrt 2).
It also records how far the reference's own fp64 recurrence (oracle.recurrence_rows +
member_matrix, bit-identical to wigner.py:139-178 + dwt.py:76-93) lands from those values,
for comparison with the GPU recurrence in tests/test_gpu_parity.py.

    python oracle/gen_wigner_mp.py            # writes tests/golden/wigner_mp_b512.npz
"""
import os
import sys

import mpmath as mpm
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import so3_oracle as O  # noqa: E402

B = 512
PAIRS = [(0, 0), (1, 0), (5, 3), (-5, 3), (3, 5), (100, 50), (-100, -50), (255, 255), (511, 0),
         (300, 299), (400, -7), (50, -450)]
JS = [0, 1, 100, 511, 512, 700, 1022, 1023]
mpm.mp.dps = 50


def d_mp(l: int, m: int, mp: int, beta) -> mpm.mpf:
    if mp >= abs(m):
        sg, mu, nu = 1, m, mp
    elif -mp >= abs(m):
        sg, mu, nu = (-1) ** ((m - mp) & 1), -m, -mp
    elif m >= abs(mp):
        sg, mu, nu = (-1) ** ((m - mp) & 1), mp, m
    else:
        sg, mu, nu = 1, -mp, -m
    a, b, nd = nu - mu, mu + nu, l - nu
    pre = (-1) ** ((mu + nu) & 1) * mpm.sqrt(mpm.factorial(l + nu) * mpm.factorial(l - nu) /
                                             (mpm.factorial(l + mu) * mpm.factorial(l - mu)))
    h = beta / 2
    return sg * pre * mpm.sin(h) ** a * mpm.cos(h) ** b * mpm.jacobi(nd, a, b, mpm.cos(beta))


def main() -> None:
    rows = {"m": [], "mp": [], "l": [], "j": [], "value": [], "ref_fp64": []}
    betas64 = O.beta_nodes(B)
    for (m, mp) in PAIRS:
        lo = max(abs(m), abs(mp))
        ls = sorted({lo, lo + 1, lo + 10, (lo + B) // 2, B - 2, B - 1} & set(range(lo, B)))
        # the reference's fp64 rows for this pair: base recurrence + symmetry relation
        bm, bmp = max(abs(m), abs(mp)), min(abs(m), abs(mp))
        base = O.recurrence_rows(bm, bmp, betas64, B)
        tag = next(t for (pm, pq, t) in O.cluster_members(bm, bmp) if (pm, pq) == (m, mp))
        ref = O.member_matrix(base, tag, bm, bmp, B)
        for l in ls:
            for j in JS:
                beta = (2 * mpm.mpf(j) + 1) * mpm.pi / (4 * B)
                rows["m"].append(m)
                rows["mp"].append(mp)
                rows["l"].append(l)
                rows["j"].append(j)
                rows["value"].append(float(d_mp(l, m, mp, beta)))
                rows["ref_fp64"].append(float(ref[l - lo, j]))
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                       "wigner_mp_b512.npz")
    np.savez_compressed(out, **{k: np.asarray(v) for k, v in rows.items()})
    err = np.abs(np.asarray(rows["ref_fp64"]) - np.asarray(rows["value"]))
    print(f"{len(err)} entries; reference fp64 recurrence vs 50 digits: max abs {err.max():.3e}")


if __name__ == "__main__":
    main()
