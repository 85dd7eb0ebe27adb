"""SOFC / SOFG containers written by the REFERENCE itself (reference core.py:179-225), for the
byte-exactness tests of the streaming reader / writer (csrc/sofio.cuh).  TEST INFRASTRUCTURE
ONLY; run in the build container, where the read-only reference is mounted:

    python oracle/gen_sof_golden.py

Payloads: seeded N(0,1) complex128 (seed 4 for the B=4 grid, 5 for the B=4 coefficients).
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main() -> None:
    sys.path.insert(0, REF)
    import so3fft as sf
    b = 4
    n = 2 * b
    g = np.random.default_rng(4)
    grid = g.standard_normal(n ** 3) + 1j * g.standard_normal(n ** 3)
    c = np.random.default_rng(5)
    coeffs = c.standard_normal(sf.coeff_count(b)) + 1j * c.standard_normal(sf.coeff_count(b))
    sf.write_samples(os.path.join(OUT, "ref_b4.sofg"), sf.So3SampleGrid(b, grid))
    sf.write_coefficients(os.path.join(OUT, "ref_b4.sofc"), sf.So3Coefficients(b, coeffs))


if __name__ == "__main__":
    main()
