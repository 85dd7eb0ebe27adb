"""Extended-precision (x87 80-bit long double) restatement of the FSOFT / iFSOFT stages --
TEST INFRASTRUCTURE ONLY (accuracy diagnosis; imported by tools/parity_full.py and tests/).

The fp64 oracle (oracle/so3_oracle.py) is bit-identical to the reference, so comparing the GPU
with it measures the DIFFERENCE of two fp64 computations.  To say which of the two is closer to
the exact result, this module evaluates the same formulas with a 64-bit mantissa (11 more bits
than fp64):

* Wigner-d columns by the reference's three-term recurrence (wigner.py:139-178) with the seed
  (wigner.py:117-136) normalised through a 40-digit mpmath log-gamma;
* the relation signs and reflections of wigner.py:210-256 / dwt.py:76-93;
* per-cluster analysis v_l (T @ (w s)) and synthesis c @ T (dwt.py:109-125) with long-double
  quadrature weights (quadrature.py:66-73);
* the torus DFT of one beta slice (fft.py:72-76) by numpy's long-double pocketfft;
* one beta slice of the whole inverse transform (soft.py:152-173), vectorised over ALL clusters.

The recurrence in long double drifts by about 2^-11 of fp64's drift (fp64 reaches 3e-12
absolute at l = 511 against 50-digit values), so these values serve as "truth" for
fp64 errors down to ~1e-14 of the coefficient scale.
"""

from __future__ import annotations

import functools

import numpy as np

from . import so3_oracle as O

LD = np.longdouble
CLD = np.clongdouble


def _pi() -> LD:
    import mpmath
    mpmath.mp.dps = 40
    return LD(mpmath.nstr(mpmath.pi, 30))


def betas_ld(b: int) -> np.ndarray:
    """beta_j = (2j+1) pi / (4B) in long double (quadrature.py:61)."""
    j = np.arange(2 * b, dtype=LD)
    return (2 * j + 1) * _pi() / (4 * LD(b))


def weights_ld(b: int) -> np.ndarray:
    """w_B(j) = (2 pi / B^2) sin(beta_j) sum_{i<B} sin((2i+1) beta_j) / (2i+1) (quadrature.py:66-73)."""
    be = betas_ld(b)
    odd = 2 * np.arange(b, dtype=LD) + 1
    terms = np.sin(np.outer(be, odd)) / odd
    return (2 * _pi() / (LD(b) * LD(b))) * np.sin(be) * terms.sum(axis=1)


@functools.lru_cache(maxsize=None)
def log_norm(m: int, mp: int) -> LD:
    """log sqrt((2m)! / ((m+m')! (m-m')!)) for 0 <= m' <= m (wigner.py:124), 40 digits."""
    import mpmath
    mpmath.mp.dps = 40
    v = 0.5 * (mpmath.loggamma(2 * m + 1) - mpmath.loggamma(m + mp + 1) - mpmath.loggamma(m - mp + 1))
    return LD(mpmath.nstr(v, 30))


def base_rows_ld(m: int, mp: int, b: int, be: np.ndarray | None = None) -> np.ndarray:
    """d^l_{m,m'}(beta_j), l = m..B-1, base pair 0 <= m' <= m, long double (wigner.py:117-178)."""
    be = betas_ld(b) if be is None else be
    half = be / 2
    c, s = np.cos(half), np.sin(half)
    out = np.empty((b - m, be.shape[0]), dtype=LD)
    out[0] = np.exp(log_norm(m, mp) + (m + mp) * np.log(c) + (m - mp) * np.log(s))
    x = np.cos(be)
    older = np.zeros_like(x)
    now = out[0]
    for l in range(m, b - 1):
        lp = l + 1
        denom = np.sqrt(LD((lp * lp - m * m) * (lp * lp - mp * mp)))
        a = LD(lp * (2 * l + 1)) / denom
        if l == 0:
            shift, cc = LD(0), LD(0)
        else:
            shift = LD(m * mp) / LD(l * lp)
            cc = LD(lp) * np.sqrt(LD((l * l - m * m) * (l * l - mp * mp))) / (LD(l) * denom)
        new = a * (x - shift) * now - cc * older
        out[l + 1 - m] = new
        older, now = now, new
    return out


def member_rows_ld(rows: np.ndarray, tag: str, m: int, mp: int, b: int) -> np.ndarray:
    """Member matrix of a relation (dwt.py:76-93) in long double."""
    reflect, sl, sm, smp, _ = O.RELATIONS[tag]
    ls = np.arange(m, b)
    sign = (1 - 2 * ((sl * ls + sm * m + smp * mp) % 2)).astype(LD)
    vals = rows[:, ::-1] if reflect else rows
    return sign[:, None] * vals


def analysis_cluster_ld(b: int, bm: int, bmp: int, spectrum: np.ndarray) -> list[tuple[int, int, np.ndarray]]:
    """[(m, m', coefficients l = L..B-1)] of one cluster from the [m bin, j, m' bin] fp64
    spectrum (taken as exact), long double (soft.py:134-143, dwt.py:109-116)."""
    n = 2 * b
    rows = base_rows_ld(bm, bmp, b)
    w = weights_ld(b)
    ls = np.arange(bm, b, dtype=LD)
    v = (2 * ls + 1) / (8 * _pi() * LD(b))
    out = []
    for (m, mp, tag) in O.cluster_members(bm, bmp):
        mat = member_rows_ld(rows, tag, bm, bmp, b)
        s = spectrum[m % n, :, mp % n]
        ws_re = w * s.real.astype(LD)
        ws_im = w * s.imag.astype(LD)
        out.append((m, mp, v * (mat @ ws_re) + 1j * (v * (mat @ ws_im))))
    return out


def synthesis_cluster_ld(b: int, bm: int, bmp: int, coeffs: np.ndarray) -> list[tuple[int, int, np.ndarray]]:
    """[(m, m', spectrum column over j)] of one cluster, long double (soft.py:157-162, dwt.py:119-125)."""
    rows = base_rows_ld(bm, bmp, b)
    out = []
    for (m, mp, tag) in O.cluster_members(bm, bmp):
        mat = member_rows_ld(rows, tag, bm, bmp, b)
        c = coeffs[O.pair_slots(m, mp, b)]
        out.append((m, mp, c.real.astype(LD) @ mat + 1j * (c.imag.astype(LD) @ mat)))
    return out


def slice_dft_ld(plane: np.ndarray, sign: int) -> np.ndarray:
    """Unnormalised 2-D DFT exp(sign 2 pi i pq / n) of one slice in long double (fft.py:72-76)."""
    x = np.asarray(plane).astype(CLD)
    n0, n1 = x.shape
    if sign > 0:
        return np.fft.ifft2(x) * (n0 * n1)
    return np.fft.fft2(x)


def inverse_slice_ld(coeffs: np.ndarray, b: int, j: int) -> np.ndarray:
    """Slice j (alpha x gamma, n x n) of the inverse transform (soft.py:152-173), long double.

    Every cluster's Wigner column at beta_j and at its mirror beta_{n-1-j} (reflected members)
    is run by ONE recurrence vectorised over all clusters; the spectrum plane is then
    transformed by slice_dft_ld(-1).
    """
    n = 2 * b
    bases = np.array(O.base_pairs(b), dtype=np.int64)
    M, MP = bases[:, 0], bases[:, 1]
    be = betas_ld(b)
    bj = np.array([be[j], be[n - 1 - j]], dtype=LD)
    lnorm = np.array([log_norm(int(m), int(mp)) for m, mp in bases], dtype=LD)
    half = bj / 2
    lc, ls_ = np.log(np.cos(half)), np.log(np.sin(half))
    x = np.cos(bj)
    # d[cluster, 0 = beta_j / 1 = mirror] at the current degree of each cluster
    cur = np.exp(lnorm[:, None] + (M + MP)[:, None] * lc[None, :] + (M - MP)[:, None] * ls_[None, :])
    prev = np.zeros_like(cur)
    # flattened (cluster, member) table: every order pair exactly once
    ci_l, m_l, mp_l, refl_l, sl_l, s0_l = [], [], [], [], [], []
    for ci, (bm, bmp) in enumerate(bases):
        for (m, mp, tag) in O.cluster_members(int(bm), int(bmp)):
            reflect, sl, sm, smp, _ = O.RELATIONS[tag]
            ci_l.append(ci); m_l.append(m); mp_l.append(mp); refl_l.append(1 if reflect else 0)
            sl_l.append(sl); s0_l.append((sm * int(bm) + smp * int(bmp)) % 2)
    ci_a, m_a, mp_a = np.array(ci_l), np.array(m_l), np.array(mp_l)
    refl_a, sl_a, s0_a = np.array(refl_l), np.array(sl_l), np.array(s0_l)
    L_a = M[ci_a]
    row_a, col_a = m_a % n, mp_a % n
    c_re = coeffs.real.astype(LD)
    c_im = coeffs.imag.astype(LD)
    acc_re = np.zeros(ci_a.shape[0], dtype=LD)
    acc_im = np.zeros(ci_a.shape[0], dtype=LD)
    for l in range(b):
        if l > 0:
            adv = np.nonzero(M < l)[0]   # clusters already past their seed degree
            if adv.size:
                m, mp = M[adv].astype(LD), MP[adv].astype(LD)
                lm = LD(l - 1)
                lp = lm + 1
                denom = np.sqrt((lp * lp - m * m) * (lp * lp - mp * mp))
                a = lp * (2 * lm + 1) / denom
                if l - 1 == 0:
                    shift = np.zeros_like(m)
                    cc = np.zeros_like(m)
                else:
                    shift = m * mp / (lm * lp)
                    cc = lp * np.sqrt((lm * lm - m * m) * (lm * lm - mp * mp)) / (lm * denom)
                new = a[:, None] * (x[None, :] - shift[:, None]) * cur[adv] - cc[:, None] * prev[adv]
                prev[adv] = cur[adv]
                cur[adv] = new
        act = np.nonzero(L_a <= l)[0]
        d = cur[ci_a[act], refl_a[act]]
        sgn = (1 - 2 * ((sl_a[act] * l + s0_a[act]) % 2)).astype(LD)
        slots = l * (4 * l * l - 1) // 3 + (m_a[act] + l) * (2 * l + 1) + (mp_a[act] + l)
        acc_re[act] += sgn * d * c_re[slots]
        acc_im[act] += sgn * d * c_im[slots]
    plane = np.zeros((n, n), dtype=CLD)
    plane[row_a, col_a] = acc_re + 1j * acc_im
    return slice_dft_ld(plane, -1)
