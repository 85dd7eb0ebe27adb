"""CPU oracle for the FSOFT / iFSOFT hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the arithmetic of the reference package
``so3fft`` (arXiv 1808.00896 Python reference, mounted read-only at
/root/reference when this file was written).  It is the *checker* for the CUDA
path and the CPU baseline (``bench.py --impl reference``, kind "port").  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
reference arm may import it.  The product package ``paper_1808_00896_b200``
never imports it and has no CPU fallback.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/so3fft).  The arithmetic is kept in the same order as
the reference (same numpy expressions for every rounding step) so the oracle is
bit-identical to the reference on the same machine; ``tests/test_oracle.py``
pins that claim against the golden vectors in ``tests/golden/`` that
``oracle/gen_golden.py`` produced by importing the reference itself.
"""

from __future__ import annotations

import math
import os
from math import lgamma

import numpy as np

__all__ = [
    "n_coeffs", "slot", "pair_slots", "beta_nodes", "angle_nodes", "beta_weights",
    "dft_lastaxis", "slice_dft", "seed_column", "recurrence_rows", "base_pairs",
    "cluster_members", "RELATIONS", "member_matrix", "analysis_column",
    "synthesis_column", "fsoft", "ifsoft", "fsoft_direct", "ifsoft_direct",
    "closed_form_d", "error_metrics", "degree_of_slot", "fft_analysis_stage", "dwt_analysis_stage",
    "dwt_synthesis_stage", "fft_synthesis_stage",
]


# ---------------------------------------------------------------------------
# layouts (core.py:43-74)
# ---------------------------------------------------------------------------

def n_coeffs(b: int) -> int:
    """B(4B^2-1)/3 -- core.py:48-51."""
    return b * (4 * b * b - 1) // 3


def slot(l: int, m: int, mp: int) -> int:
    """l-major slot of (l, m, m') -- core.py:54-61."""
    return l * (4 * l * l - 1) // 3 + (m + l) * (2 * l + 1) + (mp + l)


def pair_slots(m: int, mp: int, b: int) -> np.ndarray:
    """Slots of l = max(|m|,|m'|)..B-1 for one order pair -- core.py:64-74."""
    ls = np.arange(max(abs(m), abs(mp)), b, dtype=np.int64)
    return ls * (4 * ls * ls - 1) // 3 + (m + ls) * (2 * ls + 1) + (mp + ls)


def degree_of_slot(b: int) -> np.ndarray:
    """Degree l of every slot (used for the 1/(1+l) smooth-density inputs)."""
    return np.concatenate([np.full((2 * l + 1) ** 2, l, dtype=np.int64) for l in range(b)])


# ---------------------------------------------------------------------------
# grid and quadrature (quadrature.py:57-73)
# ---------------------------------------------------------------------------

def angle_nodes(b: int) -> np.ndarray:
    """alpha_i = gamma_i = i*pi/B -- quadrature.py:59-63."""
    idx = np.arange(2 * b, dtype=np.float64)
    return idx * math.pi / b


def beta_nodes(b: int) -> np.ndarray:
    """beta_j = (2j+1)*pi/(4B) -- quadrature.py:61."""
    idx = np.arange(2 * b, dtype=np.float64)
    return (2.0 * idx + 1.0) * math.pi / (4.0 * b)


def beta_weights(b: int) -> np.ndarray:
    """w_B(j) = (2pi/B^2) sin(beta_j) sum_i sin((2i+1)beta_j)/(2i+1) -- quadrature.py:66-73."""
    betas = beta_nodes(b)
    odd = 2.0 * np.arange(b, dtype=np.float64) + 1.0
    terms = np.sin(np.outer(betas, odd)) / odd
    return (2.0 * math.pi / (b * b)) * np.sin(betas) * terms.sum(axis=1)


# ---------------------------------------------------------------------------
# torus DFT (fft.py:28-76)
# ---------------------------------------------------------------------------

def _bitrev(n: int) -> np.ndarray:
    """Bit-reversal permutation built by doubling -- fft.py:28-32."""
    perm = np.zeros(1, dtype=np.intp)
    while perm.shape[0] < n:
        perm = np.concatenate([2 * perm, 2 * perm + 1])
    return perm


def dft_lastaxis(x: np.ndarray, sign: int) -> np.ndarray:
    """Unnormalised DFT exp(sign*2pi*i*pq/n) along the last axis -- fft.py:35-54.

    Power-of-two n: bit-reversal gather then in-place radix-2 merges with
    twiddles exp(sign*2pi*i*k/size); other n: product with the kernel matrix.
    """
    n = x.shape[-1]
    if n == 1:
        return x.copy()
    if n & (n - 1):
        g = np.arange(n)
        return x @ np.exp(sign * 2j * np.pi * np.outer(g, g) / n)
    y = np.ascontiguousarray(x[..., _bitrev(n)])
    span = 2
    while span <= n:
        h = span // 2
        tw = np.exp(sign * 2j * np.pi * np.arange(h) / span)
        view = y.reshape(y.shape[:-1] + (n // span, span))
        t = view[..., h:] * tw
        view[..., h:] = view[..., :h] - t
        view[..., :h] += t
        span *= 2
    return y


def _dft_along(x: np.ndarray, sign: int, axis: int) -> np.ndarray:
    """fft.py:57-59."""
    moved = np.moveaxis(np.asarray(x, dtype=np.complex128), axis, -1)
    return np.moveaxis(dft_lastaxis(moved, sign), -1, axis)


def slice_dft(plane: np.ndarray, sign: int) -> np.ndarray:
    """2-D DFT of one beta slice, alpha axis first then gamma -- fft.py:72-76."""
    return _dft_along(_dft_along(plane, sign, 0), sign, 1)


# ---------------------------------------------------------------------------
# Wigner-d (wigner.py:117-178, 210-256)
# ---------------------------------------------------------------------------

def seed_column(m: int, mp: int, betas: np.ndarray) -> np.ndarray:
    """d^L_{m,m'}(beta) at L = max(|m|,|m'|), product form -- wigner.py:117-136."""
    half = 0.5 * np.asarray(betas, dtype=np.float64)
    c, s = np.cos(half), np.sin(half)
    if abs(m) >= abs(mp):
        k = abs(m)
        norm = math.exp(0.5 * (lgamma(2 * k + 1) - lgamma(k + mp + 1) - lgamma(k - mp + 1)))
        if m >= 0:
            return norm * c ** (k + mp) * s ** (k - mp)
        return norm * c ** (k - mp) * (-s) ** (k + mp)
    k = abs(mp)
    norm = math.exp(0.5 * (lgamma(2 * k + 1) - lgamma(k + m + 1) - lgamma(k - m + 1)))
    if mp >= 0:
        return norm * c ** (k + m) * (-s) ** (k - m)
    return norm * c ** (k - m) * s ** (k + m)


def recurrence_coeffs(l: int, m: int, mp: int) -> tuple[float, float, float]:
    """(a_l, shift_l, c_l) of the three-term recurrence -- wigner.py:165-174."""
    lp = l + 1
    denom = math.sqrt((lp * lp - m * m) * (lp * lp - mp * mp))
    a = lp * (2 * l + 1) / denom
    if l == 0:
        return a, 0.0, 0.0
    shift = (m * mp) / (l * lp)
    c = lp * math.sqrt((l * l - m * m) * (l * l - mp * mp)) / (l * denom)
    return a, shift, c


def recurrence_rows(m: int, mp: int, betas: np.ndarray, b: int) -> np.ndarray:
    """Rows d^l_{m,m'}(beta), l = L..B-1 -- wigner.py:139-178.

    d^{l+1} = a_l (cos(beta) - shift_l) d^l - c_l d^{l-1}, d^{L-1} = 0.
    """
    lo = max(abs(m), abs(mp))
    betas = np.atleast_1d(np.asarray(betas, dtype=np.float64))
    out = np.empty((b - lo, betas.shape[0]), dtype=np.float64)
    out[0] = seed_column(m, mp, betas)
    if b - lo == 1:
        return out
    x = np.cos(betas)
    older = np.zeros_like(x)
    now = out[0]
    for l in range(lo, b - 1):
        a, shift, c = recurrence_coeffs(l, m, mp)
        new = a * (x - shift) * now - c * older
        out[l + 1 - lo] = new
        older, now = now, new
    return out


# relation tag -> (reflect, sl, sm, smp, target matrix (tm_m, tm_mp, tp_m, tp_mp))
# wigner.py:244-256
RELATIONS: dict[str, tuple[bool, int, int, int, tuple[int, int, int, int]]] = {
    "identity":         (False, 0, 0, 0, (1, 0, 0, 1)),
    "negate_both":      (False, 0, 1, 1, (-1, 0, 0, -1)),
    "swap":             (False, 0, 1, 1, (0, 1, 1, 0)),
    "swap_negate_both": (False, 0, 0, 0, (0, -1, -1, 0)),
    "negate_m":         (True, 1, 0, 1, (-1, 0, 0, 1)),
    "negate_mp":        (True, 1, 1, 0, (1, 0, 0, -1)),
    "swap_negate_m":    (True, 1, 0, 1, (0, -1, 1, 0)),
    "swap_negate_mp":   (True, 1, 1, 0, (0, 1, -1, 0)),
}

# schedule.py:115-120
_TAGS = {
    "origin": ("identity",),
    "axis": ("identity", "negate_both", "swap", "swap_negate_both"),
    "diagonal": ("identity", "negate_both", "negate_m", "negate_mp"),
    "full": ("identity", "negate_both", "swap", "swap_negate_both",
             "negate_m", "negate_mp", "swap_negate_m", "swap_negate_mp"),
}


def cluster_kind(m: int, mp: int) -> str:
    """schedule.py:123-133."""
    if m == 0:
        return "origin"
    if mp == 0:
        return "axis"
    if mp == m:
        return "diagonal"
    return "full"


def cluster_members(m: int, mp: int) -> list[tuple[int, int, str]]:
    """(member m, member m', relation tag) for the base pair 0 <= m' <= m -- schedule.py:107-133."""
    out = []
    for tag in _TAGS[cluster_kind(m, mp)]:
        t = RELATIONS[tag][4]
        out.append((t[0] * m + t[1] * mp, t[2] * m + t[3] * mp, tag))
    return out


def base_pairs(b: int) -> list[tuple[int, int]]:
    """Cluster bases in kappa order -- schedule.py:59-90, 136-153."""
    out = [(0, 0)] + [(m, 0) for m in range(1, b)] + [(m, m) for m in range(1, b)]
    rows = (b - 1) // 2
    for kappa in range((b - 1) * (b - 2) // 2):
        i, j = kappa // (b - 1) + 1, kappa % (b - 1) + 1
        assert 1 <= i <= rows
        out.append((b - i, b - j) if j > i else (i + 1, j))
    return out


def sign_column(tag: str, m: int, mp: int, b: int) -> np.ndarray:
    """(-1)^(sl*l + sm*m + smp*m') for l = L..B-1 -- wigner.py:234-241."""
    _, sl, sm, smp, _ = RELATIONS[tag]
    ls = np.arange(max(abs(m), abs(mp)), b)
    return 1.0 - 2.0 * ((sl * ls + sm * m + smp * mp) % 2)


def member_matrix(base_rows: np.ndarray, tag: str, m: int, mp: int, b: int) -> np.ndarray:
    """Member matrix = signs x (base with columns reversed if reflect) -- dwt.py:76-93."""
    vals = base_rows[:, ::-1] if RELATIONS[tag][0] else base_rows
    return sign_column(tag, m, mp, b)[:, None] * vals


def analysis_column(mat: np.ndarray, v: np.ndarray, w: np.ndarray, s: np.ndarray) -> np.ndarray:
    """v * (T @ (w * s)) -- dwt.py:109-116."""
    return v * (mat @ (w * s))


def synthesis_column(mat: np.ndarray, c: np.ndarray) -> np.ndarray:
    """c @ T -- dwt.py:119-125."""
    return c @ mat


# ---------------------------------------------------------------------------
# pipelines (soft.py:124-173)
# ---------------------------------------------------------------------------

class _Plan:
    """Per-bandwidth tables -- soft.py:80-108 (streaming policy)."""

    def __init__(self, b: int):
        self.b = b
        self.n = 2 * b
        self.betas = beta_nodes(b)
        self.w = beta_weights(b)
        ls = np.arange(b, dtype=np.float64)
        self.v = (2.0 * ls + 1.0) / (8.0 * math.pi * b)
        self.bases = base_pairs(b)


_PLANS: dict[int, _Plan] = {}


def _plan(b: int) -> _Plan:
    if b not in _PLANS:
        _PLANS[b] = _Plan(b)
    return _PLANS[b]


def _forward_block(b: int, bm: int, bmp: int, spectrum: np.ndarray) -> np.ndarray:
    """One analyze() work item: a stacked (members, B-L) block -- soft.py:134-143."""
    p = _plan(b)
    n = p.n
    lo = max(bm, bmp)
    rows = recurrence_rows(bm, bmp, p.betas, b)
    members = cluster_members(bm, bmp)
    block = np.empty((len(members), b - lo), dtype=np.complex128)
    for r, (m, mp, tag) in enumerate(members):
        block[r] = analysis_column(member_matrix(rows, tag, bm, bmp, b), p.v[lo:], p.w, spectrum[m % n, :, mp % n])
    return block


def _inverse_block(b: int, bm: int, bmp: int, flat: np.ndarray) -> np.ndarray:
    """One synthesize() work item: a stacked (members, 2B) block -- soft.py:157-162."""
    p = _plan(b)
    rows = recurrence_rows(bm, bmp, p.betas, b)
    members = cluster_members(bm, bmp)
    block = np.empty((len(members), p.n), dtype=np.complex128)
    for r, (m, mp, tag) in enumerate(members):
        block[r] = synthesis_column(member_matrix(rows, tag, bm, bmp, b), flat[pair_slots(m, mp, b)])
    return block


# Worker state inherited by the forked pool (schedule.py:189-196, 235-248): only item
# indices go to the workers and only results come back, as in the reference's run_items.
_FORK_STATE = None


def _one_blas_thread() -> None:
    """Pool initializer: one BLAS thread per forked worker (the reference's CPU plan pins
    OMP/OPENBLAS/MKL_NUM_THREADS=1; without it every worker's matvecs oversubscribe the cores)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl missing
        pass


def _invoke_item(index: int):
    worker, items = _FORK_STATE
    return index, worker(items[index])


def _pool_map(fn, items, workers):
    """run_items (schedule.py:200-257): plain loop for one worker, else a fork pool with
    dynamic imap_unordered batches of len // (8 workers) items, results put back in order."""
    global _FORK_STATE
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(it) for it in items]
    import multiprocessing as mp
    if _FORK_STATE is not None:
        raise RuntimeError("nested parallel oracle map is not supported")
    chunk = max(1, len(items) // (workers * 8))
    out = [None] * len(items)
    _FORK_STATE = (fn, items)
    try:
        with mp.get_context("fork").Pool(processes=workers, initializer=_one_blas_thread) as pool:
            for index, res in pool.imap_unordered(_invoke_item, range(len(items)), chunksize=chunk):
                out[index] = res
    finally:
        _FORK_STATE = None
    return out


def fft_analysis_stage(grid: np.ndarray, b: int, workers: int = 1, slices=None, out=None) -> np.ndarray:
    """Per-slice sign +1 DFTs into the [m bin, j, m' bin] spectrum -- soft.py:127-132.

    ``slices`` (optional) restricts the stage to those beta indices and ``out`` receives them
    (bounded CPU-baseline samples); other slices of ``out`` are left as they are.
    """
    n = 2 * b
    cube = np.asarray(grid, dtype=np.complex128).reshape(n, n, n)
    spectrum = np.empty((n, n, n), dtype=np.complex128) if out is None else out
    js = list(range(n)) if slices is None else list(slices)
    planes = _pool_map(lambda j: slice_dft(cube[:, j, :], +1), js, workers)
    for j, plane in zip(js, planes):
        spectrum[:, j, :] = plane
    return spectrum


def dwt_analysis_stage(spectrum: np.ndarray, b: int, workers: int = 1, clusters=None, out=None) -> np.ndarray:
    """Per-cluster forward DWT and scatter into l-major slots -- soft.py:134-148.

    ``clusters`` (optional) restricts the stage to a subset of base pairs; untouched slots are
    NaN, or left as they are in ``out``.
    """
    p = _plan(b)
    bases = p.bases if clusters is None else [tuple(c) for c in clusters]
    blocks = _pool_map(lambda bp: _forward_block(b, bp[0], bp[1], spectrum), bases, workers)
    if out is None:
        out = np.full(n_coeffs(b), np.nan + 0j) if clusters is not None else np.empty(n_coeffs(b), np.complex128)
    for (bm, bmp), block in zip(bases, blocks):
        for (m, mp, _), col in zip(cluster_members(bm, bmp), block):
            out[pair_slots(m, mp, b)] = col
    return out


def dwt_synthesis_stage(coeffs: np.ndarray, b: int, workers: int = 1, clusters=None, out=None) -> np.ndarray:
    """Per-cluster inverse DWT into the [m bin, j, m' bin] spectrum, Nyquist bins zero -- soft.py:154-167.

    ``clusters`` (optional) restricts the stage to a subset of base pairs (other rows stay zero,
    or as they are in ``out``).
    """
    p = _plan(b)
    n = p.n
    flat = np.asarray(coeffs, dtype=np.complex128)
    bases = p.bases if clusters is None else [tuple(c) for c in clusters]
    blocks = _pool_map(lambda bp: _inverse_block(b, bp[0], bp[1], flat), bases, workers)
    spectrum = np.zeros((n, n, n), dtype=np.complex128) if out is None else out
    for (bm, bmp), block in zip(bases, blocks):
        for (m, mp, _), col in zip(cluster_members(bm, bmp), block):
            spectrum[m % n, :, mp % n] = col
    return spectrum


def fft_synthesis_stage(spectrum: np.ndarray, b: int, workers: int = 1, slices=None, out=None) -> np.ndarray:
    """Per-slice sign -1 DFTs into the flat [i, j, k] grid -- soft.py:169-173 (``slices`` / ``out``
    as in fft_analysis_stage)."""
    n = 2 * b
    cube = np.empty((n, n, n), dtype=np.complex128) if out is None else out.reshape(n, n, n)
    js = list(range(n)) if slices is None else list(slices)
    planes = _pool_map(lambda j: slice_dft(spectrum[:, j, :], -1), js, workers)
    for j, plane in zip(js, planes):
        cube[:, j, :] = plane
    return cube.reshape(-1)


def fsoft(grid: np.ndarray, b: int, workers: int = 1, clusters=None) -> np.ndarray:
    """Forward transform of a flat (2B)^3 [i,j,k] grid -> l-major coefficients -- soft.py:124-149.

    ``clusters`` (optional) restricts the DWT stage to a subset of base pairs
    (bounded CPU-baseline samples); untouched slots are left as NaN.
    """
    return dwt_analysis_stage(fft_analysis_stage(grid, b, workers), b, workers, clusters)


def ifsoft(coeffs: np.ndarray, b: int, workers: int = 1) -> np.ndarray:
    """Inverse transform of l-major coefficients -> flat (2B)^3 grid -- soft.py:152-173."""
    return fft_synthesis_stage(dwt_synthesis_stage(coeffs, b, workers), b, workers)


# ---------------------------------------------------------------------------
# direct O(B^6) route (wigner.py:43-114, soft.py:212-256) -- independent check
# ---------------------------------------------------------------------------

def _jacobi(nd: int, a: float, bb: float, x: np.ndarray) -> np.ndarray:
    """P_n^(a,b)(x) by the standard recurrence -- wigner.py:43-68."""
    p0 = np.ones_like(x)
    if nd == 0:
        return p0
    p1 = 0.5 * (a - bb) + 0.5 * (a + bb + 2.0) * x
    for k in range(2, nd + 1):
        s = 2.0 * k + a + bb
        c1 = 2.0 * k * (k + a + bb) * (s - 2.0)
        c2 = (s - 1.0) * s * (s - 2.0)
        c3 = (s - 1.0) * (a * a - bb * bb)
        c4 = 2.0 * (k + a - 1.0) * (k + bb - 1.0) * s
        p1, p0 = ((c2 * x + c3) * p1 - c4 * p0) / c1, p1
    return p1


def closed_form_d(l: int, m: int, mp: int, beta) -> np.ndarray:
    """d^l_{m,m'}(beta) through canonicalisation + Jacobi closed form -- wigner.py:78-114."""
    beta = np.asarray(beta, dtype=np.float64)
    if mp >= abs(m):
        sg, mu, nu = 1.0, m, mp
    elif -mp >= abs(m):
        sg, mu, nu = (-1.0) ** (m - mp), -m, -mp
    elif m >= abs(mp):
        sg, mu, nu = (-1.0) ** (m - mp), mp, m
    else:
        sg, mu, nu = 1.0, -mp, -m
    a, bb, nd = nu - mu, mu + nu, l - nu
    lr = 0.5 * (lgamma(l + nu + 1) + lgamma(l - nu + 1) - lgamma(l + mu + 1) - lgamma(l - mu + 1))
    pre = (-1.0) ** (mu + nu) * math.exp(lr)
    h = 0.5 * beta
    return sg * (pre * np.sin(h) ** a * np.cos(h) ** bb * _jacobi(nd, a, bb, np.cos(beta)))


def fsoft_direct(grid: np.ndarray, b: int) -> np.ndarray:
    """Analysis sum evaluated coefficient by coefficient -- soft.py:212-233."""
    n = 2 * b
    cube = np.asarray(grid, dtype=np.complex128).reshape(n, n, n)
    al, be, w = angle_nodes(b), beta_nodes(b), beta_weights(b)
    out = np.empty(n_coeffs(b), dtype=np.complex128)
    k = 0
    for l in range(b):
        scale = (2 * l + 1) / (8.0 * math.pi * b)
        for m in range(-l, l + 1):
            ea = np.exp(1j * m * al)
            for mp in range(-l, l + 1):
                eg = np.exp(1j * mp * al)
                d = closed_form_d(l, m, mp, be)
                ker = ea[:, None, None] * (w * d)[None, :, None] * eg[None, None, :]
                out[k] = scale * np.sum(cube * ker)
                k += 1
    return out


def ifsoft_direct(coeffs: np.ndarray, b: int) -> np.ndarray:
    """Pointwise synthesis -- soft.py:236-256."""
    n = 2 * b
    al, be = angle_nodes(b), beta_nodes(b)
    cube = np.zeros((n, n, n), dtype=np.complex128)
    k = 0
    for l in range(b):
        for m in range(-l, l + 1):
            ea = np.conj(np.exp(1j * m * al))
            for mp in range(-l, l + 1):
                eg = np.conj(np.exp(1j * mp * al))
                d = closed_form_d(l, m, mp, be)
                cube += coeffs[k] * (ea[:, None, None] * d[None, :, None] * eg[None, None, :])
                k += 1
    return cube.reshape(-1)


# ---------------------------------------------------------------------------
# metrics (bench.py:122-131)
# ---------------------------------------------------------------------------

def error_metrics(ref: np.ndarray, got: np.ndarray) -> tuple[float, float]:
    """(max |got-ref|, max per-slot |got-ref|/|ref| over nonzero ref) -- bench.py:122-131."""
    diff = np.abs(np.asarray(got) - np.asarray(ref))
    mag = np.abs(ref)
    nz = mag > 0.0
    return (float(diff.max()) if diff.size else 0.0,
            float((diff[nz] / mag[nz]).max()) if np.any(nz) else 0.0)


def default_workers() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
