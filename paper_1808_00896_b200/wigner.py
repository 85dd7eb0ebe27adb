"""Wigner d- and D-functions at arbitrary angles (mirrors reference wigner.py).

The transforms never call these: the fast path regenerates its Wigner columns in registers
(csrc/dwt_mma.cuh).  They are the reference's evaluation utilities, kept so code and tests
written against ``so3fft.wigner`` run unchanged.  Every evaluation is a CUDA kernel
(csrc/direct.cuh: so3_jacobi_eval, so3_wigner_d_eval, so3_wigner_rows_eval); only argument
checks and the relation algebra (integer index / sign maps) run on the host.

Convention (wigner.py:1-30): d^1_{1,0}(beta) = +sin(beta)/sqrt(2); relations with ``reflect``
evaluate the base at pi - beta, which on the sampling grid is the reversed column order.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import validate_bandwidth

_BETA_SLACK = 1e-12   # wigner.py:40


def _torch():
    import torch
    return torch


def _device_eval(values: np.ndarray, out_shape: tuple, call) -> np.ndarray:
    """Upload `values` (float64) to the current CUDA device, run `call(ptr_in, count, ptr_out,
    stream)` and return the result on the host."""
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("so3fft_b200 needs a CUDA device (there is no CPU path)")
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64).reshape(-1)).to(dev)
    out = torch.empty(out_shape, dtype=torch.float64, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    call(ctypes.c_void_p(x.data_ptr()), x.numel(), ctypes.c_void_p(out.data_ptr()), stream)
    return out.cpu().numpy()


def _as_int(v, what: str) -> int:
    if isinstance(v, bool) or not isinstance(v, (int, np.integer)):
        raise ValueError(f"{what} must be an integer, got {v!r}")
    return int(v)


def jacobi_poly(n: int, a: float, b: float, x):
    """P_n^(a,b)(x) by the three-term recurrence (wigner.py:43-68); scalar or array x, |x| <= 1."""
    if isinstance(n, bool) or not isinstance(n, (int, np.integer)) or n < 0:
        raise ValueError(f"degree n must be a nonnegative integer, got {n!r}")
    if a <= -1.0 or b <= -1.0:
        raise ValueError(f"Jacobi exponents must exceed -1, got a={a}, b={b}")
    arr = np.asarray(x, dtype=np.float64)
    if np.any(np.abs(arr) > 1.0 + _BETA_SLACK):
        raise ValueError("Jacobi argument outside [-1, 1]")
    lib = _native.lib()
    out = _device_eval(arr, (arr.size,), lambda p, k, o, s: _native.check(
        lib.so3_jacobi_eval(int(n), float(a), float(b), p, k, o, s), "jacobi_poly"))
    return float(out[0]) if arr.ndim == 0 else out.reshape(arr.shape)


def _check_beta(beta) -> tuple[np.ndarray, bool]:
    """wigner.py:71-75."""
    arr = np.asarray(beta, dtype=np.float64)
    if np.any(arr < -_BETA_SLACK) or np.any(arr > math.pi + _BETA_SLACK):
        raise ValueError("beta outside [0, pi]")
    return arr, arr.ndim == 0


def wigner_d_direct(l: int, m: int, mp: int, beta):
    """d^l_{m,m'}(beta) from the closed form (wigner.py:92-114): canonicalisation onto m' >= |m|,
    then the Jacobi form, evaluated per angle on the GPU."""
    if l < 0 or abs(m) > l or abs(mp) > l:
        raise ValueError(f"invalid orders (l={l}, m={m}, m'={mp})")
    arr, scalar = _check_beta(beta)
    lib = _native.lib()
    out = _device_eval(arr, (arr.size,), lambda p, k, o, s: _native.check(
        lib.so3_wigner_d_eval(int(l), int(m), int(mp), p, k, o, s), "wigner_d_direct"))
    return float(out[0]) if scalar else out.reshape(arr.shape)


def wigner_d_rows(m: int, mp: int, betas: np.ndarray, bandwidth: int) -> np.ndarray:
    """(B - L, len(betas)) table d^l_{m,m'}(beta), l = L..B-1 (wigner.py:139-178): the degree
    seed and the three-term recurrence in l, one GPU thread per angle."""
    b = validate_bandwidth(bandwidth)
    low = max(abs(m), abs(mp))
    if low >= b:
        raise ValueError(f"order pair (m={m}, m'={mp}) has no degrees below B={b}")
    arr, _ = _check_beta(np.atleast_1d(betas))
    arr = arr.reshape(-1)
    lib = _native.lib()
    return _device_eval(arr, (b - low, arr.size), lambda p, k, o, s: _native.check(
        lib.so3_wigner_rows_eval(b, int(m), int(mp), p, k, o, s), "wigner_d_rows"))


def wigner_d_seed(m: int, mp: int, beta):
    """d^L_{m,m'}(beta) at L = max(|m|, |m'|) (wigner.py:117-136): row 0 of wigner_d_rows."""
    arr, scalar = _check_beta(beta)
    low = max(abs(m), abs(mp))
    row = wigner_d_rows(m, mp, arr.reshape(-1), low + 1)[0]
    return float(row[0]) if scalar else row.reshape(arr.shape)


@dataclass(frozen=True, eq=False)
class WignerColumn:
    """d^l_{m,m'}(beta) for l = max(|m|,|m'|)..B-1 at one angle (wigner.py:182-201)."""

    m: int
    mp: int
    beta: float
    bandwidth: int
    values: np.ndarray

    def __post_init__(self) -> None:
        low = max(abs(self.m), abs(self.mp))
        if self.values.shape != (self.bandwidth - low,):
            raise ValueError(f"column for (m={self.m}, m'={self.mp}) at B={self.bandwidth} "
                             f"must have {self.bandwidth - low} entries, got {self.values.shape}")

    @property
    def lowest_degree(self) -> int:
        return max(abs(self.m), abs(self.mp))


def wigner_d_column(m: int, mp: int, beta: float, bandwidth: int) -> WignerColumn:
    """Recurrence route at one angle (wigner.py:204-208)."""
    values = wigner_d_rows(m, mp, np.asarray([beta], dtype=np.float64), bandwidth)[:, 0]
    return WignerColumn(m, mp, float(beta), validate_bandwidth(bandwidth), values)


@dataclass(frozen=True)
class SymmetryRelation:
    """d^l_{target(m,m')}(beta) = (-1)^(sl l + sm m + smp m') d^l_{m,m'}(pi - beta if reflect
    else beta), target = (tm_m m + tm_mp m', tp_m m + tp_mp m') (wigner.py:211-241)."""

    tag: str
    reflect: bool
    sl: int
    sm: int
    smp: int
    tm_m: int
    tm_mp: int
    tp_m: int
    tp_mp: int

    def target(self, m: int, mp: int) -> tuple[int, int]:
        return (self.tm_m * m + self.tm_mp * mp, self.tp_m * m + self.tp_mp * mp)

    def sign(self, l: int, m: int, mp: int) -> float:
        return -1.0 if (self.sl * l + self.sm * m + self.smp * mp) % 2 else 1.0

    def sign_column(self, m: int, mp: int, bandwidth: int) -> np.ndarray:
        ls = np.arange(max(abs(m), abs(mp)), bandwidth)
        return np.where((self.sl * ls + self.sm * m + self.smp * mp) % 2 == 1, -1.0, 1.0)


# the order-pair symmetry group (wigner.py:244-256; eq. 2.8); the same table drives
# the CUDA Member derivation (csrc/common.cuh)
_RELATION_TABLE = (
    # tag                reflect sl sm smp  target (tm_m, tm_mp, tp_m, tp_mp)
    ("identity",          False, 0, 0, 0, (1, 0, 0, 1)),
    ("negate_both",       False, 0, 1, 1, (-1, 0, 0, -1)),
    ("swap",              False, 0, 1, 1, (0, 1, 1, 0)),
    ("swap_negate_both",  False, 0, 0, 0, (0, -1, -1, 0)),
    ("negate_m",          True,  1, 0, 1, (-1, 0, 0, 1)),
    ("negate_mp",         True,  1, 1, 0, (1, 0, 0, -1)),
    ("swap_negate_m",     True,  1, 0, 1, (0, -1, 1, 0)),
    ("swap_negate_mp",    True,  1, 1, 0, (0, 1, -1, 0)),
)
SYMMETRY_RELATIONS: dict[str, SymmetryRelation] = {
    tag: SymmetryRelation(tag, refl, sl, sm, smp, *tgt) for tag, refl, sl, sm, smp, tgt in _RELATION_TABLE
}


def apply_symmetry(column: WignerColumn, relation: SymmetryRelation) -> WignerColumn:
    """The related pair's column from a base column (wigner.py:259-264)."""
    new_m, new_mp = relation.target(column.m, column.mp)
    signs = relation.sign_column(column.m, column.mp, column.bandwidth)
    beta = math.pi - column.beta if relation.reflect else column.beta
    return WignerColumn(new_m, new_mp, beta, column.bandwidth, signs * column.values)


def wigner_D(l: int, m: int, mp: int, alpha: float, beta: float, gamma: float) -> complex:
    """D^l_{m,m'}(alpha, beta, gamma) = e^{-i m alpha} d^l_{m,m'}(beta) e^{-i m' gamma} (wigner.py:267-270)."""
    d = wigner_d_direct(l, m, mp, beta)
    return complex(np.exp(-1j * m * alpha) * d * np.exp(-1j * mp * gamma))
