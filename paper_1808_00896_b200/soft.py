"""Drop-in FSOFT / iFSOFT on B200: plans and transforms (mirrors reference soft.py).

Reference surface kept (pkg/src/so3fft/soft.py):
    make_plan(bandwidth, matrix_policy="streaming", partitioner="kappa")   soft.py:80-108
    fsoft_sequential(samples, plan) / fsoft_parallel(samples, plan, threads) soft.py:176-183
    ifsoft_sequential(coeffs, plan) / ifsoft_parallel(coeffs, plan, threads) soft.py:186-193
Every transform runs the CUDA path of libso3fft_b200.so (include/so3fft_b200.h);
there is no CPU path.  ``threads`` is validated like the reference
(schedule.py:216-217) and otherwise has no effect: results are identical for
every value, which is the reference's own guarantee (soft.py:7-10).

Input/output types follow the input: numpy in -> numpy out (host buffers,
copied in and out by the library, the reference's contract); torch complex128
CUDA tensors in -> torch tensors out on the same device, on the current stream.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from collections.abc import Mapping
from typing import Any, NamedTuple

import numpy as np

from . import _native
from .wigner import SYMMETRY_RELATIONS
from .core import (
    So3Coefficients,
    So3SampleGrid,
    _is_torch,
    coeff_count,
    degree_scale,
    grid_size,
    order_pair_slots,
    validate_bandwidth,
)

_MATRIX_POLICIES = ("streaming", "precomputed")
_PARTITIONERS = ("kappa", "sigma")


class OrderPair(NamedTuple):
    m: int
    mp: int


# relation tags per cluster kind, reference schedule.py:115-120
_TAGS = {
    "origin": ("identity",),
    "axis": ("identity", "negate_both", "swap", "swap_negate_both"),
    "diagonal": ("identity", "negate_both", "negate_m", "negate_mp"),
    "full": ("identity", "negate_both", "swap", "swap_negate_both",
             "negate_m", "negate_mp", "swap_negate_m", "swap_negate_mp"),
}


class SymmetryCluster(NamedTuple):
    """Base pair and its orbit (reference schedule.py:93-103); members are (pair, SymmetryRelation)."""
    kind: str
    base: OrderPair
    members: tuple


def cluster_for_base(m: int, mp: int) -> SymmetryCluster:
    """reference schedule.py:123-133."""
    if not 0 <= mp <= m:
        raise ValueError(f"base pair must satisfy 0 <= m' <= m, got ({m}, {mp})")
    kind = "origin" if m == 0 else "axis" if mp == 0 else "diagonal" if mp == m else "full"
    members = []
    for tag in _TAGS[kind]:
        rel = SYMMETRY_RELATIONS[tag]
        members.append((OrderPair(*rel.target(m, mp)), rel))
    return SymmetryCluster(kind, OrderPair(m, mp), tuple(members))


# ---- the paper's remapping of the order-pair triangle onto flat work indices --------------
# sigma: row-major triangle 0 <= m' <= m (schedule.py:40-52); kappa: the strict lower triangle
# 1 <= m' < m <= B-1 folded into a (B-1)/2 x (B-1) rectangle so that an integer divmod
# splits it (schedule.py:55-90).

def sigma_index(m: int, mp: int) -> int:
    """Triangle index of a pair with 0 <= m' <= m (reference schedule.py:40-44)."""
    if not 0 <= mp <= m:
        raise ValueError(f"require 0 <= m' <= m, got (m={m}, m'={mp})")
    return m * (m + 1) // 2 + mp


def sigma_inverse(sigma: int) -> OrderPair:
    """Inverse of sigma_index by the same floating-point closed form (schedule.py:47-52)."""
    if sigma < 0:
        raise ValueError(f"sigma must be >= 0, got {sigma}")
    m = int(math.floor(math.sqrt(2.0 * sigma + 0.25) - 0.5))
    return OrderPair(m, sigma - m * (m + 1) // 2)


def rect_to_orders(i: int, j: int, bandwidth: int) -> OrderPair:
    """Rectangle cell (i, j), 1 <= i <= (B-1)//2, 1 <= j <= B-1 -> strict-lower-triangle
    pair (schedule.py:59-70).  Cells right of the diagonal fold onto the far corner."""
    b = validate_bandwidth(bandwidth)
    rows = (b - 1) // 2
    if not 1 <= i <= rows:
        raise ValueError(f"row i={i} outside [1, {rows}] for B={b}")
    if not 1 <= j <= b - 1:
        raise ValueError(f"column j={j} outside [1, {b - 1}] for B={b}")
    if b % 2 == 1 and i == rows and j > rows:
        raise ValueError(f"cell (i={i}, j={j}) beyond the half row of odd B={b}")
    return OrderPair(b - i, b - j) if j > i else OrderPair(i + 1, j)


def kappa_count(bandwidth: int) -> int:
    """(B-1)(B-2)/2 strict-lower-triangle pairs (schedule.py:73-76)."""
    b = validate_bandwidth(bandwidth)
    return (b - 1) * (b - 2) // 2


def kappa_split(kappa: int, bandwidth: int) -> tuple[int, int]:
    """Integer split of a work index into its rectangle cell (schedule.py:79-84)."""
    b = validate_bandwidth(bandwidth)
    if not 0 <= kappa < kappa_count(b):
        raise ValueError(f"kappa={kappa} outside [0, {kappa_count(b)}) for B={b}")
    return kappa // (b - 1) + 1, kappa % (b - 1) + 1


def kappa_to_orders(kappa: int, bandwidth: int) -> OrderPair:
    """Base order pair of work index kappa (schedule.py:87-90)."""
    i, j = kappa_split(kappa, bandwidth)
    return rect_to_orders(i, j, bandwidth)


def enumerate_clusters(bandwidth: int, partitioner: str = "kappa") -> list[SymmetryCluster]:
    """All symmetry clusters below B in the reference's order (schedule.py:136-158).

    "kappa": origin, axis, diagonal, then the kappa rectangle; "sigma": triangle order.
    The GPU launch order is cluster_schedule(); both cover the (2B-1)^2 order pairs
    exactly once.
    """
    b = validate_bandwidth(bandwidth)
    if partitioner == "kappa":
        bases = [(0, 0)] + [(m, 0) for m in range(1, b)] + [(m, m) for m in range(1, b)]
        bases += [tuple(kappa_to_orders(k, b)) for k in range(kappa_count(b))]
    elif partitioner == "sigma":
        bases = [tuple(sigma_inverse(s)) for s in range(b * (b + 1) // 2)]
    else:
        raise ValueError(f"unknown partitioner {partitioner!r}")
    return [cluster_for_base(m, mp) for m, mp in bases]


@dataclass(frozen=True, eq=False)
class SampleAngles:
    """Per-axis angles of the grid (reference quadrature.py:26-39)."""
    bandwidth: int
    alphas: np.ndarray = field(repr=False)
    betas: np.ndarray = field(repr=False)
    gammas: np.ndarray = field(repr=False)


@dataclass(frozen=True, eq=False)
class QuadratureWeights:
    """Beta weights w_B(j) (reference quadrature.py:42-54)."""
    bandwidth: int
    values: np.ndarray = field(repr=False)


def sample_angles(bandwidth: int) -> SampleAngles:
    """alpha_i = gamma_i = i pi / B, beta_j = (2j+1) pi / (4B) (quadrature.py:57-63), from the C library."""
    b = validate_bandwidth(bandwidth)
    al = np.empty(2 * b)
    be = np.empty(2 * b)
    _native.check(_native.lib().so3_sample_angles(b, _dptr(al), _dptr(be)), "sample_angles")
    return SampleAngles(b, al, be, al.copy())


def quadrature_weights(bandwidth: int) -> QuadratureWeights:
    """w_B(j) (quadrature.py:66-73), computed by the C library in long double."""
    b = validate_bandwidth(bandwidth)
    w = np.empty(2 * b)
    _native.check(_native.lib().so3_quadrature_weights(b, _dptr(w)), "quadrature_weights")
    return QuadratureWeights(b, w)


def cluster_schedule(bandwidth: int) -> tuple[np.ndarray, np.ndarray]:
    """GPU launch order of the symmetry clusters: (bases int32 [K,2], member counts int32 [K])."""
    b = validate_bandwidth(bandwidth)
    k = int(_native.lib().so3_cluster_count(b))
    bases = np.empty((k, 2), dtype=np.int32)
    mem = np.empty(k, dtype=np.int32)
    _native.check(_native.lib().so3_cluster_schedule(
        b, bases.ctypes.data_as(_native._i32p), mem.ctypes.data_as(_native._i32p)), "cluster_schedule")
    return bases, mem


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_native._dp)


def _torch():
    import torch
    return torch


def _resolve_device(device):
    """'cuda' / None -> the CURRENT CUDA device (torch's own convention), 'cuda:k' / k -> device k."""
    torch = _torch()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    if d.type != "cuda":
        raise ValueError(f"so3fft_b200 plans live on a CUDA device, got {device!r}")
    return torch.device("cuda", torch.cuda.current_device() if d.index is None else d.index)


class _MatrixTable(Mapping):
    """plan.matrices of a "precomputed" plan (soft.py:100-106): OrderPair -> WignerMatrix of every
    order pair, computed on access by the GPU recurrence (dwt.build_wigner_matrix +
    derive_cluster_matrices) and cached per cluster for the last few clusters."""

    def __init__(self, plan):
        self._plan = plan
        self._cache: dict = {}

    def __getitem__(self, pair):
        from .dwt import build_wigner_matrix, derive_cluster_matrices
        m, mp = int(pair[0]), int(pair[1])
        b = self._plan.bandwidth
        if max(abs(m), abs(mp)) >= b:
            raise KeyError(pair)
        base = (max(abs(m), abs(mp)), min(abs(m), abs(mp)))
        if base not in self._cache:
            if len(self._cache) >= 8:
                self._cache.pop(next(iter(self._cache)))
            mats = derive_cluster_matrices(build_wigner_matrix(*base, b, self._plan.angles.betas),
                                           cluster_for_base(*base))
            self._cache[base] = mats
        return self._cache[base][OrderPair(m, mp)]

    def __iter__(self):
        b = self._plan.bandwidth
        return (OrderPair(m, mp) for m in range(-b + 1, b) for mp in range(-b + 1, b))

    def __len__(self):
        return (2 * self._plan.bandwidth - 1) ** 2


class TransformPlan:
    """Reusable per-bandwidth GPU state (reference soft.py:56-77).

    Holds the native plan (beta tables, weights, twiddles, cluster schedule,
    scratch spectrum) on one CUDA device.  ``matrix_policy`` is accepted for API
    compatibility; Wigner matrices are never stored (they are regenerated in
    registers by the recurrence), so "precomputed" computes the same values; its
    ``matrices`` mapping serves each pair's matrix on access instead of storing the table.
    """

    def __init__(self, bandwidth: int, matrix_policy: str, partitioner: str, batch: int, device):
        torch = _torch()
        self.bandwidth = bandwidth
        self.matrix_policy = matrix_policy
        self.partitioner = partitioner
        self.batch = batch
        if not torch.cuda.is_available():
            raise RuntimeError("so3fft_b200 needs a CUDA device (there is no CPU path)")
        self.device = _resolve_device(device)
        self.angles = sample_angles(bandwidth)
        # "precomputed": the per-pair matrices are served on access (GPU recurrence), never
        # stored -- the reference's table is 1.47 TB at B = 512, and the kernels regenerate the
        # rows in registers faster than they could stream them
        self.matrices = _MatrixTable(self) if matrix_policy == "precomputed" else None
        self.weights = quadrature_weights(bandwidth)
        self.degree_scale = degree_scale(bandwidth)
        self._clusters = None
        self._slot_table = None
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            torch.empty(1, device=self.device)   # make the primary context current
            _native.check(_native.lib().so3_plan_create(bandwidth, batch, ctypes.byref(handle)), "make_plan")
        self._handle = handle
        self.n_clusters = int(_native.lib().so3_cluster_count(bandwidth))

    # -- reference attributes, built lazily (O(B^2) Python objects / O(B^3) ints)
    @property
    def clusters(self) -> list[SymmetryCluster]:
        if self._clusters is None:
            self._clusters = enumerate_clusters(self.bandwidth, self.partitioner)
        return self._clusters

    @property
    def work_items(self) -> list[tuple[int, SymmetryCluster]]:
        return list(enumerate(self.clusters))

    @property
    def slot_table(self) -> dict:
        if self._slot_table is None:
            self._slot_table = {pair: order_pair_slots(pair.m, pair.mp, self.bandwidth)
                                for c in self.clusters for pair, _ in c.members}
        return self._slot_table

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._handle is None:
            raise ValueError("plan has been released")
        return self._handle

    def set_dwt_variant(self, variant: str) -> None:
        """DWT kernel family: "mma" (default: FP64 DMMA) or "simt" (DFMA + warp butterfly)."""
        code = {"mma": 0, "simt": 1}.get(variant)
        if code is None:
            raise ValueError(f"unknown DWT variant {variant!r}")
        _native.check(_native.lib().so3_plan_set_dwt_variant(self.handle, code), "set_dwt_variant")

    def set_knob(self, name: str, value: int) -> None:
        """Tuning knob of the native plan (see include/so3fft_b200.h so3_plan_set_knob)."""
        _native.check(_native.lib().so3_plan_set_knob(self.handle, name.encode(), int(value)), "set_knob")

    @property
    def device_bytes(self) -> int:
        return int(_native.lib().so3_plan_device_bytes(self.handle))

    def release(self) -> None:
        if getattr(self, "_handle", None) is not None:
            _native.lib().so3_plan_destroy(self._handle)
            self._handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.release()
        except Exception:
            pass

    def __repr__(self) -> str:
        return (f"TransformPlan(bandwidth={self.bandwidth}, batch={self.batch}, device={self.device}, "
                f"matrix_policy={self.matrix_policy!r}, partitioner={self.partitioner!r})")


def make_plan(bandwidth: int, matrix_policy: str = "streaming", partitioner: str = "kappa", *,
              batch: int = 1, device=None) -> TransformPlan:
    """Build the reusable plan for one bandwidth (reference soft.py:80-108).

    Extensions: ``batch`` functions per call (configs' B=32 x 64 case) and
    ``device`` (default: the current CUDA device).
    """
    b = validate_bandwidth(bandwidth)
    if matrix_policy not in _MATRIX_POLICIES:
        raise ValueError(f"matrix_policy must be one of {_MATRIX_POLICIES}, got {matrix_policy!r}")
    if partitioner not in _PARTITIONERS:
        raise ValueError(f"unknown partitioner {partitioner!r}")
    if isinstance(batch, bool) or not isinstance(batch, (int, np.integer)) or batch < 1:
        raise ValueError(f"batch must be an integer >= 1, got {batch!r}")
    return TransformPlan(b, matrix_policy, partitioner, int(batch), device)


def _check_plan(data_bandwidth: int, plan: TransformPlan, what: str) -> int:
    """reference soft.py:118-121."""
    if data_bandwidth != plan.bandwidth:
        raise ValueError(f"{what} bandwidth {data_bandwidth} does not match plan bandwidth {plan.bandwidth}")
    return plan.bandwidth


def _check_threads(threads) -> None:
    """reference schedule.py:216-217."""
    if isinstance(threads, bool) or not isinstance(threads, (int, np.integer)) or threads < 1:
        raise ValueError(f"threads must be an integer >= 1, got {threads!r}")


def _stream(plan: TransformPlan):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(plan.device).cuda_stream)


def _device_buffer(t, count: int, plan: TransformPlan, what: str):
    """A caller-supplied device buffer the kernels read or write ``count`` complex128 (or, for
    float buffers, float64) elements of: checked before its pointer crosses the C ABI."""
    torch = _torch()
    if not _is_torch(t) or not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if t.device != plan.device:
        raise ValueError(f"{what} on {t.device}, plan on {plan.device}")
    if t.dtype != torch.complex128:
        raise ValueError(f"{what} must be complex128, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if t.numel() != count:
        raise ValueError(f"{what} must hold {count} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


def _disjoint(a, a_bytes: int, b, b_bytes: int, what: str) -> None:
    pa = a.data_ptr() if _is_torch(a) else a.ctypes.data
    pb = b.data_ptr() if _is_torch(b) else b.ctypes.data
    if pa < pb + b_bytes and pb < pa + a_bytes:
        raise ValueError(f"{what}: output must not overlap the input")


def _run(plan: TransformPlan, data, out_count: int, dev_fn: str, host_fn: str, out=None):
    """Dispatch a whole transform on device tensors or host arrays (batch-aware)."""
    torch = _torch()
    lib = _native.lib()
    total = out_count * plan.batch
    if _is_torch(data):
        if not data.is_cuda:
            data = data.to(plan.device)
        if data.device != plan.device:
            raise ValueError(f"data on {data.device}, plan on {plan.device}")
        data = data.contiguous()
        if data.dtype != torch.complex128:
            raise ValueError("device data must be complex128")
        if out is None:
            out = torch.empty(total, dtype=torch.complex128, device=plan.device)
        else:
            _device_buffer(out, total, plan, "out")
            _disjoint(out, 16 * total, data, 16 * data.numel(), dev_fn)
        with torch.cuda.device(plan.device):
            _native.check(getattr(lib, dev_fn)(plan.handle, ctypes.c_void_p(data.data_ptr()),
                                               ctypes.c_void_p(out.data_ptr()), _stream(plan)), dev_fn)
        return out
    arr = np.ascontiguousarray(data, dtype=np.complex128)
    if out is None:
        out = np.empty(total, dtype=np.complex128)
    else:
        if not isinstance(out, np.ndarray) or out.dtype != np.complex128 or not out.flags.c_contiguous \
                or not out.flags.writeable or out.size != total:
            raise ValueError(f"out must be a writeable C-contiguous complex128 numpy array of {total} elements")
        _disjoint(out, 16 * total, arr, 16 * arr.size, host_fn)
    with torch.cuda.device(plan.device):
        _native.check(getattr(lib, host_fn)(plan.handle, ctypes.c_void_p(arr.ctypes.data),
                                            ctypes.c_void_p(out.ctypes.data), _stream(plan)), host_fn)
    return out


def _fsoft(samples: So3SampleGrid, plan: TransformPlan, out=None) -> So3Coefficients:
    b = _check_plan(samples.bandwidth, plan, "sample")
    if plan.batch != 1:
        raise ValueError(f"plan is for batch={plan.batch}; use fsoft_batch")
    n = grid_size(b)
    data = samples.data
    if (data.shape[0] if hasattr(data, "shape") else len(data)) != n ** 3:
        raise ValueError(f"sample data must have length {n ** 3}")
    res = _run(plan, data, coeff_count(b), "so3_fsoft", "so3_fsoft_host", out)
    return So3Coefficients(b, res)


def _ifsoft(coeffs: So3Coefficients, plan: TransformPlan, out=None) -> So3SampleGrid:
    b = _check_plan(coeffs.bandwidth, plan, "coefficient")
    if plan.batch != 1:
        raise ValueError(f"plan is for batch={plan.batch}; use ifsoft_batch")
    data = coeffs.data
    if (data.shape[0] if hasattr(data, "shape") else len(data)) != coeff_count(b):
        raise ValueError(f"coefficient data must have length {coeff_count(b)}")
    res = _run(plan, data, grid_size(b) ** 3, "so3_ifsoft", "so3_ifsoft_host", out)
    return So3SampleGrid(b, res)


def fsoft_sequential(samples: So3SampleGrid, plan: TransformPlan, *, out=None) -> So3Coefficients:
    """Forward transform (reference soft.py:176-178)."""
    return _fsoft(samples, plan, out)


def fsoft_parallel(samples: So3SampleGrid, plan: TransformPlan, threads: int, *, out=None) -> So3Coefficients:
    """Forward transform; identical values for every ``threads`` (reference soft.py:181-183)."""
    _check_threads(threads)
    return _fsoft(samples, plan, out)


def ifsoft_sequential(coeffs: So3Coefficients, plan: TransformPlan, *, out=None) -> So3SampleGrid:
    """Inverse transform (reference soft.py:186-188)."""
    return _ifsoft(coeffs, plan, out)


def ifsoft_parallel(coeffs: So3Coefficients, plan: TransformPlan, threads: int, *, out=None) -> So3SampleGrid:
    """Inverse transform; identical values for every ``threads`` (reference soft.py:191-193)."""
    _check_threads(threads)
    return _ifsoft(coeffs, plan, out)


def fsoft_batch(samples, plan: TransformPlan, *, out=None):
    """Forward transform of plan.batch functions: samples (batch, (2B)^3) -> (batch, C(B))."""
    b = plan.bandwidth
    flat = samples.reshape(-1)
    if flat.shape[0] != plan.batch * grid_size(b) ** 3:
        raise ValueError(f"expected {plan.batch} x {grid_size(b) ** 3} samples")
    res = _run(plan, flat, coeff_count(b), "so3_fsoft", "so3_fsoft_host", out)
    return res.reshape(plan.batch, coeff_count(b))


def ifsoft_batch(coeffs, plan: TransformPlan, *, out=None):
    """Inverse transform of plan.batch functions: (batch, C(B)) -> (batch, (2B)^3)."""
    b = plan.bandwidth
    flat = coeffs.reshape(-1)
    if flat.shape[0] != plan.batch * coeff_count(b):
        raise ValueError(f"expected {plan.batch} x {coeff_count(b)} coefficients")
    res = _run(plan, flat, grid_size(b) ** 3, "so3_ifsoft", "so3_ifsoft_host", out)
    return res.reshape(plan.batch, grid_size(b) ** 3)


# ------------------------------------------------------------------ stages (device tensors only)

def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _grid_count(plan: TransformPlan) -> int:
    return plan.batch * grid_size(plan.bandwidth) ** 3


def _coef_count(plan: TransformPlan) -> int:
    return plan.batch * coeff_count(plan.bandwidth)


def fft_analysis(plan: TransformPlan, samples, spectrum) -> None:
    """K1: weighted torus spectrum spectrum[f][m'][m][j] of device samples (fft.py:72-76, soft.py:130-132)."""
    ps = _device_buffer(samples, _grid_count(plan), plan, "samples")
    pz = _device_buffer(spectrum, _grid_count(plan), plan, "spectrum")
    with _torch().cuda.device(plan.device):
        _native.check(_native.lib().so3_fft_analysis(plan.handle, ps, pz, _stream(plan)), "fft_analysis")


def fft_synthesis(plan: TransformPlan, spectrum, samples) -> None:
    """K4: samples from spectrum[f][m'][m][j] (soft.py:164-172); spectrum is read only."""
    pz = _device_buffer(spectrum, _grid_count(plan), plan, "spectrum")
    ps = _device_buffer(samples, _grid_count(plan), plan, "samples")
    with _torch().cuda.device(plan.device):
        _native.check(_native.lib().so3_fft_synthesis(plan.handle, pz, ps, _stream(plan)), "fft_synthesis")


def dwt_analysis(plan: TransformPlan, spectrum, coeffs, begin: int = 0, end: int | None = None) -> None:
    """K2: forward DWT of clusters [begin, end) of the launch schedule (dwt.py:109-116)."""
    end = plan.n_clusters if end is None else end
    pz = _device_buffer(spectrum, _grid_count(plan), plan, "spectrum")
    pc = _device_buffer(coeffs, _coef_count(plan), plan, "coeffs")
    with _torch().cuda.device(plan.device):
        _native.check(_native.lib().so3_dwt_analysis(plan.handle, pz, pc, begin, end, _stream(plan)), "dwt_analysis")


def dwt_synthesis(plan: TransformPlan, coeffs, spectrum, begin: int = 0, end: int | None = None) -> None:
    """K3: inverse DWT of clusters [begin, end) (dwt.py:119-125)."""
    end = plan.n_clusters if end is None else end
    pc = _device_buffer(coeffs, _coef_count(plan), plan, "coeffs")
    pz = _device_buffer(spectrum, _grid_count(plan), plan, "spectrum")
    with _torch().cuda.device(plan.device):
        _native.check(_native.lib().so3_dwt_synthesis(plan.handle, pc, pz, begin, end, _stream(plan)), "dwt_synthesis")


def wigner_rows(plan: TransformPlan, m: int, mp: int):
    """d^l_{m,m'}(beta_j) for l = L..B-1 on the plan's grid, from the GPU recurrence
    (wigner_d_rows wigner.py:139-178 + derive_cluster_matrices dwt.py:76-93): (B-L, 2B) float64 tensor."""
    torch = _torch()
    b = plan.bandwidth
    lo = max(abs(m), abs(mp))
    if lo >= b:
        raise ValueError(f"order pair (m={m}, m'={mp}) has no degrees below B={b}")
    out = torch.empty((b - lo, 2 * b), dtype=torch.float64, device=plan.device)
    with _torch().cuda.device(plan.device):
        _native.check(_native.lib().so3_wigner_rows(plan.handle, m, mp, _ptr(out), _stream(plan)), "wigner_rows")
    return out


# ------------------------------------------------------------------ direct transforms (oracle route)

DIRECT_BANDWIDTH_CAP = 12


def _direct(data, bandwidth: int, max_bandwidth: int, out_count: int, fn: str):
    """soft.py:196-201 cap semantics; runs the CUDA direct kernels on the current device."""
    torch = _torch()
    if bandwidth > max_bandwidth:
        raise ValueError(f"direct transform capped at B={max_bandwidth} (got B={bandwidth}); "
                         "raise max_bandwidth explicitly if you really want this")
    host = not _is_torch(data)
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(np.ascontiguousarray(data, dtype=np.complex128)).to(dev) if host else data.contiguous()
    out = torch.empty(out_count, dtype=torch.complex128, device=x.device)
    with torch.cuda.device(x.device):
        _native.check(getattr(_native.lib(), fn)(bandwidth, ctypes.c_void_p(x.data_ptr()),
                                                 ctypes.c_void_p(out.data_ptr()),
                                                 ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)), fn)
    return out.cpu().numpy() if host else out


def fsoft_direct(samples: So3SampleGrid, max_bandwidth: int = DIRECT_BANDWIDTH_CAP) -> So3Coefficients:
    """Reference forward transform evaluated as the defining sum on the GPU (soft.py:212-233)."""
    b = validate_bandwidth(samples.bandwidth)
    return So3Coefficients(b, _direct(samples.data, b, max_bandwidth, coeff_count(b), "so3_fsoft_direct"))


def ifsoft_direct(coeffs: So3Coefficients, max_bandwidth: int = DIRECT_BANDWIDTH_CAP) -> So3SampleGrid:
    """Reference inverse transform evaluated as the defining sum on the GPU (soft.py:236-256)."""
    b = validate_bandwidth(coeffs.bandwidth)
    return So3SampleGrid(b, _direct(coeffs.data, b, max_bandwidth, grid_size(b) ** 3, "so3_ifsoft_direct"))
