"""Fermat number transforms and fast cyclic convolution on the B200
(drop-in for fntdsp/fnt.py; same names, arguments, dtypes and errors).

Plans are validated on the host exactly like make_plan (fnt.py:60-83) and
mirrored on the device by libfntgpu (fntgpu_plan_create). fnt / ifnt /
cyclic_convolve_* run hand-written sm_100a kernels (k_transform.cu): the two
shipped shift-add plans (aeq32, cdc64) in registers with rotate-only twiddles,
any other valid plan in a shared-memory kernel. Inputs are numpy arrays in host
memory (the reference's contract); they are copied to the device, transformed,
and copied back as int64.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .complexity import COUNTER
from .fermat import FermatParams


class InvalidPlanError(ValueError):
    """Radix/modulus/length triple does not support a radix-2 transform."""


def _bitrev_table(n: int) -> np.ndarray:
    lg = n.bit_length() - 1
    idx = np.arange(n, dtype=np.int64)
    out = np.zeros(n, dtype=np.int64)
    for b in range(lg):
        out |= ((idx >> b) & 1) << (lg - 1 - b)
    return out


def _stage_tables(root: int, n: int, F: int) -> tuple:
    lg = n.bit_length() - 1
    return tuple(np.array([pow(root, j * (n >> (s + 1)), F) for j in range(1 << s)],
                          dtype=np.int64) for s in range(lg))


_PLAN_LOCK = threading.RLock()


class _DevicePlan:
    """Owner of the libfntgpu plan handle (device twiddle tables)."""

    def __init__(self, t: int, n: int, alpha: int):
        self.handle = C.c_void_p()
        self._lib = None
        lib = _lib.load()
        _lib.check(lib.fntgpu_plan_create(t, n, alpha, C.byref(self.handle)), "plan_create")
        self._lib = lib

    def __del__(self):
        if self._lib is not None and self.handle:
            try:
                self._lib.fntgpu_plan_destroy(self.handle)
            except Exception:  # interpreter shutdown
                pass


@dataclass(frozen=True)
class TransformPlan:
    """Validated (modulus, radix, length) triple with its schedule (fnt.py:24-33)."""

    params: FermatParams
    n: int
    alpha: int
    alpha_inv: int
    n_inv: int
    bitrev: np.ndarray = field(repr=False)
    fwd_twiddles: tuple = field(repr=False)
    inv_twiddles: tuple = field(repr=False)
    _dev: list = field(default_factory=list, repr=False, compare=False)

    def device_plan(self) -> _DevicePlan:
        """The GPU copy of this plan, created lazily on first use. The host
        twiddle tables are authoritative (callers may edit them, cli.py:84-86):
        if they no longer match what the device holds, they are re-uploaded."""
        with _PLAN_LOCK:  # plans are shared by every thread (fnt.py: immutable, reentrant)
            if not self._dev:
                # the device starts from the canonical tables of (t, n, alpha)
                F = self.params.F
                canon = (_stage_tables(self.alpha, self.n, F),
                         _stage_tables(self.alpha_inv, self.n, F))
                self._dev.append(_DevicePlan(self.params.t, self.n, self.alpha))
                self._dev.append(self._tables_digest(*canon))
            dig = self._tables_digest()
            if dig != self._dev[1]:
                fwd = np.ascontiguousarray(np.concatenate(self.fwd_twiddles), dtype=np.int64)
                inv = np.ascontiguousarray(np.concatenate(self.inv_twiddles), dtype=np.int64)
                lib = _lib.load()
                _lib.check(lib.fntgpu_plan_set_twiddles(
                    self._dev[0].handle, fwd.ctypes.data_as(C.c_void_p),
                    inv.ctypes.data_as(C.c_void_p)), "plan_set_twiddles")
                self._dev[1] = dig
            return self._dev[0]

    def _tables_digest(self, fwd=None, inv=None) -> bytes:
        fwd = self.fwd_twiddles if fwd is None else fwd
        inv = self.inv_twiddles if inv is None else inv
        return b"".join(np.asarray(t, np.int64).tobytes() for t in fwd) + b"|" + b"".join(
            np.asarray(t, np.int64).tobytes() for t in inv)


def make_plan(params: FermatParams, alpha: int, n: int) -> TransformPlan:
    """Validate that alpha has order exactly n mod F and precompute the tables."""
    F = params.F
    if n < 2 or n & (n - 1):
        raise InvalidPlanError(f"length must be a power of two >= 2, got {n}")
    if not 0 < alpha < F:
        raise InvalidPlanError(f"radix {alpha} is not a canonical nonzero residue")
    if pow(alpha, n, F) != 1:
        raise InvalidPlanError(f"radix {alpha} does not satisfy alpha^{n} = 1 (mod {F})")
    if pow(alpha, n // 2, F) != F - 1:
        raise InvalidPlanError(
            f"radix {alpha} has order < {n} mod {F} (alpha^{n // 2} != -1)")
    a_inv = pow(alpha, -1, F)
    return TransformPlan(params=params, n=n, alpha=alpha, alpha_inv=a_inv,
                         n_inv=pow(n, -1, F), bitrev=_bitrev_table(n),
                         fwd_twiddles=_stage_tables(alpha, n, F),
                         inv_twiddles=_stage_tables(a_inv, n, F))


def _as_i64(x) -> np.ndarray:
    return np.asarray(x, dtype=np.int64)


def _check_len(plan: TransformPlan, a: np.ndarray) -> None:
    if a.shape[-1] != plan.n:
        raise ValueError(f"expected length {plan.n}, got {a.shape[-1]}")


@_lib.on_api_stream
def _transform(plan: TransformPlan, x, inverse: bool) -> np.ndarray:
    a = _as_i64(x)
    _check_len(plan, a)
    if a.size == 0:
        return np.empty(a.shape, dtype=np.int64)
    dp = plan.device_plan()
    d = _lib.to_device(a)
    lib = _lib.load()
    _lib.check(lib.fntgpu_fnt(dp.handle, int(inverse), _lib.ptr(d), _lib.ptr(d), a.size // plan.n,
                              0, _lib.stream_handle()), "fnt")
    return _lib.to_host(d).reshape(a.shape)


def fnt(plan: TransformPlan, x: np.ndarray) -> np.ndarray:
    """Forward transform along the last axis (fnt.py:106-108, Eq. 1)."""
    return _transform(plan, x, False)


def ifnt(plan: TransformPlan, X: np.ndarray) -> np.ndarray:
    """Inverse transform including the N^-1 scale (fnt.py:111-114, Eq. 2)."""
    return _transform(plan, X, True)


def _broadcast_pair(plan, a, b):
    """Shapes for pointwise products of two (..., n) arrays (numpy broadcasting)."""
    shape = np.broadcast_shapes(a.shape, b.shape)
    return shape


@_lib.on_api_stream
def _conv_real(plan: TransformPlan, x: np.ndarray, h: np.ndarray, flags: int) -> np.ndarray:
    shape = _broadcast_pair(plan, x, h)
    size = int(np.prod(shape))
    if size == 0:
        return np.empty(shape, dtype=np.int64)
    batch = size // plan.n
    xb = np.broadcast_to(x, shape)
    if h.ndim == 1 or h.size == plan.n:
        hv, h_stride = h.reshape(plan.n), 0
    else:
        hv, h_stride = np.broadcast_to(h, shape), plan.n
    dx = _lib.to_device(np.ascontiguousarray(xb))
    dh = _lib.to_device(np.ascontiguousarray(hv))
    dz = _lib.empty(shape, np.int64)
    lib = _lib.load()
    _lib.check(lib.fntgpu_cyclic_convolve_real(plan.device_plan().handle, _lib.ptr(dx), _lib.ptr(dh),
                                               h_stride, _lib.ptr(dz), batch, flags,
                                               _lib.stream_handle()), "cyclic_convolve_real")
    return _lib.to_host(dz)


def cyclic_convolve_real(plan: TransformPlan, x: np.ndarray, h: np.ndarray) -> np.ndarray:
    """ifnt(fnt(x) * fnt(h)): one general product per bin (fnt.py:117-125)."""
    x = _as_i64(x)
    _check_len(plan, x)
    h = _as_i64(h)
    _check_len(plan, h)
    out = _conv_real(plan, x, h, 0)
    COUNTER.add(out.size)
    return out


@_lib.on_api_stream
def _conv_complex(plan, xr, xi, yr, yi, flags):
    shape = np.broadcast_shapes(xr.shape, xi.shape, yr.shape, yi.shape)
    size = int(np.prod(shape))
    if size == 0:
        e = np.empty(shape, dtype=np.int64)
        return e, e.copy()
    batch = size // plan.n
    xs = [np.ascontiguousarray(np.broadcast_to(a, shape)) for a in (xr, xi)]
    if yr.size == plan.n and yi.size == plan.n:
        ys, stride = [a.reshape(plan.n) for a in (yr, yi)], 0
    else:
        ys, stride = [np.ascontiguousarray(np.broadcast_to(a, shape)) for a in (yr, yi)], plan.n
    d = [_lib.to_device(a) for a in (*xs, *ys)]
    zr = _lib.empty(shape, np.int64)
    zi = _lib.empty(shape, np.int64)
    lib = _lib.load()
    _lib.check(lib.fntgpu_cyclic_convolve_complex(
        plan.device_plan().handle, *[_lib.ptr(t) for t in d], stride, _lib.ptr(zr), _lib.ptr(zi),
        batch, flags, _lib.stream_handle()), "cyclic_convolve_complex")
    return _lib.to_host(zr), _lib.to_host(zi)


def cyclic_convolve_complex(plan: TransformPlan, x_re: np.ndarray, x_im: np.ndarray,
                            y_re: np.ndarray, y_im: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Complex cyclic convolution, 2 general products per bin (fnt.py:128-161)."""
    q = plan.params.b
    if q < 2:
        raise ValueError(f"complex decomposition needs b >= 2, got b={q}")
    arrs = [_as_i64(a) for a in (x_re, x_im, y_re, y_im)]
    for a in arrs:
        _check_len(plan, a)
    zr, zi = _conv_complex(plan, *arrs, 0)
    COUNTER.add(2 * zr.size)
    return zr, zi


def _encode_check(v: np.ndarray, p: FermatParams) -> None:
    if v.size and np.abs(v).max() > p.half:
        raise ValueError("input exceeds the encodable signed range")


def convolve_signed_real(plan: TransformPlan, x: np.ndarray, h: np.ndarray) -> np.ndarray:
    """Exact integer cyclic convolution of signed sequences (fnt.py:164-170).
    Encoding and decoding are fused into the convolution kernel."""
    x = _as_i64(x)
    h = _as_i64(h)
    _encode_check(x, plan.params)
    _encode_check(h, plan.params)
    _check_len(plan, x)
    _check_len(plan, h)
    out = _conv_real(plan, x, h, _lib.DECODE_SIGNED)
    COUNTER.add(out.size)
    return out


def convolve_signed_complex(plan: TransformPlan, x_re: np.ndarray, x_im: np.ndarray,
                            y_re: np.ndarray, y_im: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Complex counterpart of convolve_signed_real (fnt.py:173-183)."""
    arrs = [_as_i64(a) for a in (x_re, x_im, y_re, y_im)]
    for a in arrs:
        _encode_check(a, plan.params)
    q = plan.params.b
    if q < 2:
        raise ValueError(f"complex decomposition needs b >= 2, got b={q}")
    for a in arrs:
        _check_len(plan, a)
    zr, zi = _conv_complex(plan, *arrs, _lib.DECODE_SIGNED)
    COUNTER.add(2 * zr.size)
    return zr, zi


@_lib.on_api_stream
def _residue_map(v: np.ndarray, p: FermatParams, signed_out: bool, decode_only: bool = False):
    if v.size == 0:
        return np.empty(v.shape, dtype=np.int64)
    d = _lib.to_device(v)
    lib = _lib.load()
    _lib.check(lib.fntgpu_residue_map(p.t, int(decode_only), _lib.ptr(d), _lib.ptr(d), v.size,
                                      _lib.stream_handle()), "residue_map")
    return _lib.to_host(d).reshape(v.shape)


_DEFAULT_PLANS: dict | None = None


def default_plans() -> dict[str, TransformPlan]:
    """The three shipped plans (fnt.py:186-195). A fresh dict each call, like the
    reference (callers may mutate the tables, e.g. selftest --fault-inject)."""
    from .fermat import sqrt2
    f17 = FermatParams(2)
    f65537 = FermatParams(4)
    return {
        "mod17": make_plan(f17, 2, 8),
        "aeq32": make_plan(f65537, 2, 32),
        "cdc64": make_plan(f65537, sqrt2(f65537), 64),
    }
