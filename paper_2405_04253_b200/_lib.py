"""ctypes binding of libfntgpu.so (C ABI in include/fntgpu.h).

The product path: every compute entry point of the shim goes through here to
hand-written sm_100a kernels. There is no CPU fallback -- if the library or a GPU
is missing, calls raise.

PyTorch is used only as plumbing: device allocation, host<->device copies and
the current CUDA stream handle.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import functools
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("FNTGPU_LIB", str(_PKG / "libfntgpu.so")))  # override: A/B builds

ABI_VERSION = 1

OK, EINVAL, ECUDA, EUNSUPPORTED = 0, -1, -2, -3
EPLAN_LENGTH, EPLAN_RADIX, EPLAN_ORDER, EPLAN_SUBORD, EPLAN_MODULUS = -10, -11, -12, -13, -14

NONE, I8, I16, I32, I64, F64, C128 = 0, 1, 2, 3, 4, 5, 6
DECODE_SIGNED = 1
AEQ_FWD_FNT, AEQ_FWD_DIRECT = 0, 1
AEQ_IN_PLANAR, AEQ_IN_DECIM = 0, 1

vp = C.c_void_p


class CdcTaps(C.Structure):
    _fields_ = [("b_plus", C.c_uint32 * 64), ("b_minus", C.c_uint32 * 64),
                ("n_taps", C.c_int32), ("kernel", C.c_int32)]


class CdcIO(C.Structure):
    _fields_ = [("n_streams", C.c_int32), ("in_dtype", C.c_int32),
                ("xr", vp), ("xi", vp), ("x_stride", C.c_int64),
                ("x_first", C.c_int64), ("x_count", C.c_int64), ("length", C.c_int64),
                ("out_first", C.c_int64), ("out_count", C.c_int64),
                ("out_dtype", C.c_int32), ("pad0", C.c_int32),
                ("yr", vp), ("yi", vp), ("y_stride", C.c_int64), ("inv_scale", C.c_double),
                ("qr", vp), ("qi", vp), ("q_stride", C.c_int64), ("q_scale", C.c_double),
                ("q_max", C.c_int32), ("pad1", C.c_int32), ("decim_acc", vp),
                ("q_shift", C.c_int32), ("pad2", C.c_int32), ("q_tie", C.c_int8 * 128),
                ("in_scale", C.c_double), ("in_max", C.c_int32), ("pad3", C.c_int32),
                ("in_clipped", vp)]


class DecimIO(C.Structure):
    _fields_ = [("n_links", C.c_int32), ("sps", C.c_int32), ("acc", vp), ("length", C.c_int64),
                ("phase", vp), ("gap", vp)]


class AeqParams(C.Structure):
    _fields_ = [("sig_scale", C.c_double), ("tap_scale", C.c_double), ("mu", C.c_double),
                ("radii", C.c_double * 8), ("n_radii", C.c_int32), ("forward", C.c_int32),
                ("kernel", C.c_int32), ("reserved", C.c_int32)]


class AeqState(C.Structure):
    _fields_ = [("w", C.c_double * 256), ("w_int", C.c_int32 * 256), ("hist", C.c_int32 * 64),
                ("saturations", C.c_int64), ("symbols", C.c_int64), ("n_err", C.c_int64),
                ("reserved", C.c_int64)]


class AeqIO(C.Structure):
    _fields_ = [("n_streams", C.c_int32), ("in_mode", C.c_int32), ("in_dtype", C.c_int32),
                ("adapt", C.c_int32), ("x", vp), ("x_stream_stride", C.c_int64),
                ("x_row_stride", C.c_int64), ("qr", vp), ("qi", vp), ("q_stride", C.c_int64),
                ("phase", vp), ("n_blocks", C.c_int64), ("mu_blocks", vp), ("y", vp),
                ("y_stream_stride", C.c_int64), ("y_row_stride", C.c_int64), ("err", vp),
                ("err_stream_stride", C.c_int64)]


class TdAeqIO(C.Structure):
    _fields_ = [("n_streams", C.c_int32), ("n_radii", C.c_int32), ("n", C.c_int64), ("x", vp),
                ("x_stream_stride", C.c_int64), ("x_row_stride", C.c_int64), ("w", vp), ("mu", vp),
                ("radii", C.c_double * 8), ("y", vp), ("y_stream_stride", C.c_int64),
                ("y_row_stride", C.c_int64)]


AEQ_STATE_BYTES = C.sizeof(AeqState)

# (symbol, restype, argtypes) for every function declared in include/fntgpu.h
SIGNATURES = {
    "fntgpu_abi_version": (C.c_int, []),
    "fntgpu_last_error": (C.c_char_p, []),
    "fntgpu_device_count": (C.c_int, []),
    "fntgpu_plan_create": (C.c_int, [C.c_int, C.c_int, C.c_int64, C.POINTER(vp)]),
    "fntgpu_plan_destroy": (C.c_int, [vp]),
    "fntgpu_plan_set_twiddles": (C.c_int, [vp, vp, vp]),
    "fntgpu_plan_info": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int)]),
    "fntgpu_fnt": (C.c_int, [vp, C.c_int, vp, vp, C.c_int64, C.c_int, vp]),
    "fntgpu_cyclic_convolve_real": (C.c_int, [vp, vp, vp, C.c_int64, vp, C.c_int64, C.c_int, vp]),
    "fntgpu_cyclic_convolve_complex": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, vp, vp,
                                                 C.c_int64, C.c_int, vp]),
    "fntgpu_residue_map": (C.c_int, [C.c_int, C.c_int, vp, vp, C.c_int64, vp]),
    "fntgpu_struct_sizes": (C.c_int, [C.POINTER(C.c_int64), C.c_int]),
    "fntgpu_quantize_real": (C.c_int, [vp, C.c_int64, C.c_double, C.c_int32, C.c_int, vp, vp, vp]),
    "fntgpu_cdc64_process": (C.c_int, [C.POINTER(CdcTaps), C.POINTER(CdcIO), vp]),
    "fntgpu_decim_phase": (C.c_int, [C.POINTER(DecimIO), vp]),
    "fntgpu_aeq_init": (C.c_int, [vp, C.c_int, C.POINTER(AeqParams), vp]),
    "fntgpu_aeq_process": (C.c_int, [vp, C.POINTER(AeqParams), C.POINTER(AeqIO), vp]),
    "fntgpu_aeq_update_taps": (C.c_int, [vp, C.POINTER(AeqParams), vp, vp, C.c_double, vp, vp]),
    "fntgpu_td_aeq": (C.c_int, [C.POINTER(TdAeqIO), vp]),
    "fntgpu_copy2d_async": (C.c_int, [vp, C.c_int64, vp, C.c_int64, C.c_int64, C.c_int64, vp]),
    "fntgpu_aeq_selfcheck": (C.c_int, [C.POINTER(AeqParams), C.c_int64, C.c_int64, vp, vp]),
}

_LIB = None


class FntGpuError(RuntimeError):
    """A CUDA / library failure inside libfntgpu.so."""


def load(build_if_missing: bool = True):
    """Load libfntgpu.so (building it in-tree with nvcc if it is absent)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        if not build_if_missing:
            raise FntGpuError(f"{LIB_PATH} is missing; run paper_2405_04253_b200._build")
        from . import _build
        _build.build()
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fntgpu_abi_version() != ABI_VERSION:
        raise FntGpuError("libfntgpu.so ABI version mismatch; rebuild the extension")
    _LIB = lib
    return lib


def last_error() -> str:
    msg = load().fntgpu_last_error()
    return msg.decode() if msg else ""


def check(rc: int, where: str = "") -> None:
    if rc == OK:
        return
    msg = last_error()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise FntGpuError(f"{where}: {msg}" if where else msg)


# ---------------------------------------------------------------------------
# device plumbing (torch)

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise FntGpuError("no CUDA device: the FNT kernels have no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def stream_handle():
    return vp(torch().cuda.current_stream().cuda_stream)


_tls = threading.local()


@contextlib.contextmanager
def api_stream():
    """Stream for one drop-in API call (fnt / convolutions / quantize_real / the CDC and
    AEQ engines). A caller inside its own torch stream context keeps that stream; a
    caller on the default stream gets its host thread's own non-blocking stream, so
    calls from different threads -- one engine per thread, the reference's threading
    convention -- overlap on the GPU instead of serializing on
    the legacy default stream. Every drop-in call returns host arrays, i.e. it has
    synchronized its stream before returning, so device state left by one call is
    complete when any thread makes the next."""
    t = torch()
    if not t.cuda.is_available():  # the call itself reports the missing device
        yield
        return
    dev = device()
    if t.cuda.current_stream(dev) != t.cuda.default_stream(dev):
        yield
        return
    s = getattr(_tls, "streams", None)
    if s is None:
        s = _tls.streams = {}
    st = s.get(dev.index)
    if st is None:
        st = s[dev.index] = t.cuda.Stream(device=dev)
    with t.cuda.stream(st):
        yield


def on_api_stream(fn):
    """Decorator: run `fn` inside api_stream()."""
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        with api_stream():
            return fn(*args, **kwargs)
    return wrapper


def ptr(t) -> vp:
    return vp(t.data_ptr()) if t is not None else vp(0)


_NP2T = {}


# Device -> host copies of the drop-in calls' larger results go through two pinned
# staging chunks per host thread (DMA at the pinned rate, chunk k + 1's DMA
# overlapping chunk k's host memcpy): measured on the B200 box, 5-6.6 GB/s vs 2-2.8
# GB/s for pageable cudaMemcpy at 8-64 MB, whose driver staging also serialized the
# copies of concurrent threads (the drop-in chain moves ~40 MB per link). Host ->
# device copies stay pageable: there the driver's pipelined staging (13-17 GB/s)
# beats a single-threaded memcpy into pinned memory (11-12 GB/s).
_SMALL_COPY = 1 << 18
_STAGED_D2H = 4 << 20
_STAGED_H2D = False
_CHUNK = 4 << 20


class _Stage(threading.local):
    def __init__(self):
        self.bufs = [None, None]
        self.events = [None, None]


_stage = _Stage()


def _stage_buf(i: int, nbytes: int):
    b = _stage.bufs[i]
    if b is None or b.numel() < nbytes:
        size = min(_CHUNK, max(1 << 20, 1 << (nbytes - 1).bit_length()))
        b = torch().empty(size, dtype=torch().uint8, pin_memory=True)
        _stage.bufs[i] = b
    return b


_PINNED = None


def _pinned_ok() -> bool:
    """Page-locked staging is available (else the plain pageable copies are used)."""
    global _PINNED
    if _PINNED is None:
        try:
            _stage_buf(0, 1 << 20)
            _PINNED = True
        except RuntimeError:
            _PINNED = False
    return _PINNED


def _stage_ready(i: int) -> None:
    ev = _stage.events[i]
    if ev is not None:
        ev.synchronize()  # the previous copy through staging chunk i has completed
        _stage.events[i] = None


def to_device(a: np.ndarray):
    """Contiguous host array -> device tensor (same dtype)."""
    t = torch()
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:
        a = a.copy()
    if a.size == 0:
        return t.empty(a.shape, dtype=_torch_dtype(a.dtype), device=device())
    if a.nbytes <= _SMALL_COPY or not _STAGED_H2D or not _pinned_ok():
        return t.from_numpy(a).to(device(), non_blocking=False)
    d = t.empty(a.shape, dtype=_torch_dtype(a.dtype), device=device())
    src = a.reshape(-1).view(np.uint8)
    dst = d.view(-1).view(t.uint8)
    st = t.cuda.current_stream()
    for k, off in enumerate(range(0, a.nbytes, _CHUNK)):
        n = min(_CHUNK, a.nbytes - off)
        i = k & 1
        _stage_ready(i)
        b = _stage_buf(i, n)
        np.copyto(b.numpy()[:n], src[off:off + n])
        dst[off:off + n].copy_(b[:n], non_blocking=True)
        ev = t.cuda.Event()
        ev.record(st)
        _stage.events[i] = ev
    return d


def empty(shape, np_dtype):
    t = torch()
    return t.empty(tuple(shape), dtype=_torch_dtype(np.dtype(np_dtype)), device=device())


def zeros(shape, np_dtype):
    t = torch()
    return t.zeros(tuple(shape), dtype=_torch_dtype(np.dtype(np_dtype)), device=device())


def to_host(x) -> np.ndarray:
    """Device tensor -> a new numpy array (synchronous, like Tensor.cpu())."""
    t = torch()
    nbytes = x.numel() * x.element_size()
    if nbytes < _STAGED_D2H or not x.is_cuda or not _pinned_ok():
        return x.cpu().numpy()
    x = x.contiguous()
    out = np.empty(tuple(x.shape), dtype=_numpy_dtype(x.dtype))
    src = x.view(-1).view(t.uint8)
    dst = out.reshape(-1).view(np.uint8)
    st = t.cuda.current_stream()
    offs = list(range(0, nbytes, _CHUNK))

    def issue(k):
        off = offs[k]
        n = min(_CHUNK, nbytes - off)
        i = k & 1
        _stage_ready(i)
        b = _stage_buf(i, n)
        b[:n].copy_(src[off:off + n], non_blocking=True)
        ev = t.cuda.Event()
        ev.record(st)
        _stage.events[i] = ev

    issue(0)
    for k, off in enumerate(offs):
        if k + 1 < len(offs):
            issue(k + 1)  # the next chunk's DMA overlaps this chunk's memcpy
        i = k & 1
        n = min(_CHUNK, nbytes - off)
        _stage_ready(i)
        np.copyto(dst[off:off + n], _stage.bufs[i].numpy()[:n])
    return out


def _numpy_dtype(dt):
    t = torch()
    m = {t.int8: np.int8, t.int16: np.int16, t.int32: np.int32, t.int64: np.int64,
         t.float64: np.float64, t.complex128: np.complex128, t.uint8: np.uint8,
         t.float32: np.float32}
    return np.dtype(m[dt])


def _torch_dtype(dt: np.dtype):
    t = torch()
    m = {np.dtype(np.int8): t.int8, np.dtype(np.int16): t.int16, np.dtype(np.int32): t.int32,
         np.dtype(np.int64): t.int64, np.dtype(np.float64): t.float64,
         np.dtype(np.complex128): t.complex128, np.dtype(np.uint8): t.uint8,
         np.dtype(np.float32): t.float32}
    return m[np.dtype(dt)]


def dtype_code(dt) -> int:
    dt = np.dtype(dt)
    return {np.dtype(np.int8): I8, np.dtype(np.int16): I16, np.dtype(np.int32): I32,
            np.dtype(np.int64): I64, np.dtype(np.float64): F64,
            np.dtype(np.complex128): C128}[dt]


def env_forward_mode() -> int:
    """Default AEQ forward path: FNT (the paper's algorithm) unless overridden."""
    v = os.environ.get("FNTGPU_AEQ_FORWARD", "fnt").lower()
    return AEQ_FWD_DIRECT if v == "direct" else AEQ_FWD_FNT
