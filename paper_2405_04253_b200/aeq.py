"""FNT-AEQ: 4x4 real-valued MIMO radius-directed block equalizer on the B200
(drop-in for fntdsp/aeq.py).

The stream state (float taps w, 14-bit taps w_int, overlap history, saturation
and symbol counters) lives in device memory (fntgpu_aeq_state); `process` runs
the whole block recursion inside one kernel launch (k_aeq.cu: one warp per
stream, taps in registers across blocks). Host attributes (`w`, `taps`,
`history`, `saturations`, `symbols_processed`) read the device state on access,
and assigning them writes it back, so code written against the reference object
keeps working.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cdc import BudgetError
from .complexity import COUNTER
from .fixedpoint import QuantSpec, check_overflow, split_taps
from .fnt import TransformPlan, default_plans

#: output / input stream order of the 4x4 real MIMO: X and Y polarizations, I and Q
STREAMS = ("XI", "XQ", "YI", "YQ")
TAP_MAG_MAX = 2 ** 14 - 1  # largest 14-bit tap magnitude


def qam16_radii() -> np.ndarray:
    """The three ring radii of 16QAM scaled to unit mean energy (levels +-1, +-3:
    |s|^2 in {2, 10, 18} / 10) (aeq.py:29-31)."""
    return np.sqrt(np.array([2.0, 10.0, 18.0]) / 10.0)


@dataclass
class AeqConfig:
    block_n: int = 32
    l_taps: int = 16
    mu: float = 1e-3
    radii: np.ndarray = field(default_factory=qam16_radii)
    tap_bits: int = 14
    group_bits: int = 7
    sig_spec: QuantSpec = field(default_factory=lambda: QuantSpec(5, 8.0))
    tap_scale: float = float(1 << 13)

    def __post_init__(self) -> None:
        if self.l_taps != self.block_n // 2:
            raise ValueError("l_taps must equal block_n / 2")
        if self.mu < 0:
            raise ValueError("mu must be >= 0")
        self.radii = np.sort(np.asarray(self.radii, dtype=float))


def rde_error(y_i: np.ndarray, y_q: np.ndarray, radii: np.ndarray) -> np.ndarray:
    """Radius-directed error R^2 - |y|^2, R the ring nearest to |y| (the first one on a
    tie), shared by the I and Q outputs of a polarization (aeq.py:53-58). Host helper;
    the kernels decide the ring without the square root (aeq_common.cuh rde)."""
    power = np.asarray(y_i) ** 2 + np.asarray(y_q) ** 2
    dist = np.abs(np.sqrt(power)[..., None] - radii)
    return radii[dist.argmin(axis=-1)] ** 2 - power


@dataclass
class RvMimoTaps:
    """The 16 real FIR filters as 14-bit integers w_int[s_out, s_in, lag], with their
    7-bit sign-magnitude groups (aeq.py:61-81)."""

    w_int: np.ndarray
    high: np.ndarray = field(init=False)
    low: np.ndarray = field(init=False)

    def __post_init__(self) -> None:
        self.resplit()

    def resplit(self) -> None:
        groups = split_taps(self.w_int)
        self.high = groups.high
        self.low = groups.low

    @classmethod
    def center_spike(cls, l_taps: int, spike: int) -> "RvMimoTaps":
        """Identity MIMO: `spike` at the centre lag of the four direct filters."""
        w = np.zeros((4, 4, l_taps), dtype=np.int64)
        w[np.arange(4), np.arange(4), l_taps // 2] = spike
        return cls(w)


AEQ_KERNELS = {"auto": 0, "warp": 1, "pol": 2}  # FNTGPU_AEQ_KERNEL_*
_aeq_kernel = "auto"


def set_aeq_kernel(name: str) -> str:
    """Select the equalizer's stream layout for parameter blocks built afterwards
    (auto / warp: one warp per stream / pol: two warps per stream, one per
    polarization); returns the previous selection. Outputs are identical."""
    global _aeq_kernel
    if name not in AEQ_KERNELS:
        raise ValueError(f"unknown AEQ kernel {name!r}: one of {sorted(AEQ_KERNELS)}")
    prev, _aeq_kernel = _aeq_kernel, name
    return prev


def aeq_params(config: AeqConfig, forward: int | None = None) -> _lib.AeqParams:
    """The C-ABI parameter block for an AeqConfig."""
    prm = _lib.AeqParams()
    prm.sig_scale = float(config.sig_spec.scale)
    prm.tap_scale = float(config.tap_scale)
    prm.mu = float(config.mu)
    radii = np.asarray(config.radii, dtype=float)
    if not 1 <= radii.size <= 8:
        raise NotImplementedError("the GPU equalizer supports 1..8 ring radii")
    for i, r in enumerate(radii):
        prm.radii[i] = float(r)
    prm.n_radii = int(radii.size)
    prm.forward = _lib.env_forward_mode() if forward is None else int(forward)
    prm.kernel = AEQ_KERNELS[_aeq_kernel]
    return prm


def aeq_selfcheck(config: AeqConfig, lo: int = -(1 << 31), hi: int = 1 << 31) -> tuple[int, int]:
    """Device self-check of the equalizer's division and ring-decision shortcuts for
    this config (fntgpu_aeq_selfcheck): (division mismatches over every int32 y_int
    in [lo, hi), ring-decision mismatches). Both must be 0."""
    t = _lib.torch()
    out = t.zeros(2, dtype=t.int64, device=_lib.device())
    prm = aeq_params(config)
    _lib.check(_lib.load().fntgpu_aeq_selfcheck(C.byref(prm), int(lo), int(hi), _lib.ptr(out),
                                                 _lib.stream_handle()), "aeq_selfcheck")
    d, r = out.cpu().tolist()
    return int(d), int(r)


def mu_block_array(n_blocks: int, hop: int, mu_schedule, default_mu: float) -> np.ndarray:
    """mu of each block: mu_schedule(b * hop), or config.mu (aeq.py:187-188)."""
    if mu_schedule is None:
        return np.full(n_blocks, default_mu, dtype=np.float64)
    fast = getattr(mu_schedule, "block_mu", None)  # linksim.GearSchedule: vectorized
    if fast is not None:
        table = fast(n_blocks, hop)
        if table is not None:
            return table
    out = np.empty(n_blocks, dtype=np.float64)
    for b in range(n_blocks):
        m = mu_schedule(b * hop)
        out[b] = default_mu if m is None else float(m)
    return out


class FntAeq:
    """Block equalizer state: taps, overlap history, error trace (aeq.py:84-190)."""

    def __init__(self, config: AeqConfig, plan: TransformPlan | None = None,
                 forward: int | None = None):
        self.config = config
        self.plan = plan if plan is not None else default_plans()["aeq32"]
        if self.plan.n != config.block_n:
            raise ValueError("plan length does not match block_n")
        self.budget = check_overflow(np.full(config.l_taps, (1 << config.group_bits) - 1),
                                     config.sig_spec, self.plan.params)
        if not self.budget.passed:
            raise BudgetError(str(self.budget))
        p = self.plan
        if not (p.params.t == 4 and p.n == 32 and p.alpha == 2):
            raise NotImplementedError(
                "the GPU FNT-AEQ implements the aeq32 plan (F4, alpha=2, N=32) only")
        self.err_trace: list[float] = []
        self._tap_spectra = None
        self._prm = aeq_params(config, forward)
        with _lib.api_stream():
            self._state = _lib.zeros((_lib.AEQ_STATE_BYTES,), np.uint8)
            lib = _lib.load()
            _lib.check(lib.fntgpu_aeq_init(_lib.ptr(self._state), 1, C.byref(self._prm),
                                           _lib.stream_handle()), "aeq_init")
            # complete before the engine is used from any thread's stream
            _lib.torch().cuda.current_stream().synchronize()

    # -- device state views -----------------------------------------------------

    @_lib.on_api_stream
    def _read(self) -> _lib.AeqState:
        raw = _lib.to_host(self._state)
        return _lib.AeqState.from_buffer_copy(raw.tobytes())

    @_lib.on_api_stream
    def _write(self, st: _lib.AeqState) -> None:
        raw = np.frombuffer(bytes(st), dtype=np.uint8).copy()
        self._state.copy_(_lib.torch().from_numpy(raw).to(self._state.device))
        _lib.torch().cuda.current_stream().synchronize()

    @property
    def w(self) -> np.ndarray:
        return np.array(self._read().w, dtype=np.float64).reshape(4, 4, 16)

    @w.setter
    def w(self, value) -> None:
        st = self._read()
        v = np.ascontiguousarray(np.asarray(value, dtype=np.float64).reshape(256))
        C.memmove(st.w, v.ctypes.data, v.nbytes)
        self._write(st)

    @property
    def taps(self) -> RvMimoTaps:
        return RvMimoTaps(np.array(self._read().w_int, dtype=np.int64).reshape(4, 4, 16))

    @taps.setter
    def taps(self, value: RvMimoTaps) -> None:
        st = self._read()
        v = np.ascontiguousarray(np.asarray(value.w_int, dtype=np.int32).reshape(256))
        C.memmove(st.w_int, v.ctypes.data, v.nbytes)
        self._write(st)

    @property
    def history(self) -> np.ndarray:
        return np.array(self._read().hist, dtype=np.int64).reshape(4, 16)

    @history.setter
    def history(self, value) -> None:
        st = self._read()
        v = np.ascontiguousarray(np.asarray(value, dtype=np.int32).reshape(64))
        C.memmove(st.hist, v.ctypes.data, v.nbytes)
        self._write(st)

    @property
    def saturations(self) -> int:
        return int(self._read().saturations)

    @property
    def symbols_processed(self) -> int:
        return int(self._read().symbols)

    # -- forward / update -------------------------------------------------------

    @_lib.on_api_stream
    def _launch(self, x: np.ndarray, n_blocks: int, adapt: bool, mu_blocks: np.ndarray | None):
        hop = self.config.l_taps
        n = n_blocks * hop
        lo, hi = (int(x.min()), int(x.max())) if x.size else (0, 0)
        if max(-lo, hi) > self.plan.params.half:
            raise ValueError("input exceeds the encodable signed range")
        if -128 <= lo and hi <= 127:
            dt, align = np.int8, 16
        else:
            dt, align = np.int32, 4
        ld = -(-n // align) * align
        host = np.zeros((4, ld), dtype=dt)
        host[:, :n] = x[:, :n]
        dx = _lib.to_device(host)
        dy = _lib.empty((4, n), np.float64)
        derr = _lib.empty((max(n_blocks, 1),), np.float64) if adapt else None
        dmu = _lib.to_device(mu_blocks) if (adapt and mu_blocks is not None) else None
        io = _lib.AeqIO()
        io.n_streams = 1
        io.in_mode = _lib.AEQ_IN_PLANAR
        io.in_dtype = _lib.dtype_code(dt)
        io.adapt = int(adapt)
        io.x = dx.data_ptr()
        io.x_stream_stride = 4 * ld
        io.x_row_stride = ld
        io.n_blocks = n_blocks
        io.mu_blocks = dmu.data_ptr() if dmu is not None else None
        io.y = dy.data_ptr()
        io.y_stream_stride = 4 * n
        io.y_row_stride = n
        io.err = derr.data_ptr() if derr is not None else None
        io.err_stream_stride = max(n_blocks, 1)
        lib = _lib.load()
        _lib.check(lib.fntgpu_aeq_process(_lib.ptr(self._state), C.byref(self._prm), C.byref(io),
                                          _lib.stream_handle()), "aeq_process")
        y = _lib.to_host(dy)
        if adapt:
            self.err_trace.extend(_lib.to_host(derr)[:n_blocks].tolist())
        return y

    def equalize_block(self, x_new: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """4 x hop new samples -> (y float (4, hop), x_block (4, 2 hop)) (aeq.py:118-144)."""
        hop = self.config.l_taps
        x_new = np.asarray(x_new, dtype=np.int64)
        if x_new.shape != (4, hop):
            raise ValueError(f"expected (4, {hop}) block, got {x_new.shape}")
        x_block = np.concatenate([self.history, x_new], axis=1)
        if np.abs(x_block).max() > self.plan.params.half:
            raise ValueError("input exceeds the encodable signed range")
        with COUNTER.scope("aeq-fnt"):
            COUNTER.add(2 * 16 * self.plan.n)  # prod.size (aeq.py:137-138)
        y = self._launch(x_new, 1, False, None)
        return y, x_block

    @_lib.on_api_stream
    def update_taps(self, x_block: np.ndarray, y: np.ndarray, mu: float | None = None) -> None:
        """Block-accumulated RDE update, requantize, resplit (aeq.py:148-170)."""
        cfg = self.config
        mu = cfg.mu if mu is None else mu
        xb = np.ascontiguousarray(np.asarray(x_block, dtype=np.int64).reshape(4, 32))
        yy = np.ascontiguousarray(np.asarray(y, dtype=np.float64).reshape(4, 16))
        dxb = _lib.to_device(xb)
        dy = _lib.to_device(yy)
        derr = _lib.empty((1,), np.float64)
        lib = _lib.load()
        _lib.check(lib.fntgpu_aeq_update_taps(_lib.ptr(self._state), C.byref(self._prm),
                                              _lib.ptr(dxb), _lib.ptr(dy), float(mu),
                                              _lib.ptr(derr), _lib.stream_handle()),
                   "aeq_update_taps")
        self.err_trace.append(float(_lib.to_host(derr)[0]))
        self._tap_spectra = None

    def process(self, x: np.ndarray, adapt: bool = True, mu_schedule=None) -> np.ndarray:
        """Stream 4 x n samples through the equalize/update loop (aeq.py:172-190)."""
        hop = self.config.l_taps
        x = np.asarray(x, dtype=np.int64)
        n_blocks = x.shape[1] // hop
        if n_blocks == 0:
            return np.zeros((4, 0))
        if x.shape[0] != 4:
            raise ValueError(f"expected (4, {hop}) block, got {(x.shape[0], hop)}")
        with COUNTER.scope("aeq-fnt"):
            COUNTER.add(2 * 16 * self.plan.n * n_blocks)
        mu_blocks = mu_block_array(n_blocks, hop, mu_schedule, self.config.mu) if adapt else None
        return self._launch(x, n_blocks, adapt, mu_blocks)


@_lib.on_api_stream
def td_aeq_float(x: np.ndarray, config: AeqConfig, mu_schedule=None,
                 w0: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Per-symbol float 4x4 RDE baseline (aeq.py:193-249): returns (outputs, final taps).

    Not on the FNT path (the paper's float comparator). Runs on the GPU
    (k_td_aeq, one warp per stream, every product and sum rounded separately in
    the reference's order), so the results equal the reference's numba kernel bit
    for bit. 16 taps per filter (the reference's AeqConfig default)."""
    t = _lib.torch()
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.ndim != 2 or x.shape[0] != 4:
        raise ValueError("x must have shape (4, n)")
    n = x.shape[1]
    L = config.l_taps
    if L != 16:
        raise NotImplementedError("the GPU float comparator runs 16-tap filters")
    if w0 is None:
        w = np.zeros((4, 4, L))
        for s in range(4):
            w[s, s, L // 2] = 1.0
    else:
        w = np.ascontiguousarray(np.asarray(w0, dtype=np.float64)).copy()
    mu_arr = None
    if mu_schedule is None:
        mu_arr = np.full(n, config.mu)
    elif getattr(mu_schedule, "block_mu", None) is not None:
        mu_arr = mu_schedule.block_mu(n, 1)  # per symbol index
    if mu_arr is None:
        mu_arr = np.array([mu_schedule(i) for i in range(n)], dtype=np.float64)
    radii = np.asarray(config.radii, dtype=float)
    if not 1 <= radii.size <= 8:
        raise NotImplementedError("the GPU equalizer supports 1..8 ring radii")
    dev = _lib.device()
    dx = t.from_numpy(x).to(dev)
    dw = t.from_numpy(w).to(dev)
    dmu = t.from_numpy(np.ascontiguousarray(mu_arr)).to(dev)
    dy = t.empty((4, n), dtype=t.float64, device=dev)
    io = _lib.TdAeqIO()
    io.n_streams, io.n_radii, io.n = 1, int(radii.size), n
    io.x, io.x_stream_stride, io.x_row_stride = dx.data_ptr(), 4 * n, n
    io.w, io.mu = dw.data_ptr(), dmu.data_ptr()
    for i, r in enumerate(radii):
        io.radii[i] = float(r)
    io.y, io.y_stream_stride, io.y_row_stride = dy.data_ptr(), 4 * n, n
    with COUNTER.scope("aeq-td"):
        _lib.check(_lib.load().fntgpu_td_aeq(C.byref(io), _lib.stream_handle()), "td_aeq")
        COUNTER.add(16 * L * n)
    return dy.cpu().numpy(), dw.cpu().numpy()
