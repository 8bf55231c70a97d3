"""FNT-CDC: residue-domain overlap-save chromatic-dispersion compensation on the
B200 (drop-in for fntdsp/cdc.py).

`FntCdcEngine.process_int / process` run the fused sm_100a kernel k_cdc64 (one
thread per 64-sample overlap-save block: FNT-64 -> tap product -> IFNT-64 ->
discard overlap -> decode, one HBM round trip per sample). Tap design and tap
quantization are one-time host setup, as in the reference.
The float FD/TD baselines are not part of the FNT path; they are provided for
API completeness on the GPU through PyTorch's FFT (library code).
"""

from __future__ import annotations

import ctypes as C
import math
from pathlib import Path
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .complexity import COUNTER
from .fermat import FermatParams
from .fixedpoint import BudgetReport, QuantSpec, check_overflow, quantize
from .fnt import TransformPlan, convolve_signed_complex, default_plans, fnt

SPEED_OF_LIGHT = 299792458.0


class BudgetError(ValueError):
    """Configuration would overflow the convolution budget."""


@dataclass
class CdcConfig:
    z_km: float
    fs_hz: float
    dispersion_ps_nm_km: float = 17.0
    wavelength_nm: float = 1550.0
    n_taps: int = 32
    tap_bits: int = 6
    block_n: int = 64
    scheme: str = "fnt"  # fnt | fd-float | td-float

    def __post_init__(self) -> None:
        if self.n_taps > self.block_n // 2 + 1:
            raise ValueError(
                f"n_taps={self.n_taps} exceeds overlap-save validity "
                f"{self.block_n // 2 + 1} for block_n={self.block_n}")

    @property
    def accumulated_dispersion(self) -> float:
        """beta = D lambda^2 L / c in s^2, with D in s/m^2, lambda and L in m
        (cdc.py:47-52; the float64 products in the reference's order)."""
        wl_m = self.wavelength_nm * 1e-9
        return self.dispersion_ps_nm_km * 1e-6 * wl_m * wl_m * (self.z_km * 1e3) / SPEED_OF_LIGHT


def required_taps(cfg: CdcConfig) -> int:
    """Odd tap count spanning the dispersive spread, 2 floor(beta fs^2 / 2) + 1
    (cdc.py:55-58)."""
    return 1 + 2 * int(cfg.accumulated_dispersion * cfg.fs_hz ** 2 / 2)


def design_cd_taps(cfg: CdcConfig) -> np.ndarray:
    """Unit-energy inverse all-pass chirp exp(-j pi t^2 / beta) sampled at t = (n - c) / fs,
    c = n_taps // 2 (cdc.py:61-77); a unit impulse at c for z = 0."""
    c = cfg.n_taps // 2
    if cfg.z_km == 0:
        return np.eye(1, cfg.n_taps, c, dtype=complex)[0]
    beta = cfg.accumulated_dispersion
    t = (np.arange(cfg.n_taps) - c) / cfg.fs_hz
    chirp = np.exp(-1j * math.pi * t * t / beta)
    return chirp / np.linalg.norm(chirp)


def quantize_taps(taps: np.ndarray, bits: int) -> tuple[np.ndarray, np.ndarray, float]:
    """6-bit (say) taps on the largest power-of-two scale that keeps the biggest
    component within 2^(bits-1) - 1 (cdc.py:80-86): (re, im, scale)."""
    top = 2 ** (bits - 1) - 1
    peak = max(np.abs(taps.real).max(), np.abs(taps.imag).max())
    scale = 2.0 ** math.floor(math.log2(top / peak))
    q = quantize(taps, QuantSpec(bits, scale))
    return q.re, q.im, scale


def overlap_save_block_count(length: int, block_n: int = 64) -> int:
    """n_blocks of _overlap_save_blocks (cdc.py:89-95)."""
    hop = block_n // 2
    return -(-(length + hop) // hop)


def _int_input(x) -> np.ndarray:
    """The reference feeds samples through np.asarray(..., dtype=int64) (encode)."""
    a = np.asarray(x)
    if a.dtype.kind in "iu":
        return a
    return a.astype(np.int64)


def _device_dtype(a: np.ndarray, half: int) -> np.dtype:
    """Narrowest kernel input dtype holding a; raises like encode_signed_array."""
    if a.size == 0 or a.dtype == np.int8:
        return np.dtype(np.int8)
    if a.dtype in (np.int16, np.uint8, np.uint16) and half >= 32767:
        return np.dtype(np.int32)  # always encodable: no host scan needed
    lo, hi = int(a.min()), int(a.max())
    if max(-lo, hi) > half:
        raise ValueError("input exceeds the encodable signed range")
    if -128 <= lo and hi <= 127:
        return np.dtype(np.int8)
    return np.dtype(np.int32)


# Kernel behind fntgpu_cdc64_process for int8 planes (fntgpu_cdc_taps.kernel): "auto"
# (the measured-faster one: the tcgen05 split-integer matrix form for int16 /
# requantized / statistics outputs, the shift-add butterflies otherwise), "shift",
# "tc" (mma.sync matrix form) or "umma" (tcgen05 matrix form). All bit-exact; other
# input dtypes always take the shift-add kernel.
CDC_KERNELS = {"auto": 0, "shift": 1, "tc": 2, "umma": 3}
_cdc_kernel = os.environ.get("FNTGPU_CDC_KERNEL", "auto")
if _cdc_kernel not in CDC_KERNELS:
    raise ValueError(f"FNTGPU_CDC_KERNEL must be one of {sorted(CDC_KERNELS)}")


def set_cdc_kernel(name: str) -> str:
    """Select the CDC kernel for tap descriptors built afterwards; returns the previous."""
    global _cdc_kernel
    if name not in CDC_KERNELS:
        raise ValueError(f"unknown CDC kernel {name!r}: one of {sorted(CDC_KERNELS)}")
    prev, _cdc_kernel = _cdc_kernel, name
    return prev


@dataclass
class FntCdcEngine:
    """Residue-domain overlap-save dispersion equalizer for one polarization
    (cdc.py:98-180)."""

    config: CdcConfig
    sig_spec: QuantSpec
    plan: TransformPlan = None
    taps: np.ndarray = field(default=None, repr=False)

    def __post_init__(self) -> None:
        if self.plan is None:
            self.plan = default_plans()["cdc64"]
        if self.plan.n != self.config.block_n:
            raise ValueError("plan length does not match block_n")
        if self.taps is None:
            self.taps = design_cd_taps(self.config)
        self.tap_re, self.tap_im, self.tap_scale = quantize_taps(self.taps, self.config.tap_bits)
        self.budget = check_overflow(np.maximum(np.abs(self.tap_re), np.abs(self.tap_im)),
                                     self.sig_spec, self.plan.params, complex_mode=True)
        if not self.budget.passed:
            raise BudgetError(str(self.budget))
        self.support_warning = self.config.n_taps < required_taps(self.config)
        self._cache_tap_spectra()

    def _padded_taps(self) -> tuple[np.ndarray, np.ndarray]:
        hr = np.zeros(self.plan.n, dtype=np.int64)
        hi = np.zeros(self.plan.n, dtype=np.int64)
        hr[:self.config.n_taps] = self.tap_re
        hi[:self.config.n_taps] = self.tap_im
        return hr, hi

    def _cache_tap_spectra(self) -> None:
        """b+- = (H_r +- 2^8 H_i) mod F from two GPU transforms (cdc.py:124-135)."""
        p = self.plan.params
        F = p.F
        j = 1 << (p.b // 2)
        hr, hi = self._padded_taps()
        H = fnt(self.plan, np.stack([hr % F, hi % F]))
        self._b_plus = (H[0] + j * H[1]) % F
        self._b_minus = (H[0] - j * H[1]) % F
        self._taps_c = None

    def _fast(self) -> bool:
        p = self.plan
        return p.params.t == 4 and p.n == 64 and p.alpha == 4080

    def c_taps(self) -> _lib.CdcTaps:
        """The C-ABI tap descriptor (b+-, n_taps) for fntgpu_cdc64_process."""
        if self._taps_c is None:
            t = _lib.CdcTaps()
            for k in range(64):
                t.b_plus[k] = int(self._b_plus[k])
                t.b_minus[k] = int(self._b_minus[k])
            t.n_taps = int(self.config.n_taps)
            self._taps_c = t
        self._taps_c.kernel = CDC_KERNELS[_cdc_kernel]
        return self._taps_c

    @property
    def output_scale(self) -> float:
        return self.sig_spec.scale * self.tap_scale

    # -- block API ------------------------------------------------------------

    def process_block(self, xr: np.ndarray, xi: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """One 64-sample block in, the 32 newest outputs out (cdc.py:158-163)."""
        hop = self.plan.n // 2
        hr, hi = self._padded_taps()
        zr, zi = convolve_signed_complex(self.plan, np.asarray(xr), np.asarray(xi), hr, hi)
        return zr[hop:], zi[hop:]

    # -- stream API -----------------------------------------------------------

    @_lib.on_api_stream
    def _run(self, xr, xi, out_dtype: int):
        xr = _int_input(xr)
        xi = _int_input(xi)
        if xr.ndim != 1 or xi.ndim != 1:
            raise ValueError("process_int expects one-dimensional sample streams")
        if xr.shape != xi.shape:
            raise ValueError(f"operands could not be broadcast together with shapes "
                             f"{xr.shape} {xi.shape}")
        L = xr.size
        half = self.plan.params.half
        dt = max(_device_dtype(xr, half), _device_dtype(xi, half), key=lambda d: d.itemsize)
        hop = self.plan.n // 2
        n_blocks = overlap_save_block_count(L, self.plan.n)
        with COUNTER.scope("cdc-fnt"):
            COUNTER.add(2 * self.plan.n * n_blocks)  # u+.size + u-.size (cdc.py:151)
        if L == 0:
            return None, L
        if not self._fast():
            return self._run_generic(xr, xi, out_dtype), L
        dxr = _lib.to_device(xr.astype(dt, copy=False))
        dxi = _lib.to_device(xi.astype(dt, copy=False))
        io = _lib.CdcIO()
        io.n_streams = 1
        io.in_dtype = _lib.dtype_code(dt)
        io.xr, io.xi = dxr.data_ptr(), dxi.data_ptr()
        io.x_stride = L
        io.x_first, io.x_count, io.length = 0, L, L
        io.out_first, io.out_count = 0, L
        io.out_dtype = out_dtype
        if out_dtype == _lib.C128:
            y = _lib.empty((L,), np.complex128)
            io.yr = y.data_ptr()
            io.inv_scale = 1.0 / self.output_scale
            outs = (y,)
        else:
            yr = _lib.empty((L,), np.int64)
            yi = _lib.empty((L,), np.int64)
            io.yr, io.yi = yr.data_ptr(), yi.data_ptr()
            outs = (yr, yi)
        io.y_stride = L
        lib = _lib.load()
        _lib.check(lib.fntgpu_cdc64_process(C.byref(self.c_taps()), C.byref(io),
                                            _lib.stream_handle()), "cdc64_process")
        del hop
        return tuple(_lib.to_host(o) for o in outs), L

    def _run_generic(self, xr, xi, out_dtype):
        """Plans other than cdc64: overlap-save blocks through the GPU complex
        convolution kernel (table-driven transform), then the same slicing."""
        n = self.plan.n
        hop = n // 2
        n_blocks = overlap_save_block_count(xr.size, n)
        pad = np.zeros((2, hop + n_blocks * hop + hop), dtype=np.int64)
        pad[0, hop:hop + xr.size] = xr
        pad[1, hop:hop + xi.size] = xi
        idx = np.arange(n_blocks)[:, None] * hop + np.arange(n)[None, :]
        hr, hi = self._padded_taps()
        zr, zi = convolve_signed_complex(self.plan, pad[0][idx], pad[1][idx], hr, hi)
        c = self.config.n_taps // 2
        yr = zr[:, hop:].reshape(-1)[c:c + xr.size]
        yi = zi[:, hop:].reshape(-1)[c:c + xr.size]
        if out_dtype == _lib.C128:
            return ((yr + 1j * yi) / self.output_scale,)
        return (yr, yi)

    def process_int(self, xr: np.ndarray, xi: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """Full stream, integer output aligned with the input (cdc.py:165-175)."""
        outs, L = self._run(xr, xi, _lib.I64)
        if outs is None:
            return np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.int64)
        return outs[0], outs[1]

    def process(self, xr: np.ndarray, xi: np.ndarray) -> np.ndarray:
        """Full stream rescaled to complex float: y * (1/output_scale) (cdc.py:177-180)."""
        outs, L = self._run(xr, xi, _lib.C128)
        if outs is None:
            return np.zeros(0, dtype=np.complex128)
        return outs[0]


@_lib.on_api_stream
def fd_cdc_float(x: np.ndarray, cfg: CdcConfig, taps: np.ndarray | None = None) -> np.ndarray:
    """Float FFT overlap-save baseline (cdc.py:183-198), on the GPU via torch.fft.
    Not part of the FNT hot path (comparator only)."""
    t = _lib.torch()
    if taps is None:
        taps = design_cd_taps(cfg)
    n = cfg.block_n
    hop = n // 2
    x = np.asarray(x, dtype=complex)
    nb = overlap_save_block_count(x.size, n)
    pad = np.zeros(hop + nb * hop + hop, dtype=complex)
    pad[hop:hop + x.size] = x
    idx = np.arange(nb)[:, None] * hop + np.arange(n)[None, :]
    H = t.fft.fft(t.from_numpy(np.concatenate([taps, np.zeros(n - len(taps))])).to(_lib.device()))
    with COUNTER.scope("cdc-fd"):
        Y = t.fft.fft(t.from_numpy(pad[idx]).to(_lib.device()), dim=-1) * H
        y = t.fft.ifft(Y, dim=-1)[:, hop:].reshape(-1).cpu().numpy()
        COUNTER.add(nb * (2 * 2 * n * int(math.log2(n)) + 4 * n))
    c = cfg.n_taps // 2
    return y[c:c + x.size]


def td_cdc_float(x: np.ndarray, cfg: CdcConfig, taps: np.ndarray | None = None) -> np.ndarray:
    """Direct float FIR baseline (cdc.py:201-210), on the GPU via torch conv1d.
    Not part of the FNT hot path (comparator only)."""
    t = _lib.torch()
    if taps is None:
        taps = design_cd_taps(cfg)
    x = np.asarray(x, dtype=complex)
    L, K = x.size, len(taps)
    with COUNTER.scope("cdc-td"):
        dev = _lib.device()
        xs = t.from_numpy(np.stack([x.real, x.imag])).to(dev)[:, None, :]
        h = t.from_numpy(np.asarray(taps)[::-1].copy())
        hr = h.real.to(dev)[None, None, :]
        hi = h.imag.to(dev)[None, None, :]
        pad = t.nn.functional.pad
        xr = pad(xs[0:1], (K - 1, K - 1))
        xi = pad(xs[1:2], (K - 1, K - 1))
        conv = t.nn.functional.conv1d
        yr = (conv(xr, hr) - conv(xi, hi))[0, 0]
        yi = (conv(xr, hi) + conv(xi, hr))[0, 0]
        y = (yr + 1j * yi).cpu().numpy()
        COUNTER.add(4 * K * L)
    c = K // 2
    return y[c:c + L]


def save_taps(path, tap_re: np.ndarray, tap_im: np.ndarray, scale: float) -> None:
    """Integer taps as "re im" lines under a "# scale <repr>" header (cdc.py:213-217)."""
    lines = [f"# scale {scale!r}"] + [f"{int(a)} {int(b)}" for a, b in zip(tap_re, tap_im)]
    Path(path).write_text("".join(line + "\n" for line in lines))


def load_taps(path) -> tuple[np.ndarray, np.ndarray, float]:
    """Inverse of save_taps (cdc.py:220-233): (re, im, scale), scale 1.0 without a header."""
    scale, pairs = 1.0, []
    for raw in Path(path).read_text().splitlines():
        text = raw.strip()
        if text.startswith("# scale"):
            scale = float(text.split()[-1])
        elif text:
            a, b = text.split()
            pairs.append((int(a), int(b)))
    cols = np.array(pairs, dtype=np.int64).reshape(-1, 2)
    return cols[:, 0].copy(), cols[:, 1].copy(), scale


__all__ = ["BudgetError", "CdcConfig", "FntCdcEngine", "design_cd_taps", "fd_cdc_float",
           "td_cdc_float", "required_taps", "quantize_taps", "save_taps", "load_taps",
           "FermatParams", "BudgetReport"]
