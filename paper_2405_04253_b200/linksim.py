"""Link configuration, FEC metrology helpers, and the link simulator that drives
the GPU receiver for the CLI `sweep` (the parts of fntdsp/linksim.py the FNT hot
path touches, plus its host-side data generation).

`LinkConfig` carries the reference's fields and derived quantities so callers
configure the engines exactly as before. `run_single` / `run_link` reproduce the
reference's sweep point by point: the transmitter, channel and front-end
conditioning are host-side numpy data generation in the reference's operation
order (a seeded run yields the reference's samples bit for bit), and every DSP
stage after them runs on the GPU -- quantize_real, FntCdcEngine.process (or the
float FD/TD-CDC comparators), FntAeq.process (or the float TD-AEQ kernel), and
the BER/EVM metrology (metrology.py).
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass, field

import numpy as np

from .aeq import AeqConfig
from .cdc import CdcConfig
from .fixedpoint import QuantSpec

HD_FEC_BER = 3.8e-3
_OUTER_MODULUS = math.sqrt(18.0 / 10.0)


@dataclass
class LinkConfig:
    """Same fields and derived quantities as fntdsp.linksim.LinkConfig (linksim.py:32-83)."""

    baud: float = 40e9
    n_symbols: int = 1 << 17
    rrc_rolloff: float = 0.1
    rrc_span: int = 64
    z_km: float = 0.0
    dispersion_ps_nm_km: float = 17.0
    wavelength_nm: float = 1550.0
    snr_db: tuple = (13.0, 14.0, 15.0, 16.0, 17.0, 18.0)
    pol_rotation_deg: float = 45.0
    dgd_symbols: float = 0.2
    iq_skew_samples: float = 0.1
    sps: int = 2
    seed: int = 1234
    discard_symbols: int = 20000
    n_cdc_taps: int = 32
    sig_bits: int = 5
    cdc_tap_bits: int = 6
    aeq_l_taps: int = 16
    mu1: float = 2e-3
    mu2: float = 1e-4
    gear_symbols: int = 20000
    schemes: tuple = ("fnt", "float")
    load_fraction: float = 0.8

    @property
    def fs(self) -> float:
        return self.baud * self.sps

    @property
    def sig_scale(self) -> float:
        """Quantizer scale putting the outer 16QAM modulus at load_fraction."""
        return self.load_fraction * (2 ** (self.sig_bits - 1) - 1) / _OUTER_MODULUS

    def sig_spec(self) -> QuantSpec:
        return QuantSpec(self.sig_bits, self.sig_scale)

    def cdc_config(self, scheme: str = "fnt") -> CdcConfig:
        return CdcConfig(z_km=self.z_km, fs_hz=self.fs,
                         dispersion_ps_nm_km=self.dispersion_ps_nm_km,
                         wavelength_nm=self.wavelength_nm, n_taps=self.n_cdc_taps,
                         tap_bits=self.cdc_tap_bits, scheme=scheme)

    def aeq_config(self) -> AeqConfig:
        return AeqConfig(block_n=2 * self.aeq_l_taps, l_taps=self.aeq_l_taps, mu=self.mu2,
                         sig_spec=self.sig_spec())

    def mu_schedule(self):
        return GearSchedule(self)


class GearSchedule:
    """LinkConfig.mu_schedule (linksim.py:82-83): mu1 before gear_symbols, mu2 after.
    Called per symbol index like the reference's lambda (reading the config's current
    fields, as the lambda's closure does); FntAeq additionally takes the whole
    per-block table from block_mu instead of one Python call per block."""

    __slots__ = ("cfg",)

    def __init__(self, cfg):
        self.cfg = cfg

    def __call__(self, i):
        c = self.cfg
        return c.mu1 if i < c.gear_symbols else c.mu2

    def block_mu(self, n_blocks: int, hop: int):
        """mu of blocks 0 .. n_blocks-1 (symbol index b * hop), or None when a field
        is not a plain number (the caller then calls the schedule per block)."""
        c = self.cfg
        try:
            mu1, mu2, gear = float(c.mu1), float(c.mu2), c.gear_symbols
            i = np.arange(n_blocks, dtype=np.int64) * hop
            return np.where(i < gear, mu1, mu2).astype(np.float64)
        except (TypeError, ValueError):
            return None


@dataclass
class Metrics:
    scheme: str
    snr_db: float
    ber: float
    evm_db: float
    est_snr_db: float
    q_db: float
    n_bits: int
    clip_fraction: float
    converged: bool
    stage_power: dict = field(default_factory=dict)

    def as_row(self) -> dict:
        d = asdict(self)
        d.pop("stage_power")
        return d


def fec_crossing_snr(snrs, bers, threshold: float = HD_FEC_BER) -> float:
    """SNR at which a BER curve falls through the FEC threshold: the first adjacent
    pair (in SNR order) bracketing it, interpolated linearly in log10(BER)
    (linksim.py:439-454)."""
    order = np.argsort(np.asarray(snrs, dtype=float))
    x = np.asarray(snrs, dtype=float)[order]
    y = np.asarray(bers, dtype=float)[order]
    logt = math.log10(threshold)
    for (x0, x1), (y0, y1) in zip(zip(x[:-1], x[1:]), zip(y[:-1], y[1:])):
        if not (y0 >= threshold >= y1 and y1 > 0):
            continue
        l0, l1 = math.log10(y0), math.log10(y1)
        if l0 == l1:
            return float(x0)
        frac = (l0 - logt) / (l0 - l1)
        return float(x0 + frac * (x1 - x0))
    raise ValueError("BER curve does not cross the FEC threshold")


def penalty_at_fec(rows: list[Metrics], scheme_a: str, scheme_b: str,
                   threshold: float = HD_FEC_BER) -> float:
    """FEC-threshold SNR of scheme_a minus that of scheme_b (linksim.py:457-466)."""
    def at_fec(name):
        curve = [(m.snr_db, m.ber) for m in rows if m.scheme == name]
        return fec_crossing_snr([c[0] for c in curve], [c[1] for c in curve], threshold)
    return at_fec(scheme_a) - at_fec(scheme_b)


# ---------------------------------------------------------------- link simulator
# Host-side data generation (linksim.py:105-246, 272-277): numpy in the reference's
# operation order, so seeded runs give the reference's samples bit for bit.

_GRAY_LEVELS = np.array([-3.0, -1.0, 3.0, 1.0])   # level of Gray bit pair b0 b1 (index 2 b0 + b1)
_QAM_NORM = math.sqrt(10.0)
SPEED_OF_LIGHT = 299792458.0


@dataclass
class TxData:
    bits: np.ndarray       # (2, n_symbols, 4)
    symbols: np.ndarray    # (2, n_symbols) complex, unit average energy
    wave: np.ndarray       # (2, n_symbols * sps), unit average power


def _gray_16qam(bits: np.ndarray) -> np.ndarray:
    i = _GRAY_LEVELS[bits[..., 0] * 2 + bits[..., 1]]
    q = _GRAY_LEVELS[bits[..., 2] * 2 + bits[..., 3]]
    return (i + 1j * q) / _QAM_NORM


def _circular(x: np.ndarray, taps: np.ndarray) -> np.ndarray:
    """Zero-delay circular filtering: taps centred on the origin."""
    kernel = np.zeros(len(x), dtype=complex)
    kernel[:len(taps)] = taps
    kernel = np.roll(kernel, -(len(taps) // 2))
    return np.fft.ifft(np.fft.fft(x) * np.fft.fft(kernel))


def _delayed(x: np.ndarray, tau: float) -> np.ndarray:
    """Circular fractional delay by tau samples (real stays real)."""
    y = np.fft.ifft(np.fft.fft(x) * np.exp(-2j * np.pi * np.fft.fftfreq(len(x)) * tau))
    return y.real if np.isrealobj(x) else y


def _unit_power(w: np.ndarray) -> np.ndarray:
    return w / math.sqrt(np.mean(np.abs(w) ** 2))


def generate_tx(cfg: LinkConfig, rng: np.random.Generator) -> TxData:
    """Random Gray 16QAM on both polarizations, RRC-shaped at cfg.sps."""
    from .linkgen import rrc_taps
    bits = rng.integers(0, 2, size=(2, cfg.n_symbols, 4))
    symbols = _gray_16qam(bits)
    shaping = rrc_taps(cfg.sps, cfg.rrc_span, cfg.rrc_rolloff)
    wave = np.zeros((2, cfg.n_symbols * cfg.sps), dtype=complex)
    for p in range(2):
        up = np.zeros(cfg.n_symbols * cfg.sps, dtype=complex)
        up[::cfg.sps] = symbols[p]
        wave[p] = _unit_power(_circular(up, shaping))
    return TxData(bits=bits, symbols=symbols, wave=wave)


def apply_channel(wave: np.ndarray, cfg: LinkConfig, snr_db: float,
                  rng: np.random.Generator) -> tuple[np.ndarray, dict]:
    """Dispersion all-pass, DGD, real polarization rotation, IQ skew, AWGN."""
    report = {"p_in": float(np.mean(np.abs(wave) ** 2))}
    f = np.fft.fftfreq(wave.shape[-1], 1.0 / cfg.fs)
    lam = cfg.wavelength_nm * 1e-9
    beta = math.pi * lam * lam * (cfg.dispersion_ps_nm_km * 1e-6) * (cfg.z_km * 1e3) / SPEED_OF_LIGHT
    x = np.fft.ifft(np.fft.fft(wave, axis=-1) * np.exp(-1.0 * 1j * beta * f * f), axis=-1)
    tau = cfg.dgd_symbols * cfg.sps / 2.0
    x = np.stack([_delayed(x[0], tau), _delayed(x[1], -tau)])
    th = math.radians(cfg.pol_rotation_deg)
    x = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]]) @ x
    if cfg.iq_skew_samples:
        x = np.stack([p.real + 1j * _delayed(p.imag, cfg.iq_skew_samples) for p in x])
    report["p_channel"] = float(np.mean(np.abs(x) ** 2))
    if np.isfinite(snr_db):
        lin = 10.0 ** (snr_db / 10.0)
        for p in range(2):
            sigma = math.sqrt(np.mean(np.abs(x[p]) ** 2) / lin / 2.0)
            x[p] = x[p] + sigma * (rng.standard_normal(x.shape[-1])
                                   + 1j * rng.standard_normal(x.shape[-1]))
    report["p_out"] = float(np.mean(np.abs(x) ** 2))
    return x, report


def _gram_schmidt(x: np.ndarray) -> np.ndarray:
    i_n = x.real / math.sqrt(np.mean(x.real * x.real))
    q_o = x.imag - np.mean(x.imag * i_n) * i_n
    return (i_n + 1j * (q_o / math.sqrt(np.mean(q_o * q_o)))) / math.sqrt(2.0)


def rx_frontend(rx: np.ndarray, cfg: LinkConfig, scheme: str) -> tuple[np.ndarray, dict]:
    """GSOP, matched filter, unit power (host); then on the GPU the quantizer and the
    FNT-CDC ("fnt") or the float CDC comparators; the sampling phase with the
    reference's float64 metric. Returns the symbol-rate streams (2, n) and a report."""
    from .cdc import FntCdcEngine, design_cd_taps, fd_cdc_float, td_cdc_float
    from .fixedpoint import quantize_real
    from .linkgen import rrc_taps
    from .stream import reference_phase
    mf = rrc_taps(cfg.sps, cfg.rrc_span, cfg.rrc_rolloff)
    conditioned = [_unit_power(_circular(_gram_schmidt(rx[p]), mf)) for p in range(2)]
    report = {"p_frontend": float(np.mean([np.mean(np.abs(c) ** 2) for c in conditioned]))}
    cdc_cfg = cfg.cdc_config(scheme)
    if scheme == "fnt":
        spec = cfg.sig_spec()
        engine = FntCdcEngine(cdc_cfg, spec)
        report["cdc_budget"] = str(engine.budget)
        report["cdc_support_warning"] = engine.support_warning
        equalized, n_clip = [], 0
        for c in conditioned:
            (xr, cr), (xi, ci) = quantize_real(c.real, spec), quantize_real(c.imag, spec)
            n_clip += cr + ci
            equalized.append(engine.process(xr, xi))
        report["clip_fraction"] = n_clip / (2 * 2 * rx.shape[-1])
    elif scheme in ("float", "fd-float", "td-float"):
        taps = design_cd_taps(cdc_cfg)
        comparator = td_cdc_float if scheme == "td-float" else fd_cdc_float
        equalized = [comparator(c, cdc_cfg, taps) for c in conditioned]
        report["clip_fraction"] = 0.0
    else:
        raise ValueError(f"unknown scheme {scheme!r}")
    phase = reference_phase(equalized, cfg.sps)
    report["decimation_phase"] = phase
    return np.stack([e[phase::cfg.sps] for e in equalized]), report


def _q_factor_db(ber: float) -> float:
    """Q factor in dB from the BER of Gray-coded QAM: 20 log10(sqrt(2) erfcinv(2 BER))."""
    if ber <= 0:
        return math.inf
    from scipy.special import erfcinv
    q = math.sqrt(2.0) * float(erfcinv(2.0 * ber))
    return 20.0 * math.log10(q)


def run_single(cfg: LinkConfig, scheme: str, snr_db: float) -> Metrics:
    """One scheme at one SNR point (linksim.py:386-426): the whole chain plus
    metrology, with the reference's per-(seed, SNR) random stream."""
    import torch
    from . import metrology as M
    from .aeq import FntAeq, td_aeq_float
    from .fixedpoint import quantize_real
    rng = np.random.default_rng(np.random.SeedSequence(
        [cfg.seed, int(round(snr_db * 1000)) if np.isfinite(snr_db) else -1]))
    tx = generate_tx(cfg, rng)
    rx, ch_report = apply_channel(tx.wave, cfg, snr_db, rng)
    dec, fe_report = rx_frontend(rx, cfg, scheme)
    streams = np.stack([dec[0].real, dec[0].imag, dec[1].real, dec[1].imag])
    trace = None
    if scheme == "fnt":
        spec = cfg.sig_spec()
        eq = FntAeq(cfg.aeq_config())
        y = eq.process(np.stack([quantize_real(s, spec)[0] for s in streams]), adapt=True,
                       mu_schedule=cfg.mu_schedule())
        trace = eq.err_trace
    else:
        y, _ = td_aeq_float(streams, cfg.aeq_config(), mu_schedule=cfg.mu_schedule())
    n = min(y.shape[1], tx.symbols.shape[1])
    from . import _lib
    y_pols = torch.from_numpy(np.stack([y[0] + 1j * y[1], y[2] + 1j * y[3]])[:, :n]).to(
        _lib.device())[None]
    sym, bits = M.numpy_reference_inputs(tx.bits[:, :n], tx.symbols[:, :n])
    ber, evm_db, ok = (v[0] for v in M.align_and_count(y_pols, sym, bits, cfg.discard_symbols))
    ber, evm_db, ok = float(ber), float(evm_db), bool(ok)
    if trace is not None and len(trace) > 20:
        ok = ok and float(np.mean(trace[-10:])) <= float(np.mean(trace[5:15]))
    return Metrics(scheme=scheme, snr_db=snr_db, ber=ber, evm_db=evm_db, est_snr_db=-evm_db,
                   q_db=_q_factor_db(ber), n_bits=(n - cfg.discard_symbols) * 8,
                   clip_fraction=fe_report.get("clip_fraction", 0.0), converged=ok,
                   stage_power={**ch_report, "frontend": fe_report.get("p_frontend")})


def run_link(cfg: LinkConfig) -> list[Metrics]:
    """Every configured scheme over the SNR list, ordered by (scheme, SNR)."""
    rows = [run_single(cfg, scheme, snr) for scheme in cfg.schemes for snr in cfg.snr_db]
    return sorted(rows, key=lambda m: (m.scheme, m.snr_db))
