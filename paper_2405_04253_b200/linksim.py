"""Link configuration, FEC metrology helpers and the GPU CDC->AEQ chain
(the parts of fntdsp/linksim.py the FNT hot path touches).

The reference's link *simulator* (Tx, channel, front end; linksim.py:105-246) is
host-side data generation and is out of scope as a product;
`LinkConfig` here carries the same fields and derived quantities so callers
configure the engines exactly as before, and `rx_equalize` runs the ★ glue of
linksim.py:283-308 / 399-406 on the GPU: CDC per polarization (fused
requantization and decimation statistics), decimation-phase choice, and the
FNT-AEQ on the decimated streams.
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
        max_int = (1 << (self.sig_bits - 1)) - 1
        return self.load_fraction * max_int / _OUTER_MODULUS

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
        return lambda i: self.mu1 if i < self.gear_symbols else self.mu2


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
    """SNR where a BER curve crosses the FEC threshold, log-interpolated (linksim.py:439-454)."""
    snrs = np.asarray(snrs, dtype=float)
    bers = np.asarray(bers, dtype=float)
    order = np.argsort(snrs)
    snrs, bers = snrs[order], bers[order]
    logt = math.log10(threshold)
    for i in range(len(snrs) - 1):
        b0, b1 = bers[i], bers[i + 1]
        if b0 >= threshold >= b1 and b1 > 0:
            l0, l1 = math.log10(b0), math.log10(b1)
            if l0 == l1:
                return float(snrs[i])
            frac = (l0 - logt) / (l0 - l1)
            return float(snrs[i] + frac * (snrs[i + 1] - snrs[i]))
    raise ValueError("BER curve does not cross the FEC threshold")


def penalty_at_fec(rows: list[Metrics], scheme_a: str, scheme_b: str,
                   threshold: float = HD_FEC_BER) -> float:
    def crossing(scheme):
        pts = [(m.snr_db, m.ber) for m in rows if m.scheme == scheme]
        return fec_crossing_snr([p[0] for p in pts], [p[1] for p in pts], threshold)
    return crossing(scheme_a) - crossing(scheme_b)


def run_single(cfg: LinkConfig, scheme: str, snr_db: float) -> Metrics:
    raise NotImplementedError(
        "the link simulator (Tx/channel/front end) is host-side data generation, out of "
        "scope for the GPU hot path; use paper_2405_04253_b200.stream.rx_equalize on "
        "quantized front-end samples")


def run_link(cfg: LinkConfig) -> list[Metrics]:
    raise NotImplementedError(run_single.__doc__ or "see run_single")
