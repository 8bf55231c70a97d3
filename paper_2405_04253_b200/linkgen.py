"""On-device synthetic link generator (bench input data).

Produces the FNT-CDC input of BASELINE configs 4/5 directly in HBM: Gray 16QAM
at 2 samples/symbol, root-raised-cosine shaping (roll-off 0.1, 64-symbol span),
chromatic dispersion (D = 17 ps/nm/km at 1550 nm), a Haar-random Jones matrix
per link, AWGN at a per-link SNR, then the receiver front end (Gram-Schmidt
orthonormalisation, matched filter, unit-power normalisation) and the 5-bit
quantizer -- the signal model of the reference simulator (linksim.py:183-291),
with circular FFT filtering as there.

This is data generation, not the product path: it uses PyTorch tensors and
cuFFT (library code) and is statistically, not bitwise, equivalent to the
reference's numpy generator (different RNG; tests/test_gpu_linkgen.py compares
the level histograms and spectra with oracle/linkgen_np, the pinned restatement
of the reference generator). Bit-exact parity tests use inputs produced by the
reference itself (tests/golden/).

Randomness is counter-based: torch's CUDA generator is Philox4x32-10, and every
group of `chunk` links is drawn from a generator keyed by (seed, global index of
the group's first link) -- never by rank or shard. A shard [first, first + n)
therefore holds exactly the links an unsharded run holds at those indices, for
any number of GPUs (config 5 strong scaling; config 4 keys its segments the same
way by global segment index).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib

SPEED_OF_LIGHT = 299792458.0


def rrc_taps(sps: int, span: int, beta: float) -> np.ndarray:
    """Unit-energy root-raised-cosine impulse response over `span` symbols."""
    n = span * sps + 1
    t = (np.arange(n) - (n - 1) / 2) / sps
    h = np.empty(n)
    for k, tk in enumerate(t):
        if abs(tk) < 1e-12:
            h[k] = 1.0 - beta + 4 * beta / math.pi
        elif beta > 0 and abs(abs(tk) - 1 / (4 * beta)) < 1e-9:
            h[k] = (beta / math.sqrt(2)) * ((1 + 2 / math.pi) * math.sin(math.pi / (4 * beta))
                                            + (1 - 2 / math.pi) * math.cos(math.pi / (4 * beta)))
        else:
            h[k] = ((math.sin(math.pi * tk * (1 - beta))
                     + 4 * beta * tk * math.cos(math.pi * tk * (1 + beta)))
                    / (math.pi * tk * (1 - (4 * beta * tk) ** 2)))
    return h / np.linalg.norm(h)


class DeviceLinkGenerator:
    """Generates quantized front-end I/Q for many dual-pol links on the GPU."""

    def __init__(self, n_symbols: int, z_km: float = 75.0, baud: float = 40e9, sps: int = 2,
                 rolloff: float = 0.1, span: int = 64, dispersion_ps_nm_km: float = 17.0,
                 wavelength_nm: float = 1550.0, sig_scale: float | None = None,
                 sig_bits: int = 5, dgd_symbols: float = 0.0, iq_skew_samples: float = 0.0):
        t = _lib.torch()
        dev = _lib.device()
        self.n_sym = n_symbols
        self.sps = sps
        self.L = n_symbols * sps
        self.sig_scale = (0.8 * ((1 << (sig_bits - 1)) - 1) / math.sqrt(1.8)
                          if sig_scale is None else sig_scale)
        self.max_int = (1 << (sig_bits - 1)) - 1
        L = self.L
        taps = rrc_taps(sps, span, rolloff)
        if taps.size > L:
            raise ValueError(f"n_symbols * sps = {L} is shorter than the {taps.size}-tap RRC "
                             f"pulse (circular shaping needs at least span * sps + 1 samples)")
        th = np.zeros(L, dtype=complex)
        th[:taps.size] = taps
        th = np.roll(th, -(taps.size // 2))
        self.H_rrc = t.fft.fft(t.from_numpy(th).to(dev))
        fs = baud * sps
        f = t.fft.fftfreq(L, 1.0 / fs, dtype=t.float64, device=dev)
        lam = wavelength_nm * 1e-9
        phase = math.pi * lam * lam * (dispersion_ps_nm_km * 1e-6) * (z_km * 1e3) / SPEED_OF_LIGHT
        self.H_tx = self.H_rrc * t.exp(-1j * phase * f * f)  # shaping + dispersion
        # DGD: pol X delayed by +tau, pol Y by -tau samples (apply_channel, linksim.py:220-222);
        # IQ skew: the quadrature part delayed by iq_skew samples (linksim.py:227-229)
        fn = t.fft.fftfreq(L, dtype=t.float64, device=dev)
        tau = dgd_symbols * sps / 2.0
        self.H_pol = None
        if tau:
            self.H_pol = t.stack([t.exp(-2j * math.pi * fn * tau), t.exp(2j * math.pi * fn * tau)])
        self.H_skew = t.exp(-2j * math.pi * fn * iq_skew_samples) if iq_skew_samples else None
        self.levels = t.tensor([-3.0, -1.0, 3.0, 1.0], dtype=t.float64, device=dev) / math.sqrt(10.0)

    def generate(self, n_links: int, seed: int, snr_db=(16.0, 22.0), chunk: int = 32,
                 out=None, symbols: bool = False, first_link: int = 0):
        """Returns (xr, xi): (2*n_links, L) int8 device tensors for the links with
        global indices [first_link, first_link + n_links); row 2l = pol X of link l,
        row 2l+1 = pol Y. Link i's samples depend only on (seed, i) (and `chunk`):
        the Philox generator of each aligned group of `chunk` links is keyed by the
        group's global index. With symbols=True also returns the transmitted symbol
        indices (n_links, 2, n_sym) uint8 = 4*li_I + li_Q with Gray level index
        li = 2 b0 + b1 (the reference's bits_to_symbols, linksim.py:107-112)."""
        t = _lib.torch()
        dev = _lib.device()
        L = self.L
        if out is None:
            xr = t.empty((2 * n_links, L), dtype=t.int8, device=dev)
            xi = t.empty((2 * n_links, L), dtype=t.int8, device=dev)
        else:
            xr, xi = out
        sidx = t.empty((n_links, 2, self.n_sym), dtype=t.uint8, device=dev) if symbols else None
        end = first_link + n_links
        for g0 in range(first_link - first_link % chunk, end, chunk):
            g = t.Generator(device=dev)
            g.manual_seed(int(seed) * 1_000_003 + g0)
            xq_r, xq_i, li = self._chunk(chunk, g, snr_db)
            a, b = max(g0, first_link), min(g0 + chunk, end)   # global links kept
            ra, rb = a - g0, b - g0                            # rows of the group
            xr[2 * (a - first_link):2 * (b - first_link)] = xq_r[ra:rb].reshape(2 * (b - a), L)
            xi[2 * (a - first_link):2 * (b - first_link)] = xq_i[ra:rb].reshape(2 * (b - a), L)
            if symbols:
                sidx[a - first_link:b - first_link] = li[ra:rb]
        return (xr, xi, sidx) if symbols else (xr, xi)

    def tx_reference(self, sidx):
        """Symbol indices -> (symbols complex128, bits int8 (..., 4)) on the device."""
        t = _lib.torch()
        li_i = (sidx >> 2).long()
        li_q = (sidx & 3).long()
        sym = t.complex(self.levels[li_i], self.levels[li_q])
        bits = t.stack([li_i >> 1, li_i & 1, li_q >> 1, li_q & 1], dim=-1).to(t.int8)
        return sym, bits

    def _chunk(self, c: int, g, snr_db):
        t = _lib.torch()
        dev = _lib.device()
        L, n = self.L, self.n_sym
        li_i = t.randint(0, 4, (c, 2, n), generator=g, device=dev)
        li_q = t.randint(0, 4, (c, 2, n), generator=g, device=dev)
        sym_i = self.levels[li_i]
        sym_q = self.levels[li_q]
        up = t.zeros((c, 2, L), dtype=t.complex128, device=dev)
        up[..., ::self.sps] = t.complex(sym_i, sym_q)
        Hx = self.H_tx if self.H_pol is None else self.H_tx * self.H_pol
        w = t.fft.ifft(t.fft.fft(up) * Hx)
        del up
        w = w / t.sqrt(t.mean(w.abs() ** 2, dim=-1, keepdim=True))
        # Haar-random 2x2 unitary per link (QR of a complex Ginibre matrix, phase-fixed)
        z = t.complex(t.randn((c, 2, 2), generator=g, device=dev, dtype=t.float64),
                      t.randn((c, 2, 2), generator=g, device=dev, dtype=t.float64)) / math.sqrt(2)
        q, r = t.linalg.qr(z)
        d = t.diagonal(r, dim1=-2, dim2=-1)
        q = q * (d / d.abs()).unsqueeze(-2)
        w = t.matmul(q, w)
        if self.H_skew is not None:
            w = t.complex(w.real, t.fft.ifft(t.fft.fft(w.imag) * self.H_skew).real)
        lo, hi = snr_db
        snr = 10.0 ** ((lo + (hi - lo) * t.rand((c, 1, 1), generator=g, device=dev,
                                                   dtype=t.float64)) / 10.0)
        pw = t.mean(w.abs() ** 2, dim=-1, keepdim=True)
        sigma = t.sqrt(pw / snr / 2.0)
        noise = t.complex(t.randn((c, 2, L), generator=g, device=dev, dtype=t.float64),
                          t.randn((c, 2, L), generator=g, device=dev, dtype=t.float64))
        w = w + sigma * noise
        del noise
        # receiver: GSOP, matched filter, unit power (linksim.py:239-246, 272-277)
        i = w.real
        qv = w.imag
        i_n = i / t.sqrt(t.mean(i * i, dim=-1, keepdim=True))
        q_o = qv - t.mean(qv * i_n, dim=-1, keepdim=True) * i_n
        q_n = q_o / t.sqrt(t.mean(q_o * q_o, dim=-1, keepdim=True))
        gs = t.complex(i_n, q_n) / math.sqrt(2.0)
        m = t.fft.ifft(t.fft.fft(gs) * self.H_rrc)
        m = m / t.sqrt(t.mean(m.abs() ** 2, dim=-1, keepdim=True))

        def quant(v):
            v = v * self.sig_scale
            v = t.sign(v) * t.floor(v.abs() + 0.5)
            return v.clamp(-self.max_int, self.max_int).to(t.int8)
        return quant(m.real), quant(m.imag), (4 * li_i + li_q).to(t.uint8)
