"""numpy restatement of the reference link model -- TEST INFRASTRUCTURE ONLY.

Regenerates, bit for bit, the quantized front-end samples of BASELINE configs
2, 3 and 5 (so full-size parity runs on the GPU box, where the reference does
not exist), and computes BER / EVM with the reference's metrology so GPU
outputs can be reported next to the reference's numbers. Pinned: the digests of
its outputs are checked against digests produced by the reference itself
(tests/golden/digests.json, written by tests/golden/make_golden.py).

Restated reference functions (fntdsp/linksim.py): bits_to_symbols 107-112,
rrc_taps 136-153, circ_filter 156-163, frac_delay 166-171, generate_tx 183-193,
cd_allpass 198-208, apply_channel 211-234, gsop 239-246, front end 272-291,
hard_decision 115-121, symbols_to_bits 124-133, carrier_recovery 312-321,
_circ_xcorr 326-330, align_and_count 333-374. fixedpoint.quantize_real 51-60.
"""

from __future__ import annotations

import math

import numpy as np

C0 = 299792458.0
QAM_NORM = math.sqrt(10.0)
AXIS = np.array([-3.0, -1.0, 3.0, 1.0])
LEVEL_BITS = {-3: (0, 0), -1: (0, 1), 1: (1, 1), 3: (1, 0)}


class Link:
    """The LinkConfig fields the generator needs (defaults of linksim.LinkConfig)."""

    def __init__(self, n_symbols, z_km, seed, snr_db=20.0, rotation_deg=45.0, dgd=0.2, skew=0.1,
                 baud=40e9, sps=2, rolloff=0.1, span=64, D=17.0, lam_nm=1550.0, sig_bits=5,
                 load=0.8, discard=20000):
        self.n_symbols, self.z_km, self.seed, self.snr_db = n_symbols, z_km, seed, snr_db
        self.rotation_deg, self.dgd, self.skew = rotation_deg, dgd, skew
        self.baud, self.sps, self.rolloff, self.span = baud, sps, rolloff, span
        self.D, self.lam_nm, self.sig_bits, self.load, self.discard = D, lam_nm, sig_bits, load, discard

    @property
    def fs(self):
        return self.baud * self.sps

    @property
    def sig_scale(self):
        return self.load * ((1 << (self.sig_bits - 1)) - 1) / math.sqrt(18.0 / 10.0)


def rrc(sps, span, beta):
    n = span * sps + 1
    t = (np.arange(n) - (n - 1) / 2) / sps
    h = np.zeros(n)
    for k, ti in enumerate(t):
        if abs(ti) < 1e-12:
            h[k] = 1.0 - beta + 4 * beta / math.pi
        elif beta > 0 and abs(abs(ti) - 1 / (4 * beta)) < 1e-9:
            h[k] = (beta / math.sqrt(2)) * (
                (1 + 2 / math.pi) * math.sin(math.pi / (4 * beta))
                + (1 - 2 / math.pi) * math.cos(math.pi / (4 * beta)))
        else:
            num = (math.sin(math.pi * ti * (1 - beta))
                   + 4 * beta * ti * math.cos(math.pi * ti * (1 + beta)))
            den = math.pi * ti * (1 - (4 * beta * ti) ** 2)
            h[k] = num / den
    return h / np.linalg.norm(h)


def circ(x, taps):
    n = len(x)
    th = np.zeros(n, dtype=complex)
    m = len(taps)
    th[:m] = taps
    th = np.roll(th, -(m // 2))
    return np.fft.ifft(np.fft.fft(x) * np.fft.fft(th))


def fdelay(x, tau):
    f = np.fft.fftfreq(len(x))
    y = np.fft.ifft(np.fft.fft(x) * np.exp(-2j * np.pi * f * tau))
    return y.real if np.isrealobj(x) else y


def symbols_of(bits):
    b = np.asarray(bits)
    return (AXIS[b[..., 0] * 2 + b[..., 1]] + 1j * AXIS[b[..., 2] * 2 + b[..., 3]]) / QAM_NORM


def transmit(L: Link, rng):
    bits = rng.integers(0, 2, size=(2, L.n_symbols, 4))
    sym = symbols_of(bits)
    shaping = rrc(L.sps, L.span, L.rolloff)
    wave = np.zeros((2, L.n_symbols * L.sps), dtype=complex)
    for p in range(2):
        up = np.zeros(L.n_symbols * L.sps, dtype=complex)
        up[::L.sps] = sym[p]
        w = circ(up, shaping)
        wave[p] = w / math.sqrt(np.mean(np.abs(w) ** 2))
    return bits, sym, wave


def dispersion(wave, L: Link, compensate=False):
    n = wave.shape[-1]
    f = np.fft.fftfreq(n, 1.0 / L.fs)
    d_si = L.D * 1e-6
    lam = L.lam_nm * 1e-9
    phase = math.pi * lam * lam * d_si * (L.z_km * 1e3) / C0
    sign = 1.0 if compensate else -1.0
    return np.fft.ifft(np.fft.fft(wave, axis=-1) * np.exp(sign * 1j * phase * f * f), axis=-1)


def awgn(x, snr_db, rng, use_math_sqrt=True):
    if np.isfinite(snr_db):
        snr = 10.0 ** (snr_db / 10.0)
        for p in range(2):
            pw = np.mean(np.abs(x[p]) ** 2)
            sigma = math.sqrt(pw / snr / 2.0) if use_math_sqrt else np.sqrt(pw / snr / 2.0)
            x[p] = x[p] + sigma * (rng.standard_normal(x.shape[-1])
                                   + 1j * rng.standard_normal(x.shape[-1]))
    return x


def channel(wave, L: Link, rng):
    """apply_channel: dispersion, DGD, real rotation, IQ skew, AWGN."""
    x = dispersion(wave, L)
    tau = L.dgd * L.sps / 2.0
    x = np.stack([fdelay(x[0], tau), fdelay(x[1], -tau)])
    th = math.radians(L.rotation_deg)
    rot = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    x = rot @ x
    if L.skew:
        x = np.stack([p.real + 1j * fdelay(p.imag, L.skew) for p in x])
    return awgn(x, L.snr_db, rng)


def channel_jones(wave, L: Link, rng, jones):
    """Config 3 / 5 harness channel: dispersion, seeded Haar Jones matrix, AWGN."""
    x = dispersion(wave, L)
    x = jones @ x
    return awgn(x, L.snr_db, rng, use_math_sqrt=False)


def gs_orth(x):
    i = x.real
    q = x.imag
    i_n = i / math.sqrt(np.mean(i * i))
    q_o = q - np.mean(q * i_n) * i_n
    q_n = q_o / math.sqrt(np.mean(q_o * q_o))
    return (i_n + 1j * q_n) / math.sqrt(2.0)


def quantize(x, scale, max_int):
    v = np.asarray(x, dtype=float) * scale
    v = np.sign(v) * np.floor(np.abs(v) + 0.5)
    return np.clip(v, -max_int, max_int).astype(np.int64)


def conditioned(rx, L: Link, use_np_sqrt=True):
    """GSOP, RRC matched filter, unit power (linksim.py:272-277) -> complex128 per pol,
    the float samples rx_frontend quantizes (linksim.py:289-291)."""
    mf = rrc(L.sps, L.span, L.rolloff)
    out = []
    for p in range(2):
        g = gs_orth(rx[p])
        m = circ(g, mf)
        out.append(m / (np.sqrt(np.mean(np.abs(m) ** 2)) if use_np_sqrt
                        else math.sqrt(np.mean(np.abs(m) ** 2))))
    return out


def front_end(rx, L: Link, use_np_sqrt=True):
    """GSOP, RRC matched filter, unit power, 5-bit quantize -> [(xr, xi)] per pol."""
    mx = (1 << (L.sig_bits - 1)) - 1
    return [(quantize(c.real, L.sig_scale, mx), quantize(c.imag, L.sig_scale, mx))
            for c in conditioned(rx, L, use_np_sqrt)]


def config2():
    """BASELINE config 2: returns (tx bits, tx symbols, [(xr, xi)] per pol)."""
    L = Link(2 ** 18, 75.0, 1, snr_db=20.0, rotation_deg=0.0, dgd=0.0, skew=0.0)
    rng = np.random.default_rng(np.random.SeedSequence([1, 20000]))
    bits, sym, wave = transmit(L, rng)
    rx = channel(wave, L, rng)
    return L, bits, sym, front_end(rx, L)


def config2_float():
    """Config 2's front-end float samples (complex128 per pol) before the 5-bit quantizer."""
    L = Link(2 ** 18, 75.0, 1, snr_db=20.0, rotation_deg=0.0, dgd=0.0, skew=0.0)
    rng = np.random.default_rng(np.random.SeedSequence([1, 20000]))
    bits, sym, wave = transmit(L, rng)
    rx = channel(wave, L, rng)
    return L, conditioned(rx, L)


def config3(snr_db: float):
    """BASELINE config 3 at one SNR point (seed 2, Haar Jones)."""
    from scipy.stats import unitary_group
    L = Link(2 ** 20, 75.0, 2, snr_db=snr_db, rotation_deg=0.0, dgd=0.0, skew=0.0)
    jones = unitary_group.rvs(2, random_state=np.random.default_rng(np.random.SeedSequence([2, 999999])))
    rng = np.random.default_rng(np.random.SeedSequence([2, int(round(snr_db * 1000))]))
    bits, sym, wave = transmit(L, rng)
    rx = channel_jones(wave, L, rng, jones)
    return L, bits, sym, front_end(rx, L)


def config5(i: int, n_symbols: int = 2 ** 18):
    """BASELINE config 5, link i: rng_i = default_rng(SeedSequence([4, i])),
    snr ~ U[16, 22] dB, Haar Jones from rng_i, then Tx / channel / front end on rng_i."""
    from scipy.stats import unitary_group
    rng = np.random.default_rng(np.random.SeedSequence([4, i]))
    snr = rng.uniform(16, 22)
    jones = unitary_group.rvs(2, random_state=rng)
    L = Link(n_symbols, 75.0, 4, snr_db=snr, rotation_deg=0.0, dgd=0.0, skew=0.0)
    bits, sym, wave = transmit(L, rng)
    rx = channel_jones(wave, L, rng, jones)
    return L, bits, sym, front_end(rx, L)


# ---------------------------------------------------------------- metrology

def hard_decision(y):
    lv = np.array([-3.0, -1.0, 1.0, 3.0])
    edges = np.array([-2.0, 0.0, 2.0])
    return (lv[np.digitize(y.real * QAM_NORM, edges)] + 1j * lv[np.digitize(y.imag * QAM_NORM, edges)]) / QAM_NORM


def bits_of(sym):
    out = np.zeros(sym.shape + (4,), dtype=np.int64)
    for axis, part in enumerate([sym.real, sym.imag]):
        lv = np.rint(part * QAM_NORM).astype(int)
        for level, (b0, b1) in LEVEL_BITS.items():
            m = lv == level
            out[..., 2 * axis + 0][m] = b0
            out[..., 2 * axis + 1][m] = b1
    return out


def carrier(y, iterations=3):
    total = 0.0
    for _ in range(iterations):
        d = hard_decision(y)
        phi = float(np.angle(np.vdot(d, y)))
        y = y * np.exp(-1j * phi)
        total += phi
    return y, total


def xcorr(y, s):
    c = np.fft.ifft(np.fft.fft(y) * np.conj(np.fft.fft(s)))
    lag = int(np.argmax(np.abs(c)))
    return lag, c[lag] / len(y)


def ber_evm(y_pols, bits, sym, discard):
    """align_and_count (linksim.py:333-374) -> (ber, evm_db, ok)."""
    n = sym.shape[1]
    assign = []
    for p in range(2):
        scores = []
        for q in range(2):
            lag, gain = xcorr(y_pols[p], sym[q])
            scores.append((abs(gain), q, lag, gain))
        scores.sort(reverse=True)
        assign.append(scores[0])
    if assign[0][1] == assign[1][1]:
        return 0.5, 0.0, False
    errors = total_bits = 0
    ev_num = ev_den = 0.0
    for p in range(2):
        _, q, lag, gain = assign[p]
        y = np.roll(y_pols[p], -lag)
        quad = np.round(np.angle(gain) / (math.pi / 2)) * (math.pi / 2)
        y = y * np.exp(-1j * quad)
        y, _ = carrier(y)
        y = y[discard:n]
        ref_sym = sym[q][discard:n]
        ref_bits = bits[q][discard:n]
        det = bits_of(hard_decision(y))
        errors += int(np.count_nonzero(det != ref_bits))
        total_bits += ref_bits.size
        ev_num += float(np.sum(np.abs(y - ref_sym) ** 2))
        ev_den += float(np.sum(np.abs(ref_sym) ** 2))
    ber = errors / total_bits
    evm_db = 10.0 * math.log10(ev_num / ev_den) if ev_num > 0 else -math.inf
    return ber, evm_db, True
