"""numpy restatement of the reference's array-at-a-time algorithm -- TEST AND
BASELINE INFRASTRUCTURE ONLY (bench.py cpu_baseline / --impl reference; tests).

It reproduces fntdsp's computation with the same numpy operations and the same
cost profile (whole-stream blocking, stage-by-stage vectorised butterflies over
int64 arrays, a Python loop over AEQ blocks with numpy's einsum), so timing it
on the GPU box's host cores stands in for timing the reference itself, which
cannot travel to the box. Parity: pinned by tests/test_np_port.py against the
reference's golden fixtures.

Restated reference functions (fntdsp/...):
  NpPlan              fnt.py:46-83     make_plan tables
  transform           fnt.py:86-114    _butterflies / fnt / ifnt
  cdc_process_int     cdc.py:89-95, 124-175
  NpAeq               aeq.py:84-190    equalize_block / update_taps / process
  quantize_real       fixedpoint.py:51-60
"""

from __future__ import annotations

import math

import numpy as np


class NpPlan:
    def __init__(self, F: int, alpha: int, n: int):
        self.F, self.alpha, self.n = F, alpha, n
        lg = n.bit_length() - 1
        self.alpha_inv = pow(alpha, -1, F)
        self.n_inv = pow(n, -1, F)
        k = np.arange(n)
        self.bitrev = np.zeros(n, dtype=np.int64)
        for b in range(lg):
            self.bitrev |= ((k >> b) & 1) << (lg - 1 - b)
        self.fwd = [np.array([pow(alpha, j * (n >> (s + 1)), F) for j in range(1 << s)], np.int64)
                    for s in range(lg)]
        self.inv = [np.array([pow(self.alpha_inv, j * (n >> (s + 1)), F) for j in range(1 << s)],
                             np.int64) for s in range(lg)]


CDC64 = NpPlan(65537, 4080, 64)
AEQ32 = NpPlan(65537, 2, 32)


def transform(p: NpPlan, x: np.ndarray, inverse: bool = False) -> np.ndarray:
    F = p.F
    a = np.asarray(x, dtype=np.int64)[..., p.bitrev]
    lead = a.shape[:-1]
    for tw in (p.inv if inverse else p.fwd):
        h = tw.shape[0]
        g = a.reshape(*lead, -1, 2, h)
        top = g[..., 0, :]
        bot = (g[..., 1, :] * tw) % F
        a = np.stack(((top + bot) % F, (top - bot) % F), axis=-2).reshape(*lead, p.n)
    if inverse:
        a = (a * p.n_inv) % F
    return a


def _enc(v, F):
    return np.where(v >= 0, v, v + F)


def _dec(r, F):
    return np.where(r <= (F - 1) // 2, r, r - F)


def quantize_real(x, scale: float, max_int: int):
    v = np.asarray(x, dtype=float) * scale
    v = np.sign(v) * np.floor(np.abs(v) + 0.5)
    clipped = int(np.count_nonzero(np.abs(v) > max_int))
    return np.clip(v, -max_int, max_int).astype(np.int64), clipped


def cdc_spectra(tap_re, tap_im, p: NpPlan = CDC64):
    F = p.F
    h = np.zeros((2, p.n), dtype=np.int64)
    h[0, :len(tap_re)] = tap_re
    h[1, :len(tap_im)] = tap_im
    H = transform(p, _enc(h, F))
    return (H[0] + 256 * H[1]) % F, (H[0] - 256 * H[1]) % F


def cdc_process_int(xr, xi, bp, bm, n_taps: int, p: NpPlan = CDC64):
    """Whole-stream overlap-save through the FNT (cdc.py:141-175)."""
    F, n = p.F, p.n
    hop = n // 2
    L = len(xr)
    nb = -(-(L + hop) // hop)
    pad = np.zeros((2, hop + nb * hop + hop), dtype=np.int64)
    pad[0, hop:hop + L] = xr
    pad[1, hop:hop + L] = xi
    win = np.lib.stride_tricks.sliding_window_view(pad, n, axis=1)[:, ::hop][:, :nb]
    Xr = transform(p, _enc(win[0], F))
    Xi = transform(p, _enc(win[1], F))
    up = (((Xr + 256 * Xi) % F) * bp) % F
    um = (((Xr - 256 * Xi) % F) * bm) % F
    zr = (transform(p, (up + um) % F, True) * (F - (1 << 15))) % F
    zi = (transform(p, (up - um) % F, True) * (F - (1 << 7))) % F
    c = n_taps // 2
    yr = _dec(zr, F)[:, hop:].reshape(-1)[c:c + L]
    yi = _dec(zi, F)[:, hop:].reshape(-1)[c:c + L]
    return yr, yi


class NpAeq:
    """FntAeq's per-block loop in numpy (aeq.py:84-190)."""

    def __init__(self, sig_scale: float, tap_scale: float = 8192.0, mu: float = 1e-4):
        self.sig, self.ts, self.mu = sig_scale, tap_scale, mu
        self.radii = np.sort(np.sqrt(np.array([2.0, 10.0, 18.0]) / 10.0))
        self.w_int = np.zeros((4, 4, 16), dtype=np.int64)
        for s in range(4):
            self.w_int[s, s, 8] = int(round(tap_scale))
        self.w = self.w_int.astype(float) / tap_scale
        self.hist = np.zeros((4, 16), dtype=np.int64)
        self.err_trace: list[float] = []
        self.sat = 0

    def _spectra(self):
        F = AEQ32.F
        sg, mg = np.sign(self.w_int), np.abs(self.w_int)
        pad = np.zeros((2, 4, 4, 32), dtype=np.int64)
        pad[0, :, :, :16] = sg * (mg >> 7)
        pad[1, :, :, :16] = sg * (mg & 127)
        return transform(AEQ32, _enc(pad, F))

    def process(self, x, mu_blocks=None, adapt=True):
        F = AEQ32.F
        x = np.asarray(x, dtype=np.int64)
        nb = x.shape[1] // 16
        out = np.zeros((4, nb * 16))
        W = self._spectra()
        for b in range(nb):
            xb = np.concatenate([self.hist, x[:, 16 * b:16 * b + 16]], axis=1)
            self.hist = x[:, 16 * b:16 * b + 16].copy()
            X = transform(AEQ32, _enc(xb, F))
            conv = _dec(transform(AEQ32, (W * X[None, None]) % F, True), F)
            y = ((conv[0] << 7) + conv[1]).sum(axis=1)[:, 16:] / (self.sig * self.ts)
            out[:, 16 * b:16 * b + 16] = y
            if not adapt:
                continue
            mu = self.mu if mu_blocks is None else mu_blocks[b]
            xf = xb / self.sig
            r2x = y[0] ** 2 + y[1] ** 2
            r2y = y[2] ** 2 + y[3] ** 2
            ex = self.radii[np.argmin(np.abs(np.sqrt(r2x)[:, None] - self.radii), -1)] ** 2 - r2x
            ey = self.radii[np.argmin(np.abs(np.sqrt(r2y)[:, None] - self.radii), -1)] ** 2 - r2y
            e = np.stack([ex, ex, ey, ey])
            self.err_trace.append(float(np.mean(np.abs(np.stack([ex, ey])))))
            if mu == 0.0:
                continue
            lags = np.lib.stride_tricks.sliding_window_view(xf, 16, axis=1)[:, 1:, ::-1]
            self.w += mu * np.einsum("sm,tmk->stk", e * y, lags)
            wi = np.rint(self.w * self.ts).astype(np.int64)
            self.sat += int(np.count_nonzero(np.abs(wi) > 16383))
            self.w_int = np.clip(wi, -16383, 16383)
            W = self._spectra()
        return out


def decimation_phase(streams, sps: int = 2) -> int:
    best, phase = None, 0
    for ph in range(sps):
        m = 0.0
        for s in streams:
            d = s[ph::sps]
            p2 = np.mean(np.abs(d) ** 2)
            m += np.mean(np.abs(d) ** 4) / (p2 * p2)
        if best is None or m < best:
            best, phase = m, ph
    return phase


def chain(xr2, xi2, tap_re, tap_im, n_taps, out_scale, sig_scale, mu_blocks):
    """One dual-pol link through CDC -> glue -> AEQ (linksim.py:283-308, 399-406)."""
    bp, bm = cdc_spectra(tap_re, tap_im)
    eqs = []
    for p in range(2):
        yr, yi = cdc_process_int(xr2[p], xi2[p], bp, bm, n_taps)
        eqs.append((yr + 1j * yi) / out_scale)
    ph = decimation_phase(eqs)
    dec = [e[ph::2] for e in eqs]
    q = np.stack([quantize_real(s, sig_scale, 15)[0]
                  for s in (dec[0].real, dec[0].imag, dec[1].real, dec[1].imag)])
    eq = NpAeq(sig_scale)
    return eq.process(q, mu_blocks=mu_blocks), eq


__all__ = ["NpPlan", "transform", "cdc_process_int", "cdc_spectra", "NpAeq", "chain",
           "quantize_real", "decimation_phase", "math"]
