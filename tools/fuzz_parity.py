#!/usr/bin/env python3
"""Randomized differential check of the drop-in API against the CPU oracle (run on
the GPU box): FntAeq with random initial taps (float and 14-bit, set independently
as the reference allows), random inputs (5-bit, full int8, wide int32 up to the
encodable +-32768), random step sizes (0, tiny, large enough to saturate), random
lengths, through both stream layouts and both forward forms; FntCdcEngine with random
6-bit taps and random stream lengths / input widths. Every case must be bit-exact
(y, w, w_int, saturations, err_trace; CDC outputs).

    python tools/fuzz_parity.py [--seconds 240] [--seed 1]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402  (the checker)
import paper_2405_04253_b200 as P  # noqa: E402
from paper_2405_04253_b200 import aeq as A  # noqa: E402


def oracle_state(oq, w, w_int, hist):
    ow, owi, oh, _ = oq._view()
    ow[...] = w
    owi[...] = w_int
    oh[...] = hist


def aeq_case(rng, stats):
    kind = rng.choice(["warp", "pol"])
    fwd = rng.choice(["fnt", "direct"])
    sig = float(rng.choice([8.94427190999916, 8.0, 3.3, 12.5]))
    ts = float(rng.choice([8192.0, 4096.0, 1000.0]))
    cfg = P.AeqConfig(sig_spec=P.QuantSpec(5, sig), tap_scale=ts, mu=1e-4)
    prev = A.set_aeq_kernel(kind)
    try:
        eq = P.FntAeq(cfg, forward=P._lib.AEQ_FWD_DIRECT if fwd == "direct" else P._lib.AEQ_FWD_FNT)
    finally:
        A.set_aeq_kernel(prev)
    oq = O.Aeq(sig, ts, mu=1e-4)
    # initial state: centre spikes plus random perturbations (sometimes near the clip)
    w_int = np.zeros((4, 4, 16), np.int64)
    for s in range(4):
        w_int[s, s, 8] = int(round(ts))
    scale = int(rng.choice([0, 30, 600, 9000]))
    w_int += rng.integers(-scale, scale + 1, w_int.shape) if scale else 0
    w_int = np.clip(w_int, -16383, 16383)
    w = w_int / ts + rng.normal(0, 1e-4, w_int.shape) * float(rng.random() < 0.5)
    hist = rng.integers(-15, 16, (4, 16))
    eq.taps = P.RvMimoTaps(w_int.copy())
    eq.w = w.copy()
    eq.history = hist.copy()
    oracle_state(oq, w, w_int, hist)
    n_blocks = int(rng.choice([1, 2, 7, 64, 301, 1000]))
    extra = int(rng.integers(0, 16))
    dist = rng.choice(["5bit", "int8", "wide"])
    n = 16 * n_blocks + extra
    if dist == "5bit":
        x = rng.integers(-15, 16, (4, n))
    elif dist == "int8":
        x = rng.integers(-128, 128, (4, n))
    else:
        x = rng.integers(-40, 41, (4, n))
        spikes = rng.random((4, n)) < 0.01
        x[spikes] = rng.integers(-32768, 32769, int(spikes.sum()))
    mode = rng.choice(["const", "gear", "zero", "big", "noadapt"])
    if mode == "const":
        mu = float(10 ** rng.uniform(-6, -2))
        sched = (lambda i, mu=mu: mu)
    elif mode == "gear":
        g = int(rng.integers(0, 16 * n_blocks + 1))
        sched = (lambda i, g=g: 2e-3 if i < g else 1e-4)
    elif mode == "zero":
        sched = (lambda i: 0.0)
    elif mode == "big":
        sched = (lambda i: 0.5)
    else:
        sched = None
    adapt = mode != "noadapt"
    y = eq.process(x, adapt=adapt, mu_schedule=sched)
    mb = np.array([sched(16 * b) for b in range(n_blocks)]) if adapt else None
    oy = oq.process(x[:, :16 * n_blocks], adapt=adapt, mu_blocks=mb)
    ok = (np.array_equal(y, oy) and np.array_equal(eq.w, oq.w, equal_nan=True)
          and np.array_equal(eq.taps.w_int, oq.w_int) and eq.saturations == oq.saturations
          and np.array_equal(np.array(eq.err_trace), np.array(oq.err_trace)))
    key = f"aeq/{kind}/{fwd}/{dist}/{mode}"
    stats[key] = stats.get(key, 0) + 1
    if not ok:
        raise AssertionError(f"AEQ mismatch: {key} n_blocks={n_blocks} sig={sig} ts={ts} scale={scale}")


def cdc_case(rng, stats):
    import dataclasses
    n_taps = int(rng.choice([1, 5, 16, 32, 33]))
    cfg = dataclasses.replace(P.LinkConfig(z_km=75.0).cdc_config("fnt"), n_taps=n_taps)
    taps = (rng.normal(size=cfg.n_taps) + 1j * rng.normal(size=cfg.n_taps))
    taps /= np.linalg.norm(taps)
    try:
        eng = P.FntCdcEngine(cfg, P.QuantSpec(5, 8.94427190999916), taps=taps)
    except P.BudgetError:
        stats["cdc/budget"] = stats.get("cdc/budget", 0) + 1
        return
    L = int(rng.choice([0, 1, 31, 32, 33, 4095, 4097, 100003]))
    wide = rng.random() < 0.3
    lim = 1000 if wide else 16
    xr = rng.integers(-lim, lim, L)
    xi = rng.integers(-lim, lim, L)
    try:
        yr, yi = eng.process_int(xr, xi)
    except ValueError:
        stats["cdc/range"] = stats.get("cdc/range", 0) + 1  # beyond the encodable bound
        return
    orr, ori = O.cdc_direct(eng.tap_re, eng.tap_im, xr, xi)
    key = f"cdc/{'wide' if wide else 'narrow'}"
    stats[key] = stats.get(key, 0) + 1
    # the oracle reduces the direct FIR mod F4 and decodes, as the reference's residue
    # arithmetic does even when wide inputs exceed the Eq. (5) budget
    if not (np.array_equal(yr, orr) and np.array_equal(yi, ori)):
        raise AssertionError(f"CDC mismatch: n_taps={n_taps} L={L} wide={wide}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240.0)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    stats: dict[str, int] = {}
    t0 = time.time()
    n = 0
    while time.time() - t0 < a.seconds:
        (aeq_case if rng.random() < 0.7 else cdc_case)(rng, stats)
        n += 1
    print(f"{n} cases, all bit-exact")
    for k in sorted(stats):
        print(f"  {k:40s} {stats[k]}")


if __name__ == "__main__":
    main()
