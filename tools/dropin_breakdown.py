#!/usr/bin/env python3
"""Per-phase host wall time of one link through the reference-facing drop-in API
(FntCdcEngine.process x 2, the decimation phase, quantize_real x 4, FntAeq.process),
run on the GPU box: python tools/dropin_breakdown.py"""
import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2405_04253_b200 as P
from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
from paper_2405_04253_b200.stream import reference_phase
n_sym = 1 << 18
cfg = P.LinkConfig(n_symbols=n_sym, z_km=75.0, seed=4)
gen = DeviceLinkGenerator(n_sym)
xr, xi = gen.generate(4, seed=5)
data = [[(xr[2 * l + p].cpu().numpy().astype(np.int64), xi[2 * l + p].cpu().numpy().astype(np.int64)) for p in range(2)] for l in range(4)]
eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
spec = cfg.sig_spec()
T = {}
def tic(k, t0):
    T[k] = T.get(k, 0) + time.perf_counter() - t0
    return time.perf_counter()
for it, fe in enumerate(data):
    if it == 1: T.clear()
    t = time.perf_counter()
    streams = [eng.process(a, b) for a, b in fe]; t = tic('cdc.process x2', t)
    ph = reference_phase(streams); t = tic('reference_phase (numpy)', t)
    dec = [s[ph::2] for s in streams]
    parts = (dec[0].real, dec[0].imag, dec[1].real, dec[1].imag)
    q = np.stack([P.quantize_real(v, spec)[0] for v in parts]); t = tic('quantize_real x4', t)
    eq = P.FntAeq(cfg.aeq_config()); t = tic('FntAeq()', t)
    from paper_2405_04253_b200.aeq import mu_block_array
    mb = mu_block_array(q.shape[1] // 16, 16, cfg.mu_schedule(), cfg.aeq_config().mu); t = tic('mu_block_array', t)
    y = eq.process(q, adapt=True, mu_schedule=cfg.mu_schedule()); t = tic('FntAeq.process (incl mu)', t)
for k, v in T.items():
    print(f"{k:28s} {1e3 * v / 3:8.2f} ms/link")
print("total", 1e3 * sum(T.values()) / 3)
