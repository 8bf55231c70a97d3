"""Calibrate the CPU baseline port against the unmodified reference (run in the
build container, where /root/reference exists; the GPU box has no reference).

bench.py's CPU baseline and `--impl reference` time oracle/np_port.chain, a numpy
restatement of the reference's CDC -> glue -> AEQ path, because the reference
cannot travel to the GPU box. This script times both on the same config-5 links
(the reference's own link model, oracle/linkgen_np), one process, and checks the
outputs are identical; the ratio goes to profiles/port_calibration_r02.json.

    PYTHONPATH=/root/reference/pkg/src python tools/calibrate_port.py
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(1, "/root/reference/pkg/src")

import fntdsp  # noqa: E402  (the unmodified reference)
from fntdsp import linksim as RL  # noqa: E402
import oracle.linkgen_np as G  # noqa: E402
import oracle.np_port as N  # noqa: E402


def reference_chain(cfg, fe):
    """linksim.py:283-308 + 399-406 on already-quantized front-end samples."""
    eng = fntdsp.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    eqs = [eng.process(xr, xi) for xr, xi in fe]
    ph = RL._decimation_phase(eqs, cfg.sps)
    dec = [e[ph::2] for e in eqs]
    spec = cfg.sig_spec()
    q = np.stack([fntdsp.quantize_real(s, spec)[0]
                  for s in (dec[0].real, dec[0].imag, dec[1].real, dec[1].imag)])
    eq = fntdsp.FntAeq(cfg.aeq_config())
    return eq.process(q, adapt=True, mu_schedule=cfg.mu_schedule())


def main():
    n_sym = 1 << 13
    cfg = RL.LinkConfig(n_symbols=n_sym, z_km=75.0, pol_rotation_deg=0.0, dgd_symbols=0.0,
                        iq_skew_samples=0.0, seed=4)
    eng = fntdsp.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    nb = n_sym // 16
    mu = np.where(np.arange(nb) * 16 < cfg.gear_symbols, cfg.mu1, cfg.mu2)
    rows = []
    for link in range(4):
        _, _, _, fe = G.config5(link, n_symbols=n_sym)
        t0 = time.perf_counter()
        y_ref = reference_chain(cfg, fe)
        t_ref = time.perf_counter() - t0
        xr2 = np.stack([fe[0][0], fe[1][0]])
        xi2 = np.stack([fe[0][1], fe[1][1]])
        t0 = time.perf_counter()
        y_port, _ = N.chain(xr2, xi2, eng.tap_re, eng.tap_im, cfg.n_cdc_taps, eng.output_scale,
                            cfg.sig_scale, mu)
        t_port = time.perf_counter() - t0
        rows.append({"link": link, "reference_s": t_ref, "port_s": t_port,
                     "identical_y": bool(np.array_equal(y_ref, y_port))})
    ratio = sum(r["reference_s"] for r in rows) / sum(r["port_s"] for r in rows)
    out = {"what": "config-5 links of 2^13 symbols (the reference's link model) through the "
                   "unmodified reference (FntCdcEngine.process, linksim._decimation_phase, "
                   "quantize_real, FntAeq.process) and through oracle/np_port.chain, one process",
           "links": rows, "reference_over_port_time": ratio,
           "all_identical": all(r["identical_y"] for r in rows),
           "host": {"cpu_count": os.cpu_count(), "numpy": np.__version__}}
    path = ROOT / "profiles" / "port_calibration_r02.json"
    path.write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
