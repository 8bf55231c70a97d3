#!/usr/bin/env python3
"""Quick GPU check of one CDC kernel against the shift-add kernel and the oracle on
random int8 streams (run under `timeout`): python tools/cdc_kernel_check.py umma"""
import sys

import numpy as np
import torch

import paper_2405_04253_b200 as P
from paper_2405_04253_b200 import cdc as cdc_mod
from paper_2405_04253_b200.stream import CdcBank
from oracle import np_port as N

kern = sys.argv[1] if len(sys.argv) > 1 else "umma"
cfg = P.LinkConfig(z_km=75.0, seed=1)
eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
rng = np.random.default_rng(3)
for S, L, lo, hi in ((1, 4096, -16, 16), (3, 50_003, -128, 128), (5, 1 << 18, -16, 16)):
    xr = rng.integers(lo, hi, (S, L)).astype(np.int8)
    xi = rng.integers(lo, hi, (S, L)).astype(np.int8)
    outs = {}
    for k in ("shift", kern):
        cdc_mod.set_cdc_kernel(k)
        yr = torch.empty((S, L), dtype=torch.int32, device="cuda")
        yi = torch.empty_like(yr)
        CdcBank(eng).run(torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda(), length=L, yr=yr, yi=yi)
        torch.cuda.synchronize()
        outs[k] = (yr.cpu().numpy(), yi.cpu().numpy())
    same = all(np.array_equal(outs["shift"][j], outs[kern][j]) for j in range(2))
    r0, i0 = N.cdc_process_int(xr[0].astype(np.int64), xi[0].astype(np.int64), eng._b_plus, eng._b_minus, 32)
    ora = np.array_equal(outs[kern][0][0], r0) and np.array_equal(outs[kern][1][0], i0)
    bad = np.argwhere(outs["shift"][0] != outs[kern][0])
    print(f"S={S} L={L} range=[{lo},{hi}) {kern}==shift: {same} oracle(stream 0): {ora} "
          f"first mismatches: {bad[:5].tolist()}", flush=True)
