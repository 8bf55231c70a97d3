"""On-device metrology (paper_2405_04253_b200.metrology) vs the reference's
BER / EVM on BASELINE config 3 (reference digests), and vs the pinned numpy
port on config-5 links. BER must be identical; EVM within 1e-9 relative (the
bar for float post-dequantization metrics is 1e-6)."""

import json

import numpy as np
import pytest

import oracle.linkgen_np as G
import paper_2405_04253_b200 as P
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _gpu_chain(cfg, fe):
    import torch
    from paper_2405_04253_b200.stream import CdcAeqChain
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    L = fe[0][0].size
    xr = torch.from_numpy(np.stack([fe[0][0], fe[1][0]]).astype(np.int8)).cuda()
    xi = torch.from_numpy(np.stack([fe[0][1], fe[1][1]]).astype(np.int8)).cuda()
    ch = CdcAeqChain(eng, cfg.aeq_config(), 1, L, cfg.sig_spec(), cfg.mu_schedule())
    ch.run(xr, xi)
    return ch


@pytest.mark.parametrize("snr", [16.0, 24.0])
def test_metrology_config3_vs_reference(snr):
    from paper_2405_04253_b200 import metrology as M
    d = json.loads((GOLDEN / "digests.json").read_text())["c3"][str(snr)]
    L, bits, sym, fe = G.config3(snr)
    cfg = P.LinkConfig(n_symbols=2 ** 20, z_km=75.0, snr_db=(snr,), pol_rotation_deg=0.0,
                       dgd_symbols=0.0, iq_skew_samples=0.0, seed=2)
    ch = _gpu_chain(cfg, fe)
    s, b = M.numpy_reference_inputs(bits, sym)
    ber, evm, ok = M.align_and_count(M.aeq_to_pols(ch.y), s, b, cfg.discard_symbols)
    assert bool(ok[0]) == d["ok"]
    assert ber[0] == d["ber"]
    assert abs(evm[0] - d["evm_db"]) <= 1e-9 * abs(d["evm_db"])


def test_metrology_batched_links_vs_numpy_port():
    """Two config-5 links scored in one batch agree with the numpy metrology."""
    import torch
    from paper_2405_04253_b200 import metrology as M
    ys, syms, bitss, ref = [], [], [], []
    for link in (7, 11):
        L, bits, sym, fe = G.config5(link, n_symbols=2 ** 16)
        cfg = P.LinkConfig(n_symbols=2 ** 16, z_km=75.0, pol_rotation_deg=0.0, dgd_symbols=0.0,
                           iq_skew_samples=0.0, seed=4, discard_symbols=2000)
        ch = _gpu_chain(cfg, fe)
        y = ch.y[0].cpu().numpy()
        ref.append(G.ber_evm(np.stack([y[0] + 1j * y[1], y[2] + 1j * y[3]]), bits, sym, 2000))
        ys.append(ch.y[0])
        syms.append(torch.from_numpy(sym).cuda())
        bitss.append(torch.from_numpy(bits.astype(np.int8)).cuda())
    ber, evm, ok = M.align_and_count(M.aeq_to_pols(torch.stack(ys)), torch.stack(syms),
                                     torch.stack(bitss), 2000)
    for i, (rb, re, rok) in enumerate(ref):
        assert bool(ok[i]) == rok and ber[i] == rb
        if rok:
            assert abs(evm[i] - re) <= 1e-9 * abs(re)
