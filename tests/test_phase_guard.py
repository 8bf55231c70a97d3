"""Decimation-phase tie guard (linksim.py:249-260).

The device decides the sampling phase from exact integer statistics of the CDC
outputs; the reference evaluates float64 means. The two can only disagree when the
two phase metrics are within float rounding of each other; such links (and NaN
metrics of an all-zero link) are re-decided with the reference's own float64
expression (stream.resolve_phase_ties). These tests exercise that path."""

import numpy as np
import pytest

import oracle as O
import paper_2405_04253_b200 as P
from paper_2405_04253_b200 import stream as ST


def _link_b_cfg():
    return P.LinkConfig(n_symbols=2 ** 14, z_km=75.0, snr_db=(18.0,), pol_rotation_deg=45.0,
                        dgd_symbols=0.0, iq_skew_samples=0.0, seed=6)


def test_reference_phase_expression_on_golden_link(golden):
    """The host-side evaluation reproduces the reference's decision (fixture b) from
    the CDC outputs (oracle restatement of process_int, CPU)."""
    g = golden("aeq")
    cfg = _link_b_cfg()
    import math
    from paper_2405_04253_b200.cdc import design_cd_taps
    c = cfg.cdc_config("fnt")
    taps = design_cd_taps(c)  # host tap design (cdc.py:61-86); quantized by the CPU oracle
    max_int = (1 << (c.tap_bits - 1)) - 1
    scale = 2.0 ** math.floor(math.log2(max_int / max(np.abs(taps.real).max(), np.abs(taps.imag).max())))
    tr, _ = O.quantize_real(taps.real, scale, max_int)
    ti, _ = O.quantize_real(taps.imag, scale, max_int)
    inv = 1.0 / (cfg.sig_scale * scale)
    streams = []
    for p in range(2):
        yr, yi = O.cdc_process_int(tr, ti, g["b_cdc_q"][p, 0], g["b_cdc_q"][p, 1])
        streams.append(yr * inv + 1j * (yi * inv))
    assert ST.reference_phase(streams) == int(g["b_phase"])
    # an all-zero link: both metrics are 0/0 = NaN in the reference, which keeps phase 0
    z = np.zeros(64, dtype=np.complex128)
    with np.errstate(invalid="ignore"):
        assert ST.reference_phase([z, z]) == 0


@pytest.mark.gpu
def test_zero_link_tie_and_forced_guard(golden, monkeypatch):
    """A batch [link b, all-zero link, link b]: the zero link's metrics are NaN (a
    tie) and its phase is decided on the host; with the guard forced open every link
    is decided on the host and the phases and AEQ outputs are unchanged."""
    import torch
    from paper_2405_04253_b200.stream import CdcAeqChain
    g = golden("aeq")
    cfg = _link_b_cfg()
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    q = g["b_cdc_q"]
    L = q.shape[-1]
    zero = np.zeros_like(q)
    links = [q, zero, q]
    xr = torch.from_numpy(np.stack([lk[p, 0] for lk in links for p in range(2)]).astype(np.int8)).cuda()
    xi = torch.from_numpy(np.stack([lk[p, 1] for lk in links for p in range(2)]).astype(np.int8)).cuda()
    ch = CdcAeqChain(eng, cfg.aeq_config(), 3, L, cfg.sig_spec(), cfg.mu_schedule())
    ch.run(xr, xi)
    assert ch.resolved == [1]
    ph = ch.phase.cpu().numpy()
    assert list(ph) == [int(g["b_phase"]), 0, int(g["b_phase"])]
    y = ch.y.cpu().numpy()
    assert np.array_equal(y[0], g["b_y"]) and np.array_equal(y[2], g["b_y"])
    oph, oy, _ = O.chain_link(eng.tap_re, eng.tap_im, eng.output_scale, cfg.sig_scale,
                              [(zero[0, 0], zero[0, 1]), (zero[1, 0], zero[1, 1])])
    assert oph == 0 and np.array_equal(y[1], oy)
    monkeypatch.setattr(ST, "PHASE_TIE_GUARD", 2.0)
    ch.run(xr, xi)
    assert ch.resolved == [0, 1, 2]
    assert list(ch.phase.cpu().numpy()) == list(ph)
    assert np.array_equal(ch.y.cpu().numpy(), y)
