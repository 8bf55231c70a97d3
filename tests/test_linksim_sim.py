"""The host link simulator behind `sweep` (linksim.generate_tx / apply_channel and
the front end's float conditioning) reproduces the reference's samples bit for bit:
compared with oracle/linkgen_np, the pinned restatement of linksim.py:105-291 (its
quantized outputs match digests the unmodified reference wrote)."""

import numpy as np

import oracle.linkgen_np as G
from paper_2405_04253_b200 import linksim as LS


def _pair(seed_seq, **kw):
    cfg = LS.LinkConfig(n_symbols=4096, z_km=kw.get("z", 20.0), pol_rotation_deg=kw.get("rot", 45.0),
                        dgd_symbols=kw.get("dgd", 0.2), iq_skew_samples=kw.get("skew", 0.1), seed=9)
    link = G.Link(4096, kw.get("z", 20.0), 9, snr_db=kw.get("snr", 17.0), rotation_deg=kw.get("rot", 45.0),
                  dgd=kw.get("dgd", 0.2), skew=kw.get("skew", 0.1))
    r1 = np.random.default_rng(np.random.SeedSequence(seed_seq))
    r2 = np.random.default_rng(np.random.SeedSequence(seed_seq))
    tx = LS.generate_tx(cfg, r1)
    rx, _ = LS.apply_channel(tx.wave, cfg, kw.get("snr", 17.0), r1)
    bits, sym, wave = G.transmit(link, r2)
    rx2 = G.channel(wave, link, r2)
    return cfg, link, tx, rx, (bits, sym, wave), rx2


def test_tx_channel_frontend_bit_identical_to_reference_model():
    for kw in ({}, {"dgd": 0.0, "skew": 0.0, "rot": 0.0}, {"z": 0.0, "snr": 30.0}):
        cfg, link, tx, rx, (bits, sym, wave), rx2 = _pair([9, 17000], **kw)
        assert np.array_equal(tx.bits, bits) and np.array_equal(tx.symbols, sym)
        assert np.array_equal(tx.wave, wave)
        assert np.array_equal(rx, rx2), kw
        from paper_2405_04253_b200.linkgen import rrc_taps
        mf = rrc_taps(cfg.sps, cfg.rrc_span, cfg.rrc_rolloff)
        ours = [LS._unit_power(LS._circular(LS._gram_schmidt(rx[p]), mf)) for p in range(2)]
        ref = G.conditioned(rx2, link)
        for a, b in zip(ours, ref):
            assert np.array_equal(a, b), kw
