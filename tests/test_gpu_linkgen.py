"""On-device link generator (bench data).

* Shard invariance: link i depends only on (seed, i) -- a shard generated alone
  equals the same rows of an unsharded run (config 5 strong scaling), and a
  config-4 window equals the same samples of any other window covering them.
* Statistical equivalence with the reference generator: the device model's
  quantized front-end samples against oracle/linkgen_np (the reference's link model
  restated bit-exactly, pinned to reference digests): level histograms and the
  average power spectrum, for the config-5 channel (Haar Jones) and for the
  reference's default channel with DGD and IQ skew (linksim.py:211-234)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_SYM = 1 << 13


def _gen(**kw):
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    import paper_2405_04253_b200 as P
    cfg = P.LinkConfig(n_symbols=N_SYM)
    return DeviceLinkGenerator(N_SYM, z_km=75.0, sig_scale=cfg.sig_scale, **kw)


def test_link_shards_identical_at_any_split():
    import torch
    g = _gen()
    xr, xi = g.generate(96, seed=4)
    for first, n in ((32, 32), (64, 32), (27, 10), (0, 5), (90, 6)):
        sr, si = g.generate(n, seed=4, first_link=first)
        assert torch.equal(sr, xr[2 * first:2 * (first + n)])
        assert torch.equal(si, xi[2 * first:2 * (first + n)])


def test_config4_windows_identical_at_any_split():
    import torch
    from bench import c4_window
    import paper_2405_04253_b200 as P
    sig = P.LinkConfig().sig_scale
    seg = 1 << 14
    fr, fi = c4_window(0, 40 * seg, sig, seg=seg)
    for a, n in ((3 * seg - 48, 5 * seg + 96), (17 * seg + 5, 9 * seg), (0, 7)):
        wr, wi = c4_window(a, n, sig, seg=seg)
        assert torch.equal(wr, fr[:, a:a + n]) and torch.equal(wi, fi[:, a:a + n])


def _hist(planes):
    h = np.zeros(31)
    for a in planes:
        v, c = np.unique(np.asarray(a).astype(np.int64), return_counts=True)
        h[v + 15] += c
    return h / h.sum()


def _psd(planes, bins=64):
    acc = np.zeros(bins)
    for a in planes:
        x = np.asarray(a, dtype=float).reshape(-1, bins)
        acc += (np.abs(np.fft.fft(x, axis=1)) ** 2).mean(axis=0)
    return acc / acc.sum()


def _compare(dev_planes, ref_planes):
    hd, hr = _hist(dev_planes), _hist(ref_planes)
    tv = 0.5 * np.abs(hd - hr).sum()
    pd, pr = _psd(dev_planes), _psd(ref_planes)
    spec = np.abs(pd - pr).max() / pr.max()
    return tv, spec


def test_statistics_match_reference_generator_config5():
    import oracle.linkgen_np as G
    n = 8
    xr, xi = _gen().generate(n, seed=4)
    dev = [t for t in xr.cpu().numpy()] + [t for t in xi.cpu().numpy()]
    ref = []
    for i in range(n):
        _, _, _, fe = G.config5(i, n_symbols=N_SYM)
        ref += [fe[0][0], fe[1][0], fe[0][1], fe[1][1]]
    tv, spec = _compare(dev, ref)
    print(f"config-5 channel: level-histogram TV {tv:.4f}, max spectral deviation {spec:.4f}")
    assert tv < 0.03 and spec < 0.15


def test_statistics_match_reference_generator_dgd_skew():
    """The reference's default channel (linksim.LinkConfig: DGD 0.2 symbol, IQ skew
    0.1 sample) against the device model with the same DGD and skew."""
    import oracle.linkgen_np as G
    n = 8
    xr, xi = _gen(dgd_symbols=0.2, iq_skew_samples=0.1).generate(n, seed=7, snr_db=(20.0, 20.0))
    dev = [t for t in xr.cpu().numpy()] + [t for t in xi.cpu().numpy()]
    ref = []
    for i in range(n):
        L = G.Link(N_SYM, 75.0, 7, snr_db=20.0, rotation_deg=45.0, dgd=0.2, skew=0.1)
        rng = np.random.default_rng(np.random.SeedSequence([7, i]))
        _, _, wave = G.transmit(L, rng)
        fe = G.front_end(G.channel(wave, L, rng), L)
        ref += [fe[0][0], fe[1][0], fe[0][1], fe[1][1]]
    tv, spec = _compare(dev, ref)
    print(f"DGD + IQ-skew channel: level-histogram TV {tv:.4f}, max spectral deviation {spec:.4f}")
    assert tv < 0.03 and spec < 0.15
