"""The pipelined host-buffer chain (stream.HostChain: chunked upload, CDC range
shards, AEQ time segments, segment-wise copy-out over three CUDA streams) returns
exactly what the device-resident chain computes, call after call."""

import numpy as np
import pytest

import paper_2405_04253_b200 as P

pytestmark = pytest.mark.gpu


def test_host_chain_pipelined_equals_resident_chain():
    import torch
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.stream import CdcAeqChain, HostChain
    n_links, n_sym = 6, 1 << 14
    L = 2 * n_sym
    cfg = P.LinkConfig(n_symbols=n_sym, z_km=75.0, seed=4)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    gen = DeviceLinkGenerator(n_sym)
    ref = CdcAeqChain(eng, cfg.aeq_config(), n_links, L, cfg.sig_spec(), cfg.mu_schedule())
    hc = HostChain(eng, cfg.aeq_config(), n_links, L, cfg.sig_spec(), cfg.mu_schedule(),
                   in_chunks=5, aeq_segments=7)
    outs = []
    for seed in (11, 12, 13):   # consecutive calls overlap on the device
        xr, xi = gen.generate(n_links, seed=seed)
        hr = torch.empty(xr.shape, dtype=torch.int8, pin_memory=True)
        hi = torch.empty(xi.shape, dtype=torch.int8, pin_memory=True)
        hr.copy_(xr)
        hi.copy_(xi)
        torch.cuda.synchronize()
        y, err = hc(hr, hi)
        hc.join()
        torch.cuda.synchronize()
        outs.append((y.numpy().copy(), err.numpy().copy()))
        ref.run(xr, xi)
        torch.cuda.synchronize()
        assert np.array_equal(outs[-1][0], ref.y.cpu().numpy())
        assert np.array_equal(outs[-1][1], ref.err.cpu().numpy())
    # back-to-back calls without a host sync in between give the same results
    xs = []
    for seed in (11, 12, 13):
        xr, xi = gen.generate(n_links, seed=seed)
        hr = torch.empty(xr.shape, dtype=torch.int8, pin_memory=True)
        hi = torch.empty(xi.shape, dtype=torch.int8, pin_memory=True)
        hr.copy_(xr)
        hi.copy_(xi)
        xs.append((hr, hi))
    torch.cuda.synchronize()
    hc(*xs[0])
    hc(*xs[1])
    y, err = hc(*xs[2])
    hc.join()
    torch.cuda.synchronize()
    assert np.array_equal(y.numpy(), outs[2][0]) and np.array_equal(err.numpy(), outs[2][1])


def test_host_cdc_pipelined_equals_process_int(golden):
    """HostCdc (pieces + range shards + 2-D copy-out) == one full-length CDC launch."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank, HostCdc
    cfg = P.LinkConfig(n_symbols=1 << 15, z_km=75.0, seed=3)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    rng = np.random.default_rng(5)
    L = 100_000 + 37
    x = [rng.integers(-15, 16, size=(2, L)).astype(np.int8) for _ in range(2)]
    hc = HostCdc(eng, 2, L, pieces=6)
    bank = CdcBank(eng)
    for _ in range(2):
        hr = torch.from_numpy(x[0]).pin_memory()
        hi = torch.from_numpy(x[1]).pin_memory()
        yr, yi = hc(hr, hi)
        hc.join()
        torch.cuda.synchronize()
        dr = torch.from_numpy(x[0]).cuda()
        di = torch.from_numpy(x[1]).cuda()
        rr = torch.empty((2, L), dtype=torch.int16, device="cuda")
        ri = torch.empty_like(rr)
        bank.run(dr, di, length=L, yr=rr, yi=ri)
        assert np.array_equal(yr.numpy(), rr.cpu().numpy())
        assert np.array_equal(yi.numpy(), ri.cpu().numpy())
        x = [x[1], x[0]]


def test_pipelined_chain_equals_resident_chain():
    """stream.PipelinedChain (batch k + 1's CDC overlapping batch k's AEQ, two buffer
    sets) gives, for back-to-back calls, exactly the one-shot chain's outputs."""
    import torch
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.stream import CdcAeqChain, PipelinedChain
    n_links, n_sym = 9, 1 << 13
    L = 2 * n_sym
    cfg = P.LinkConfig(n_symbols=n_sym, z_km=75.0, seed=4)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    gen = DeviceLinkGenerator(n_sym)
    ref = CdcAeqChain(eng, cfg.aeq_config(), n_links, L, cfg.sig_spec(), cfg.mu_schedule())
    pc = PipelinedChain(eng, cfg.aeq_config(), n_links, L, cfg.sig_spec(), cfg.mu_schedule())
    batches = [gen.generate(n_links, seed=s) for s in (21, 22, 23, 24)]
    for upto in (1, 2, 4):
        for xr, xi in batches[:upto]:
            pc(xr, xi)
        pc.join()
        torch.cuda.synchronize()
        ref.run(*batches[upto - 1])
        torch.cuda.synchronize()
        assert torch.equal(pc.y, ref.y) and torch.equal(pc.err, ref.err), upto
        assert torch.equal(pc.phase, ref.phase), upto


def _dropin_link(eng, cfg, fe):
    """One link through the reference-facing API on numpy arrays (bench.run_dropin)."""
    from paper_2405_04253_b200.stream import reference_phase
    streams = [eng.process(a, b) for a, b in fe]
    ph = reference_phase(streams)
    dec = [s[ph::2] for s in streams]
    q = np.stack([P.quantize_real(v, cfg.sig_spec())[0]
                  for v in (dec[0].real, dec[0].imag, dec[1].real, dec[1].imag)])
    eq = P.FntAeq(cfg.aeq_config())
    y = eq.process(q, adapt=True, mu_schedule=cfg.mu_schedule())
    return y, np.array(eq.err_trace), eq.w


def test_dropin_api_threads_equal_sequential():
    """Engines used from several host threads (one per thread, the reference's
    convention) run on per-thread CUDA streams concurrently and return exactly the
    single-thread results; an engine built in one thread and used in another is
    ordered too."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    n_links, n_sym = 8, 1 << 12
    cfg = P.LinkConfig(n_symbols=n_sym, z_km=75.0, seed=4)
    gen = DeviceLinkGenerator(n_sym)
    xr, xi = gen.generate(n_links, seed=21)
    data = [[(xr[2 * l + p].cpu().numpy().astype(np.int64), xi[2 * l + p].cpu().numpy().astype(np.int64))
             for p in range(2)] for l in range(n_links)]
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    seq = [_dropin_link(eng, cfg, fe) for fe in data]

    def worker(fe):
        e = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
        return _dropin_link(e, cfg, fe)

    for _ in range(2):
        with ThreadPoolExecutor(max_workers=n_links) as ex:
            par = list(ex.map(worker, data))
        for (y0, e0, w0), (y1, e1, w1) in zip(seq, par):
            assert np.array_equal(y0, y1) and np.array_equal(e0, e1) and np.array_equal(w0, w1)
    # handoff: build the AEQ engine in one thread, run it in another
    fe = data[0]
    streams = [eng.process(a, b) for a, b in fe]
    from paper_2405_04253_b200.stream import reference_phase
    ph = reference_phase(streams)
    dec = [s[ph::2] for s in streams]
    q = np.stack([P.quantize_real(v, cfg.sig_spec())[0]
                  for v in (dec[0].real, dec[0].imag, dec[1].real, dec[1].imag)])
    with ThreadPoolExecutor(max_workers=1) as ex:
        eq = ex.submit(P.FntAeq, cfg.aeq_config()).result()
    with ThreadPoolExecutor(max_workers=1) as ex:
        y = ex.submit(eq.process, q, True, cfg.mu_schedule()).result()
    assert np.array_equal(y, seq[0][0]) and np.array_equal(eq.w, seq[0][2])


def test_pinned_staging_multi_chunk_copies():
    """Drop-in arrays larger than one pinned staging chunk (16 MB) cross host <-> device
    in several double-buffered pieces (_lib.to_device / to_host): int64 in, int64 and
    complex128 out, against the CPU oracle and the single-piece path."""
    import oracle as O
    from paper_2405_04253_b200 import _lib
    rng = np.random.default_rng(33)
    p = P.default_plans()["cdc64"]
    x = rng.integers(-(1 << 40), 1 << 40, (40000, 64))          # 20.5 MB int64: 2 chunks
    assert np.array_equal(P.fnt(p, x), O.fnt(O.Plan.named("cdc64"), x))
    cfg = P.LinkConfig(z_km=75.0)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    L = (5 << 20) + 77                                          # 84 MB complex128 out: 6 chunks
    xr = rng.integers(-15, 16, L)
    xi = rng.integers(-15, 16, L)
    y = eng.process(xr, xi)
    yr, yi = eng.process_int(xr, xi)
    orr, ori = O.cdc_direct(eng.tap_re, eng.tap_im, xr, xi)
    assert np.array_equal(yr, orr) and np.array_equal(yi, ori)
    inv = 1.0 / eng.output_scale
    assert np.array_equal(y, yr * inv + 1j * (yi * inv))
    # the round trip of an odd-sized buffer through the staging chunks is the identity,
    # with the (optional) staged host-to-device path as well
    a = rng.integers(-(1 << 62), 1 << 62, (1 << 22) + 3)
    assert np.array_equal(_lib.to_host(_lib.to_device(a)), a)
    prev = _lib._STAGED_H2D
    _lib._STAGED_H2D = True
    try:
        assert np.array_equal(_lib.to_host(_lib.to_device(a)), a)
        assert np.array_equal(P.fnt(p, x), O.fnt(O.Plan.named("cdc64"), x))
    finally:
        _lib._STAGED_H2D = prev
