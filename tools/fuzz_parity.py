#!/usr/bin/env python3
"""Randomized differential check of the drop-in API against the CPU oracle (run on
the GPU box): FntAeq with random initial taps (float and 14-bit, set independently
as the reference allows), random inputs (5-bit, full int8, wide int32 up to the
encodable +-32768), random step sizes (0, tiny, large enough to saturate), random
lengths, through both stream layouts and both forward forms; FntCdcEngine with random
6-bit taps and random stream lengths / input widths; the multi-stream CdcBank on random
output ranges and input windows (int8 / int32 / float64 quantized on load); the whole
device chain; fnt / ifnt / convolutions on random plans of every prime Fermat modulus;
the pipelined host-buffer HostCdc / HostChain with random piece and segment counts.
Every case must be bit-exact (y, w, w_int, saturations, err_trace; CDC outputs).

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


def cdc_bank_case(rng, stats):
    """CdcBank.run (the device-resident multi-stream path) on random output ranges of
    random-length streams, fed a window with the overlap-save halo, int8 / int32 /
    float64 inputs (float64 quantized on load, persistent kernel) and int16 / int32
    outputs, against the oracle's direct FIR of the quantized samples."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    cfg = P.LinkConfig(z_km=75.0)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    bank = CdcBank(eng)
    S = int(rng.integers(1, 4))
    L = int(rng.choice([1, 33, 4096, 4097, 70001, 300007]))
    a = int(rng.integers(0, L))
    b = int(rng.integers(a + 1, L + 1))
    c = eng.config.n_taps // 2
    x_lo = max(0, (a + c) // 32 * 32 - 32 - int(rng.integers(0, 3)))
    x_hi = min(L, ((b - 1 + c) // 32) * 32 + 32 + int(rng.integers(0, 3)))
    kind = rng.choice(["i8", "i32", "f64"])
    q = rng.integers(-15, 16, (2, S, L))
    if kind == "f64":
        spec = eng.sig_spec
        xf = (q + (rng.random((2, S, L)) - 0.5) * 0.9) / spec.scale
        xf[rng.random((2, S, L)) < 0.001] = 9.0  # clipped samples
        qq = np.stack([[O.quantize_real(xf[p, s], spec.scale, spec.max_int)[0] for s in range(S)]
                       for p in range(2)])
        xr = torch.from_numpy(np.ascontiguousarray(xf[0][:, x_lo:x_hi])).cuda()
        xi = torch.from_numpy(np.ascontiguousarray(xf[1][:, x_lo:x_hi])).cuda()
        extra = dict(in_spec=spec, in_clipped=torch.zeros(1, dtype=torch.int64, device="cuda"))
    else:
        qq = q
        dt = torch.int8 if kind == "i8" else torch.int32
        xr = torch.from_numpy(np.ascontiguousarray(q[0][:, x_lo:x_hi])).to("cuda", dt)
        xi = torch.from_numpy(np.ascontiguousarray(q[1][:, x_lo:x_hi])).to("cuda", dt)
        extra = {}
    odt = torch.int16 if rng.random() < 0.5 else torch.int32
    yr = torch.empty((S, b - a), dtype=odt, device="cuda")
    yi = torch.empty_like(yr)
    bank.run(xr, xi, length=L, x_first=x_lo, out_first=a, out_count=b - a, yr=yr, yi=yi, **extra)
    torch.cuda.synchronize()
    for s in range(S):
        orr, ori = O.cdc_direct(eng.tap_re, eng.tap_im, qq[0, s], qq[1, s])
        if not (np.array_equal(yr[s].cpu().numpy().astype(np.int64), orr[a:b])
                and np.array_equal(yi[s].cpu().numpy().astype(np.int64), ori[a:b])):
            raise AssertionError(f"CdcBank mismatch: kind={kind} S={S} L={L} range=[{a},{b}) "
                                 f"window=[{x_lo},{x_hi})")
    key = f"cdcbank/{kind}"
    stats[key] = stats.get(key, 0) + 1


def chain_case(rng, stats):
    """The whole device-resident receiver chain (CdcAeqChain: CDC with the fused
    requantization and decimation statistics, phase decision with the tie guard,
    FNT-AEQ over both layouts) on random links of the device link model with random
    lengths and gear-shift points, against the oracle's chain per link."""
    import torch
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.stream import CdcAeqChain
    n_links = int(rng.integers(1, 6))
    n_sym = int(rng.choice([80, 300, 1024, 4096]))
    cfg = P.LinkConfig(n_symbols=n_sym, z_km=75.0, seed=4)
    cfg.gear_symbols = int(rng.integers(0, 2 * n_sym))
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    xr, xi = DeviceLinkGenerator(n_sym).generate(n_links, seed=int(rng.integers(1, 1 << 30)))
    L = 2 * n_sym  # the chain takes 2-sps streams of even length
    kind = rng.choice(["warp", "pol"])
    prev = A.set_aeq_kernel(kind)
    try:
        ch = CdcAeqChain(eng, cfg.aeq_config(), n_links, L, cfg.sig_spec(), cfg.mu_schedule())
    finally:
        A.set_aeq_kernel(prev)
    ch.run(xr, xi)
    torch.cuda.synchronize()
    for l in range(n_links):
        fe = [(xr[2 * l + p].cpu().numpy().astype(np.int64), xi[2 * l + p].cpu().numpy().astype(np.int64))
              for p in range(2)]
        ph, y, oq = O.chain_link(eng.tap_re, eng.tap_im, eng.output_scale, cfg.sig_scale, fe,
                                 cfg.mu1, cfg.mu2, cfg.gear_symbols)
        nb = y.shape[1] // 16
        ok = (int(ch.phase[l].item()) == ph and np.array_equal(ch.y[l].cpu().numpy()[:, :16 * nb], y)
              and np.array_equal(ch.err[l].cpu().numpy()[:nb], np.array(oq.err_trace)))
        if not ok:
            raise AssertionError(f"chain mismatch: link {l} of {n_links}, n_sym={n_sym}, L={L}, {kind}")
    key = f"chain/{kind}"
    stats[key] = stats.get(key, 0) + 1


def transform_case(rng, stats):
    """fnt / ifnt / cyclic_convolve_real / _complex on a random valid plan (any prime
    Fermat modulus F1..F4, any power-of-two length the modulus supports up to 256, a
    random root of exactly that order: the shift-add kernels for the two shipped
    plans, the table-driven ones otherwise) and random batch shapes, residues and
    out-of-range int64 inputs, against the oracle's C restatement."""
    t = int(rng.integers(1, 5))
    F = (1 << (1 << t)) + 1
    n = 1 << int(rng.integers(1, min(1 << t, 8) + 1))
    while True:
        alpha = pow(int(rng.integers(2, F)), (F - 1) // n, F)
        if pow(alpha, n // 2, F) == F - 1:
            break
    if rng.random() < 0.3:  # the shipped shift-add plans
        (t, n, alpha), F = (rng.choice([(4, 32, 2), (4, 64, 4080)]).tolist()), 65537
    plan = P.make_plan(P.FermatParams(t), alpha, n)
    op = O.Plan(t, n, alpha)
    shape = tuple(int(v) for v in rng.integers(1, 40, int(rng.integers(1, 3)))) + (n,)
    wide = rng.random() < 0.3
    x = rng.integers(-(1 << 40), 1 << 40, shape) if wide else rng.integers(0, F, shape)
    ok = np.array_equal(P.fnt(plan, x), O.fnt(op, x)) and np.array_equal(P.ifnt(plan, x), O.ifnt(op, x))
    xr, xi, yr, yi = (rng.integers(0, F, shape) for _ in range(4))
    ok = ok and np.array_equal(P.cyclic_convolve_real(plan, xr, yr), O.cyclic_real(op, xr, yr))
    y1 = yr.reshape(-1, n)[0]
    ok = ok and np.array_equal(P.cyclic_convolve_real(plan, xr, y1), O.cyclic_real(op, xr, y1))
    zr, zi = P.cyclic_convolve_complex(plan, xr, xi, yr, yi)
    orr, ori = O.cyclic_complex(op, xr, xi, yr, yi)
    ok = ok and np.array_equal(zr, orr) and np.array_equal(zi, ori)
    key = f"transform/F{t}/n{n}"
    stats[key] = stats.get(key, 0) + 1
    if not ok:
        raise AssertionError(f"transform mismatch: t={t} n={n} alpha={alpha} shape={shape} wide={wide}")


def host_case(rng, stats):
    """The pipelined host-buffer APIs with random piece / segment counts: HostCdc (pinned
    int8 in, int16 out) against one device-resident CDC launch, and HostChain against the
    device-resident CdcAeqChain (outputs and err_trace), call after call."""
    import torch
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.stream import CdcAeqChain, CdcBank, HostCdc, HostChain
    cfg = P.LinkConfig(z_km=75.0)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    if rng.random() < 0.5:
        S = int(rng.integers(1, 4))
        L = int(rng.integers(64, 200_000))
        x = rng.integers(-15, 16, size=(2, S, L)).astype(np.int8)
        hc = HostCdc(eng, S, L, pieces=int(rng.integers(1, 12)))
        yr, yi = hc(torch.from_numpy(x[0]).pin_memory(), torch.from_numpy(x[1]).pin_memory())
        hc.join()
        torch.cuda.synchronize()
        rr = torch.empty((S, L), dtype=torch.int16, device="cuda")
        ri = torch.empty_like(rr)
        CdcBank(eng).run(torch.from_numpy(x[0]).cuda(), torch.from_numpy(x[1]).cuda(), length=L,
                         yr=rr, yi=ri)
        ok = np.array_equal(yr.numpy(), rr.cpu().numpy()) and np.array_equal(yi.numpy(), ri.cpu().numpy())
        key = "host/cdc"
    else:
        n_links = int(rng.integers(1, 5))
        n_sym = int(rng.choice([512, 2048, 8192]))
        L = 2 * n_sym
        xr, xi = DeviceLinkGenerator(n_sym).generate(n_links, seed=int(rng.integers(1, 1 << 30)))
        ref = CdcAeqChain(eng, cfg.aeq_config(), n_links, L, cfg.sig_spec(), cfg.mu_schedule())
        hch = HostChain(eng, cfg.aeq_config(), n_links, L, cfg.sig_spec(), cfg.mu_schedule(),
                        in_chunks=int(rng.integers(1, 8)), aeq_segments=int(rng.integers(1, 12)))
        hr = torch.empty(xr.shape, dtype=torch.int8, pin_memory=True)
        hi = torch.empty(xi.shape, dtype=torch.int8, pin_memory=True)
        hr.copy_(xr)
        hi.copy_(xi)
        torch.cuda.synchronize()
        y, err = hch(hr, hi)
        hch.join()
        ref.run(xr, xi)
        torch.cuda.synchronize()
        ok = np.array_equal(y.numpy(), ref.y.cpu().numpy()) and np.array_equal(err.numpy(), ref.err.cpu().numpy())
        key = "host/chain"
    stats[key] = stats.get(key, 0) + 1
    if not ok:
        raise AssertionError(f"{key} mismatch")


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
        u = rng.random()
        (aeq_case if u < 0.5 else cdc_case if u < 0.62 else cdc_bank_case if u < 0.74
         else chain_case if u < 0.84 else transform_case if u < 0.94 else host_case)(rng, stats)
        n += 1
    print(f"{n} cases, all bit-exact")
    for k in sorted(stats):
        print(f"  {k:40s} {stats[k]}")


if __name__ == "__main__":
    main()
