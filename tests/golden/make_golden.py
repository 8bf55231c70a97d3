"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference package `fntdsp` (imported in place from /root/reference/pkg/src).

This script is the only thing in the repo that imports the reference. It runs
in the build container (the reference does not exist on the GPU box); its
outputs are small .npz fixtures plus sha256 digests of full-size outputs.
Re-run with:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Every fixture records which reference function produced it (file:line).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

REF_SRC = os.environ.get("FNTDSP_REF", "/root/reference/pkg/src")
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

import fntdsp  # noqa: E402  (reference, read-only)
from fntdsp import (COUNTER, AeqConfig, CdcConfig, FermatParams,  # noqa: E402
                    FntAeq, FntCdcEngine, LinkConfig, QuantSpec,
                    check_overflow, convolve_signed_complex,
                    convolve_signed_real, cyclic_convolve_complex,
                    cyclic_convolve_real, default_plans, fnt, ifnt,
                    quantize_real, recombine, split_taps)
from fntdsp import linksim  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def save(name: str, **arrays) -> None:
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size} B)")


# --------------------------------------------------------------------------
# transforms (fnt.py:86-114) and plans (fnt.py:60-83, 186-195)

def gen_plans() -> dict:
    plans = default_plans()
    out = {}
    for name, p in plans.items():
        out[name] = {
            "t": p.params.t, "F": p.params.F, "n": p.n, "alpha": p.alpha,
            "alpha_inv": p.alpha_inv, "n_inv": p.n_inv,
            "bitrev": p.bitrev.tolist(),
            "fwd_twiddles": [t.tolist() for t in p.fwd_twiddles],
            "inv_twiddles": [t.tolist() for t in p.inv_twiddles],
        }
    return out


def gen_transforms() -> None:
    plans = default_plans()
    rng = np.random.default_rng(101)
    arrs = {}
    for name, p in plans.items():
        F = p.params.F
        x = rng.integers(0, F, size=(64, p.n))
        arrs[f"{name}_x"] = x
        arrs[f"{name}_fnt"] = fnt(p, x)
        arrs[f"{name}_ifnt"] = ifnt(p, x)
        # arbitrary signed int64 inputs are reduced implicitly (probe t17)
        xs = rng.integers(-(1 << 40), 1 << 40, size=(16, p.n))
        arrs[f"{name}_xs"] = xs
        arrs[f"{name}_fnt_xs"] = fnt(p, xs)
        arrs[f"{name}_ifnt_xs"] = ifnt(p, xs)
        # leading axes broadcast (fnt.py:86-103): a 3-D batch
        x3 = rng.integers(0, F, size=(3, 5, p.n))
        arrs[f"{name}_x3"] = x3
        arrs[f"{name}_fnt3"] = fnt(p, x3)
        # the all-F-1 / all-zero / all-one extremes
        ext = np.stack([np.full(p.n, F - 1), np.zeros(p.n, np.int64),
                        np.ones(p.n, np.int64), np.full(p.n, F // 2)])
        arrs[f"{name}_ext"] = ext
        arrs[f"{name}_fnt_ext"] = fnt(p, ext)
        arrs[f"{name}_ifnt_ext"] = ifnt(p, ext)
    save("transforms", **arrs)


def gen_selftest() -> dict:
    """Known-answer vectors of the reference CLI selftest (cli.py:80-132)."""
    plans = default_plans()
    p17 = plans["mod17"]
    rng = np.random.default_rng(7)
    arrs = {
        "delta_fnt": fnt(p17, np.array([1, 0, 0, 0, 0, 0, 0, 0])),
        "pair_fnt": fnt(p17, np.array([1, 1, 0, 0, 0, 0, 0, 0])),
        "pair_ifnt": ifnt(p17, np.array([2, 3, 5, 9, 0, 16, 14, 10])),
        "conv17": convolve_signed_real(p17, np.array([1, 2, 0, 0, 0, 0, 0, 0]),
                                       np.array([3, 1, 0, 0, 0, 0, 0, 0])),
    }
    for name, plan in plans.items():
        x = rng.integers(0, plan.params.F, size=(50, plan.n))
        arrs[f"rt_{name}_x"] = x
        arrs[f"rt_{name}_y"] = ifnt(plan, fnt(plan, x))
    rep = check_overflow(np.full(32, 31), QuantSpec(5, 8.0), FermatParams(4),
                         complex_mode=True)
    w = rng.integers(-16383, 16384, size=64)
    s = split_taps(w)
    arrs.update(split_w=w, split_hi=s.high, split_lo=s.low,
                split_rec=recombine(s.high, s.low))
    save("selftest", **arrs)
    return {"budget_bound": rep.bound, "budget_passed": bool(rep.passed),
            "sqrt2": int(fntdsp.sqrt2(FermatParams(4)))}


# --------------------------------------------------------------------------
# convolution (fnt.py:117-183); config 1 of BASELINE.json

def gen_convolution() -> dict:
    plans = default_plans()
    p = plans["cdc64"]
    F = p.params.F
    # C1: rng(0); x first, then per-block taps
    rng = np.random.default_rng(0)
    x = rng.integers(-16, 16, (16384, 64))
    h = rng.integers(-32, 32, (16384, 64))
    COUNTER.reset()
    with COUNTER.enabled_ctx():
        z = cyclic_convolve_real(p, x % F, h % F)
        n_mult = COUNTER.total()
    zs = convolve_signed_real(p, x, h)
    digests = {"c1_cyclic_real": sha(z), "c1_signed_real": sha(zs),
               "c1_counter": int(n_mult)}
    arrs = {"c1_z_head": z[:256], "c1_zs_head": zs[:256]}
    rng = np.random.default_rng(202)
    for name in ("cdc64", "aeq32", "mod17"):
        pl = plans[name]
        Fp = pl.params.F
        lim = 16 if Fp > 257 else 2
        xr = rng.integers(-lim, lim, (128, pl.n))
        xi = rng.integers(-lim, lim, (128, pl.n))
        yr = rng.integers(-lim, lim, (128, pl.n))
        yi = rng.integers(-lim, lim, (128, pl.n))
        # residue API with broadcast of a single tap vector (fnt.py:117)
        arrs[f"{name}_xr"], arrs[f"{name}_xi"] = xr, xi
        arrs[f"{name}_yr"], arrs[f"{name}_yi"] = yr, yi
        arrs[f"{name}_real_bcast"] = cyclic_convolve_real(pl, xr % Fp, yr[0] % Fp)
        arrs[f"{name}_real"] = cyclic_convolve_real(pl, xr % Fp, yr % Fp)
        zr, zi = cyclic_convolve_complex(pl, xr % Fp, xi % Fp, yr % Fp, yi % Fp)
        arrs[f"{name}_cplx_re"], arrs[f"{name}_cplx_im"] = zr, zi
        sr = convolve_signed_real(pl, xr, yr)
        arrs[f"{name}_signed_real"] = sr
        cr, ci = convolve_signed_complex(pl, xr, xi, yr, yi)
        arrs[f"{name}_signed_cplx_re"], arrs[f"{name}_signed_cplx_im"] = cr, ci
    # extremes that still decode: full-scale x and h
    xe = np.full((2, 64), -16)
    he = np.full((2, 64), -32)
    he[1] = 31
    arrs["ext_x"], arrs["ext_h"] = xe, he
    arrs["ext_z"] = convolve_signed_real(p, xe, he)
    # over-budget inputs wrap modulo F (the GPU path must reproduce the wrap)
    xo = np.full((1, 64), 32768)
    ho = np.full((1, 64), 3)
    arrs["wrap_x"], arrs["wrap_h"] = xo, ho
    arrs["wrap_z"] = convolve_signed_real(p, xo, ho)
    save("convolution", **arrs)
    return digests


# --------------------------------------------------------------------------
# quantizer (fixedpoint.py:51-71)

def gen_quantize() -> None:
    rng = np.random.default_rng(303)
    x = rng.standard_normal(4096) * 1.3
    ties = (np.arange(-40, 41) + 0.5) / 8.94427190999916
    exact = np.arange(-20, 21) / 8.0
    special = np.array([0.0, -0.0, 1e300, -1e300, np.inf, -np.inf, 1.8749999999,
                        -1.875, 1.875, 5e-324])
    arrs = {"x": x, "ties": ties, "exact": exact, "special": special}
    for tag, spec in (("s5", QuantSpec(5, 8.94427190999916)),
                      ("s6", QuantSpec(6, 128.0)), ("s8", QuantSpec(8, 8.0))):
        for k in ("x", "ties", "exact", "special"):
            q, c = quantize_real(arrs[k], spec)
            arrs[f"{tag}_{k}_q"] = q
            arrs[f"{tag}_{k}_c"] = np.array(c)
    save("quantize", **arrs)


# --------------------------------------------------------------------------
# FNT-CDC (cdc.py:98-180); config 2 of BASELINE.json and edge cases

def _front_end_quantized(cfg: LinkConfig, snr_db: float, jones=None):
    """Reference Tx -> channel -> GSOP/matched filter -> 5-bit quantize.

    Mirrors linksim.run_single / rx_frontend (linksim.py:386-397, 263-291)
    but stops before the CDC so the integer engine inputs can be stored.
    """
    rng = np.random.default_rng(np.random.SeedSequence(
        [cfg.seed, int(round(snr_db * 1000))]))
    tx = linksim.generate_tx(cfg, rng)
    if jones is not None:
        saved = cfg.pol_rotation_deg
        cfg.pol_rotation_deg = 0.0
        rx, _ = _apply_channel_jones(tx.wave, cfg, snr_db, rng, jones)
        cfg.pol_rotation_deg = saved
    else:
        rx, _ = linksim.apply_channel(tx.wave, cfg, snr_db, rng)
    mf = linksim.rrc_taps(cfg.sps, cfg.rrc_span, cfg.rrc_rolloff)
    spec = cfg.sig_spec()
    q = []
    for pol in range(2):
        g = linksim.gsop(rx[pol])
        m = linksim.circ_filter(g, mf)
        c = m / np.sqrt(np.mean(np.abs(m) ** 2))
        xr, _ = quantize_real(c.real, spec)
        xi, _ = quantize_real(c.imag, spec)
        q.append((xr, xi))
    return tx, q


def _apply_channel_jones(wave, cfg, snr_db, rng, jones):
    """apply_channel (linksim.py:211-234) with the fixed real rotation replaced
    by a seeded Haar unitary Jones matrix (BASELINE config 3).
    With rotation 0 deg, dgd 0 and skew 0 the reference reduces to CD + AWGN,
    so the Jones matrix is applied between those two steps."""
    x = linksim.cd_allpass(wave, cfg)
    x = jones @ x
    if np.isfinite(snr_db):
        snr = 10.0 ** (snr_db / 10.0)
        for p in range(2):
            pw = np.mean(np.abs(x[p]) ** 2)
            sigma = np.sqrt(pw / snr / 2.0)
            x[p] = x[p] + sigma * (rng.standard_normal(x.shape[-1])
                                   + 1j * rng.standard_normal(x.shape[-1]))
    return x, {}


def c2_config() -> LinkConfig:
    return LinkConfig(n_symbols=2 ** 18, z_km=75.0, snr_db=(20.0,),
                      pol_rotation_deg=0.0, dgd_symbols=0.0, iq_skew_samples=0.0,
                      seed=1)


def gen_cdc() -> dict:
    cfg = c2_config()
    _, q = _front_end_quantized(cfg, 20.0)
    xr, xi = q[0]
    eng = FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    COUNTER.reset()
    with COUNTER.enabled_ctx():
        yr, yi = eng.process_int(xr, xi)
        n_mult = COUNTER.total("cdc-fnt")
    y = eng.process(xr, xi)
    digests = {
        "c2_xr": sha(xr.astype(np.int8)), "c2_xi": sha(xi.astype(np.int8)),
        "c2_yr": sha(yr), "c2_yi": sha(yi), "c2_process": sha(y),
        "c2_counter": int(n_mult), "c2_budget_bound": eng.budget.bound,
        "c2_tap_scale": eng.tap_scale, "c2_output_scale": eng.output_scale,
        "c2_support_warning": bool(eng.support_warning),
    }
    arrs = {
        "c2_xr": xr.astype(np.int8), "c2_xi": xi.astype(np.int8),
        "c2_yr_head": yr[:8192], "c2_yi_head": yi[:8192],
        "c2_yr_tail": yr[-4096:], "c2_yi_tail": yi[-4096:],
        "c2_y_head": y[:4096],
        "tap_re": eng.tap_re, "tap_im": eng.tap_im,
        "b_plus": eng._b_plus, "b_minus": eng._b_minus,
        "taps_float": eng.taps,
    }
    # process_block on one interior block (cdc.py:158-163)
    blk_r = xr[1000:1064]
    blk_i = xi[1000:1064]
    br, bi = eng.process_block(blk_r, blk_i)
    arrs.update(blk_r=blk_r, blk_i=blk_i, blk_out_r=br, blk_out_i=bi)

    # ragged lengths, full-scale and over-range values, other tap designs
    rng = np.random.default_rng(404)
    lens = [0, 1, 2, 15, 16, 17, 31, 32, 33, 63, 64, 65, 97, 1000, 4097]
    for L in lens:
        a = rng.integers(-15, 16, L)
        b = rng.integers(-15, 16, L)
        r, i = eng.process_int(a, b)
        arrs[f"len{L}_xr"], arrs[f"len{L}_xi"] = a, b
        arrs[f"len{L}_yr"], arrs[f"len{L}_yi"] = r, i
    # saturating input: all +15 / all -15 (budget extremes)
    a = np.full(500, 15)
    b = np.full(500, -15)
    r, i = eng.process_int(a, b)
    arrs.update(sat_xr=a, sat_xi=b, sat_yr=r, sat_yi=i)
    # values beyond the signal spec wrap modulo F inside the transform
    a = rng.integers(-32768, 32769, 300)
    b = rng.integers(-32768, 32769, 300)
    r, i = eng.process_int(a, b)
    arrs.update(wide_xr=a, wide_xi=b, wide_yr=r, wide_yi=i)
    # other tap designs: 33 taps (maximum for N=64), 25 km, z = 0, 17 taps
    for tag, cc in (("t33", CdcConfig(z_km=25.0, fs_hz=80e9, n_taps=33)),
                    ("z0", CdcConfig(z_km=0.0, fs_hz=80e9, n_taps=32)),
                    ("t17", CdcConfig(z_km=10.0, fs_hz=80e9, n_taps=17)),
                    ("t1", CdcConfig(z_km=5.0, fs_hz=80e9, n_taps=1))):
        e2 = FntCdcEngine(cc, QuantSpec(5, 8.0))
        a = rng.integers(-15, 16, 777)
        b = rng.integers(-15, 16, 777)
        r, i = e2.process_int(a, b)
        arrs[f"{tag}_tap_re"], arrs[f"{tag}_tap_im"] = e2.tap_re, e2.tap_im
        arrs[f"{tag}_scale"] = np.array(e2.tap_scale)
        arrs[f"{tag}_xr"], arrs[f"{tag}_xi"] = a, b
        arrs[f"{tag}_yr"], arrs[f"{tag}_yi"] = r, i
        arrs[f"{tag}_bp"], arrs[f"{tag}_bm"] = e2._b_plus, e2._b_minus
    save("cdc", **arrs)
    return digests


# --------------------------------------------------------------------------
# FNT-AEQ (aeq.py:84-190) and the CDC->AEQ glue (linksim.py:283-308, 399-406)

def _aeq_run(q, mu_schedule, adapt=True, mu=None):
    acfg = LinkConfig().aeq_config()
    if mu is not None:
        acfg = AeqConfig(block_n=32, l_taps=16, mu=mu, sig_spec=acfg.sig_spec)
    eq = FntAeq(acfg)
    COUNTER.reset()
    with COUNTER.enabled_ctx():
        y = eq.process(q, adapt=adapt, mu_schedule=mu_schedule)
        n_mult = COUNTER.total("aeq-fnt")
    return eq, y, n_mult


def _glue(cfg: LinkConfig, q):
    """rx_frontend tail + run_single AEQ input (linksim.py:283-308, 399-404)."""
    eng = FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    eq_streams = [eng.process(xr, xi) for xr, xi in q]
    phase = linksim._decimation_phase(eq_streams, cfg.sps)
    dec = np.stack([e[phase::cfg.sps] for e in eq_streams])
    streams = np.stack([dec[0].real, dec[0].imag, dec[1].real, dec[1].imag])
    spec = cfg.sig_spec()
    qa = np.stack([quantize_real(s, spec)[0] for s in streams])
    return eng, eq_streams, phase, qa


def gen_aeq() -> dict:
    arrs = {}
    digests = {}
    # (a) converging link: z = 0, no rotation (finding 4: the only converging case)
    cfg = LinkConfig(n_symbols=2 ** 15, z_km=0.0, snr_db=(20.0,), pol_rotation_deg=0.0,
                     dgd_symbols=0.0, iq_skew_samples=0.0, seed=5)
    _, q = _front_end_quantized(cfg, 20.0)
    _, eqs, phase, qa = _glue(cfg, q)
    eq, y, n_mult = _aeq_run(qa, cfg.mu_schedule())
    arrs.update(a_q=qa.astype(np.int8), a_y=y, a_w=eq.w, a_wint=eq.taps.w_int,
                a_hist=eq.history, a_err=np.array(eq.err_trace),
                a_sat=np.array(eq.saturations), a_phase=np.array(phase))
    digests["a_counter"] = int(n_mult)
    # (b) C2-like 75 km link with a 45 deg rotation (non-converging, finding 4)
    cfg = LinkConfig(n_symbols=2 ** 14, z_km=75.0, snr_db=(18.0,), pol_rotation_deg=45.0,
                     dgd_symbols=0.0, iq_skew_samples=0.0, seed=6)
    _, q = _front_end_quantized(cfg, 18.0)
    _, eqs, phase, qa = _glue(cfg, q)
    eq, y, _ = _aeq_run(qa, cfg.mu_schedule())
    arrs.update(b_q=qa.astype(np.int8), b_y=y, b_w=eq.w, b_wint=eq.taps.w_int,
                b_hist=eq.history, b_err=np.array(eq.err_trace),
                b_sat=np.array(eq.saturations), b_phase=np.array(phase))
    # glue intermediates for (b): process() output hash + phase
    arrs["b_cdc_y0_head"] = eqs[0][:2048]
    digests["b_cdc_y0"] = sha(eqs[0])
    digests["b_cdc_y1"] = sha(eqs[1])
    arrs["b_cdc_q"] = np.stack([np.stack(p) for p in q]).astype(np.int8)
    # (c) random 5-bit inputs, large constant mu -> saturations; adapt=False run
    rng = np.random.default_rng(505)
    xr = rng.integers(-15, 16, (4, 16 * 300))
    eq, y, _ = _aeq_run(xr, None, mu=0.05)
    arrs.update(c_q=xr.astype(np.int8), c_y=y, c_w=eq.w, c_wint=eq.taps.w_int,
                c_hist=eq.history, c_err=np.array(eq.err_trace),
                c_sat=np.array(eq.saturations))
    eq, y, n_mult = _aeq_run(xr[:, :16 * 64 + 7], None, adapt=False)
    arrs.update(d_q=xr[:, :16 * 64 + 7].astype(np.int8), d_y=y, d_err=np.array(eq.err_trace),
                d_hist=eq.history)
    digests["d_counter"] = int(n_mult)
    # (e) streaming state across process() calls + mu=0 blocks in the schedule
    eq = FntAeq(LinkConfig().aeq_config())
    sched = lambda i: 0.0 if (i // 16) % 5 == 3 else 3e-3  # noqa: E731
    xs = rng.integers(-15, 16, (4, 16 * 200))
    y1 = eq.process(xs[:, :16 * 77], mu_schedule=sched)
    y2 = eq.process(xs[:, 16 * 77:], mu_schedule=sched)
    arrs.update(e_q=xs.astype(np.int8), e_y1=y1, e_y2=y2, e_w=eq.w, e_wint=eq.taps.w_int,
                e_hist=eq.history, e_err=np.array(eq.err_trace), e_sat=np.array(eq.saturations))
    # (f) single-call API: equalize_block / update_taps (aeq.py:118-170)
    eq = FntAeq(LinkConfig().aeq_config())
    xb = rng.integers(-15, 16, (4, 16))
    yb, xblk = eq.equalize_block(xb)
    eq.update_taps(xblk, yb, mu=0.01)
    yb2, xblk2 = eq.equalize_block(rng.integers(-15, 16, (4, 16)))
    arrs.update(f_x=xb, f_y=yb, f_xblk=xblk, f_w=eq.w.copy(), f_y2=yb2, f_xblk2=xblk2)
    save("aeq", **arrs)
    return digests


# --------------------------------------------------------------------------
# config 3 at full size (hash-only; run with --big, ~minutes on all cores)

def _c3_point(snr_db: float):
    cfg = LinkConfig(n_symbols=2 ** 20, z_km=75.0, snr_db=(snr_db,), pol_rotation_deg=0.0,
                     dgd_symbols=0.0, iq_skew_samples=0.0, seed=2)
    from scipy.stats import unitary_group
    jones = unitary_group.rvs(2, random_state=np.random.default_rng(
        np.random.SeedSequence([2, 999999])))
    tx, q = _front_end_quantized(cfg, snr_db, jones=jones)
    eng, eqs, phase, qa = _glue(cfg, q)
    yint = [eng.process_int(xr, xi) for xr, xi in q]
    eq, y, _ = _aeq_run(qa, cfg.mu_schedule())
    y_pols = np.stack([y[0] + 1j * y[1], y[2] + 1j * y[3]])
    n = min(y_pols.shape[1], tx.symbols.shape[1])
    ber, evm, ok = linksim.align_and_count(y_pols[:, :n], tx, cfg)
    return snr_db, {
        "q_in": [sha(np.stack([xr, xi]).astype(np.int8)) for xr, xi in q],
        "cdc_int": [sha(np.stack([a, b])) for a, b in yint],
        "phase": int(phase), "aeq_in": sha(qa.astype(np.int8)),
        "aeq_y": sha(y), "w": sha(eq.w), "w_int": sha(eq.taps.w_int),
        "sat": int(eq.saturations), "err_trace": sha(np.array(eq.err_trace)),
        "ber": ber, "evm_db": evm, "ok": bool(ok),
    }


def gen_c3() -> dict:
    snrs = [14.0, 16.0, 18.0, 20.0, 22.0, 24.0]
    with ProcessPoolExecutor(max_workers=min(6, os.cpu_count() or 1)) as ex:
        res = dict(ex.map(_c3_point, snrs))
    return {str(k): v for k, v in res.items()}


# --------------------------------------------------------------------------
# float comparators (cdc.py:183-210, aeq.py:193-264): not on the FNT path

def gen_float() -> None:
    from fntdsp.aeq import td_aeq_float
    from fntdsp.cdc import fd_cdc_float, td_cdc_float
    cfg = c2_config()
    ccfg = cfg.cdc_config("fnt")
    rng = np.random.default_rng(77)
    x = (rng.standard_normal(2000) + 1j * rng.standard_normal(2000)) / np.sqrt(2)
    acfg = cfg.aeq_config()
    xa = rng.standard_normal((4, 1500))
    ya, wa = td_aeq_float(xa, acfg, mu_schedule=cfg.mu_schedule())
    save("float", x=x, fd=fd_cdc_float(x, ccfg), td=td_cdc_float(x, ccfg), xa=xa, ya=ya, wa=wa)


# --------------------------------------------------------------------------
# config 5: the first 64 links, end to end through the reference (hash-only, --big)

C5_LINKS = 64


def _c5_link(i: int):
    """rng_i = default_rng(SeedSequence([4, i])); snr_i ~ U[16, 22];
    U_i = unitary_group.rvs(2, random_state=rng_i); Tx / channel / front end on rng_i;
    then the reference's CDC -> glue -> FntAeq with the gear-shift schedule."""
    from scipy.stats import unitary_group
    rng = np.random.default_rng(np.random.SeedSequence([4, i]))
    snr = rng.uniform(16, 22)
    jones = unitary_group.rvs(2, random_state=rng)
    cfg = LinkConfig(n_symbols=2 ** 18, z_km=75.0, snr_db=(snr,), pol_rotation_deg=0.0,
                     dgd_symbols=0.0, iq_skew_samples=0.0, seed=4)
    tx = linksim.generate_tx(cfg, rng)
    rx, _ = _apply_channel_jones(tx.wave, cfg, snr, rng, jones)
    mf = linksim.rrc_taps(cfg.sps, cfg.rrc_span, cfg.rrc_rolloff)
    spec = cfg.sig_spec()
    q = []
    for pol in range(2):
        g = linksim.gsop(rx[pol])
        m = linksim.circ_filter(g, mf)
        c = m / np.sqrt(np.mean(np.abs(m) ** 2))
        q.append((quantize_real(c.real, spec)[0], quantize_real(c.imag, spec)[0]))
    eng, eqs, phase, qa = _glue(cfg, q)
    eq, y, _ = _aeq_run(qa, cfg.mu_schedule())
    return i, {
        "q_in": sha(np.stack([np.stack([xr, xi]) for xr, xi in q]).astype(np.int8)),
        "phase": int(phase), "aeq_y": sha(y), "w": sha(eq.w), "w_int": sha(eq.taps.w_int),
        "sat": int(eq.saturations), "err_trace": sha(np.array(eq.err_trace)),
    }


def gen_c5() -> dict:
    with ProcessPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        res = dict(ex.map(_c5_link, range(C5_LINKS)))
    return {str(k): v for k, v in sorted(res.items())}


def gen_cli() -> dict:
    """Reference CLI outputs (cli.py:135-318): selftest (+ fault injection),
    complexity --measure, transform / convolve on small files."""
    import contextlib
    import io
    import tempfile
    from fntdsp import cli
    out = {}

    def run(argv):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cli.main(argv)
        return rc, buf.getvalue()

    for key, argv in (("selftest", ["selftest"]), ("selftest_fault", ["selftest", "--fault-inject"]),
                      ("complexity", ["complexity"]), ("complexity_measure", ["complexity", "--measure"])):
        rc, text = run(argv)
        out[key] = {"rc": rc, "stdout": text}
    rng = np.random.default_rng(606)
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        x = rng.integers(-15, 16, 64)
        h = rng.integers(-31, 32, 64)
        h[20:] = 0
        np.savetxt(d / "x.txt", x, fmt="%d")
        np.savetxt(d / "h.txt", h, fmt="%d")
        np.savetxt(d / "xc.txt", rng.integers(-15, 16, (64, 2)), fmt="%d")
        hc = rng.integers(-15, 16, (64, 2))
        hc[16:] = 0
        np.savetxt(d / "hc.txt", hc, fmt="%d")
        np.savetxt(d / "x32.txt", rng.integers(0, 65537, 32), fmt="%d")
        np.savetxt(d / "big.txt", np.full(64, 30000), fmt="%d")
        files = {k: (d / f"{k}.txt").read_text() for k in ("x", "h", "xc", "hc", "x32", "big")}
        res = {}
        for key, argv in (
                ("fnt", ["transform", "--plan", "cdc64", "--input", str(d / "x.txt"), "--output", str(d / "o.txt")]),
                ("ifnt", ["transform", "--plan", "aeq32", "--inverse", "--input", str(d / "x32.txt"), "--output", str(d / "o.txt")]),
                ("conv", ["convolve", "--plan", "cdc64", "--x", str(d / "x.txt"), "--h", str(d / "h.txt"), "--output", str(d / "o.txt")]),
                ("convc", ["convolve", "--plan", "cdc64", "--mode", "complex", "--x", str(d / "xc.txt"), "--h", str(d / "hc.txt"), "--output", str(d / "o.txt")]),
                ("overflow", ["convolve", "--plan", "cdc64", "--x", str(d / "big.txt"), "--h", str(d / "h.txt"), "--output", str(d / "o2.txt")])):
            rc, _ = run(argv)
            res[key] = {"rc": rc, "out": (d / "o.txt").read_text()}
        out["files"] = files
        out["runs"] = res
    (OUT / "cli.json").write_text(json.dumps(out, indent=1))
    return {"n": len(out)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run config 3 (minutes)")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    digests_path = OUT / "digests.json"
    digests = json.loads(digests_path.read_text()) if digests_path.exists() else {}
    only = set(args.only.split(",")) if args.only else None

    def want(k):
        return only is None or k in only

    if want("plans"):
        (OUT / "plans.json").write_text(json.dumps(gen_plans(), indent=1))
    if want("transforms"):
        gen_transforms()
    if want("selftest"):
        digests["selftest"] = gen_selftest()
    if want("convolution"):
        digests["convolution"] = gen_convolution()
    if want("quantize"):
        gen_quantize()
    if want("cdc"):
        digests["cdc"] = gen_cdc()
    if want("aeq"):
        digests["aeq"] = gen_aeq()
    if want("cli"):
        gen_cli()
    if want("float"):
        gen_float()
    if args.big:
        digests["c3"] = gen_c3()
    if args.big or want("c5") and only is not None:
        digests["c5"] = gen_c5()
    digests["_generator"] = {"numpy": np.__version__, "fntdsp": fntdsp.__version__}
    digests_path.write_text(json.dumps(digests, indent=1, sort_keys=True))
    print("digests ->", digests_path)


if __name__ == "__main__":
    main()
