"""GPU parity: the sm_100a kernels (through the public drop-in API and the C
ABI) against the reference's golden fixtures and the pinned CPU oracle.
Integer outputs are compared bit-exactly; float64 AEQ outputs bit-exactly too
(the update reproduces numpy's operation order)."""

import numpy as np
import pytest

import oracle as O
import paper_2405_04253_b200 as P
from conftest import ROOT, SIG_SCALE, sha

pytestmark = pytest.mark.gpu

PLANS = ("mod17", "aeq32", "cdc64")


@pytest.fixture(scope="module")
def plans():
    return P.default_plans()


# ---------------------------------------------------------------- transforms

@pytest.mark.parametrize("name", PLANS)
def test_fnt_ifnt_golden(golden, plans, name):
    g = golden("transforms")
    p = plans[name]
    for k, suf in (("x", ""), ("xs", "_xs"), ("ext", "_ext")):
        assert np.array_equal(P.fnt(p, g[f"{name}_{k}"]), g[f"{name}_fnt{suf}"]), k
        assert np.array_equal(P.ifnt(p, g[f"{name}_{k}"]), g[f"{name}_ifnt{suf}"]), k
    out = P.fnt(p, g[f"{name}_x3"])
    assert out.shape == (3, 5, p.n) and out.dtype == np.int64
    assert np.array_equal(out, g[f"{name}_fnt3"])


def test_selftest_golden_vectors(golden, plans):
    g = golden("selftest")
    p17 = plans["mod17"]
    assert np.array_equal(P.fnt(p17, np.array([1, 0, 0, 0, 0, 0, 0, 0])), np.ones(8, np.int64))
    assert np.array_equal(P.fnt(p17, np.array([1, 1, 0, 0, 0, 0, 0, 0])), [2, 3, 5, 9, 0, 16, 14, 10])
    assert np.array_equal(P.ifnt(p17, np.array([2, 3, 5, 9, 0, 16, 14, 10])), [1, 1, 0, 0, 0, 0, 0, 0])
    for name in PLANS:
        p = plans[name]
        assert np.array_equal(P.ifnt(p, P.fnt(p, g[f"rt_{name}_x"])), g[f"rt_{name}_y"])
    assert np.array_equal(P.convolve_signed_real(p17, [1, 2, 0, 0, 0, 0, 0, 0], [3, 1, 0, 0, 0, 0, 0, 0]),
                          [3, 7, 2, 0, 0, 0, 0, 0])


def test_fault_injection_negative_control(plans):
    """cli.py:84-86: a corrupted twiddle table must change the transform."""
    p = P.default_plans()["mod17"]
    p.fwd_twiddles[-1][1] += 1
    assert not np.array_equal(P.fnt(p, np.array([1, 1, 0, 0, 0, 0, 0, 0])), [2, 3, 5, 9, 0, 16, 14, 10])
    p = P.default_plans()["cdc64"]
    x = np.random.default_rng(1).integers(0, 65537, (4, 64))
    good = P.fnt(p, x)
    p.fwd_twiddles[-1][1] += 1
    assert not np.array_equal(P.fnt(p, x), good)


@pytest.mark.parametrize("name", PLANS)
def test_random_round_trip_and_oracle(plans, name):
    p = plans[name]
    rng = np.random.default_rng(5)
    x = rng.integers(0, p.params.F, (1000, p.n))
    X = P.fnt(p, x)
    assert np.array_equal(X, O.fnt(O.Plan.named(name), x))
    assert np.array_equal(P.ifnt(p, X), x)


def test_other_valid_plans_generic_kernel():
    """Any plan make_plan accepts runs (table-driven kernel)."""
    for t, alpha, n in ((4, pow(3, 16, 65537), 1 << 12), (4, 4, 16), (3, 2, 16), (1, 2, 4), (4, 65536, 2)):
        p = P.make_plan(P.FermatParams(t), alpha, n)
        op = O.Plan(t, n, alpha)
        x = np.random.default_rng(n).integers(-(1 << 20), 1 << 20, (7, n))
        assert np.array_equal(P.fnt(p, x), O.fnt(op, x)), (t, alpha, n)
        assert np.array_equal(P.ifnt(p, x), O.ifnt(op, x)), (t, alpha, n)


def test_transform_errors(plans):
    with pytest.raises(ValueError, match="expected length 64, got 63"):
        P.fnt(plans["cdc64"], np.zeros(63))
    with pytest.raises(P.InvalidPlanError):
        P.make_plan(P.FermatParams(4), 2, 64)
    assert P.fnt(plans["cdc64"], np.zeros((0, 64))).shape == (0, 64)


# -------------------------------------------------------------- convolutions

@pytest.mark.parametrize("name", PLANS)
def test_convolution_golden(golden, plans, name):
    c = golden("convolution")
    p = plans[name]
    F = p.params.F
    xr, xi, yr, yi = (c[f"{name}_{k}"] for k in ("xr", "xi", "yr", "yi"))
    assert np.array_equal(P.cyclic_convolve_real(p, xr % F, yr[0] % F), c[f"{name}_real_bcast"])
    assert np.array_equal(P.cyclic_convolve_real(p, xr % F, yr % F), c[f"{name}_real"])
    zr, zi = P.cyclic_convolve_complex(p, xr % F, xi % F, yr % F, yi % F)
    assert np.array_equal(zr, c[f"{name}_cplx_re"]) and np.array_equal(zi, c[f"{name}_cplx_im"])
    assert np.array_equal(P.convolve_signed_real(p, xr, yr), c[f"{name}_signed_real"])
    sr, si = P.convolve_signed_complex(p, xr, xi, yr, yi)
    assert np.array_equal(sr, c[f"{name}_signed_cplx_re"]) and np.array_equal(si, c[f"{name}_signed_cplx_im"])


@pytest.mark.parametrize("name", ("aeq32", "cdc64"))
def test_staged_tiles_ragged_batches_vs_oracle(plans, name):
    """The shift-add kernels stage 64-vector tiles through shared memory: full
    tiles, partial last tiles and in-place transforms, per-vector and shared
    taps, against the oracle (fnt.py:106-161)."""
    p = plans[name]
    op = O.Plan.named(name)
    F = p.params.F
    rng = np.random.default_rng(17)
    for batch in (1, 63, 64, 65, 191, 1000):
        xr, xi, yr, yi = (rng.integers(-(1 << 40), 1 << 40, (batch, p.n)) for _ in range(4))
        assert np.array_equal(P.fnt(p, xr), O.fnt(op, xr)), batch
        assert np.array_equal(P.ifnt(p, xr), O.ifnt(op, xr)), batch
        xr, xi, yr, yi = (a % F for a in (xr, xi, yr, yi))
        assert np.array_equal(P.cyclic_convolve_real(p, xr, yr), O.cyclic_real(op, xr, yr)), batch
        assert np.array_equal(P.cyclic_convolve_real(p, xr, yr[0]), O.cyclic_real(op, xr, yr[0])), batch
        for y_re, y_im in ((yr, yi), (yr[-1], yi[-1])):
            zr, zi = P.cyclic_convolve_complex(p, xr, xi, y_re, y_im)
            rr, ri = O.cyclic_complex(op, xr, xi, y_re, y_im)
            assert np.array_equal(zr, rr) and np.array_equal(zi, ri), batch


def test_config1_full(golden, digests, plans):
    """BASELINE config 1: 16384 x 64, seed 0, bit-exact (reference digest)."""
    p = plans["cdc64"]
    rng = np.random.default_rng(0)
    x = rng.integers(-16, 16, (16384, 64))
    h = rng.integers(-32, 32, (16384, 64))
    P.COUNTER.reset()
    with P.COUNTER.enabled_ctx():
        z = P.cyclic_convolve_real(p, x % p.params.F, h % p.params.F)
        n = P.COUNTER.total()
    assert sha(z) == digests["convolution"]["c1_cyclic_real"]
    assert n == digests["convolution"]["c1_counter"]
    assert sha(P.convolve_signed_real(p, x, h)) == digests["convolution"]["c1_signed_real"]


def test_convolution_extremes(golden, plans):
    c = golden("convolution")
    p = plans["cdc64"]
    assert np.array_equal(P.convolve_signed_real(p, c["ext_x"], c["ext_h"]), c["ext_z"])
    assert np.array_equal(P.convolve_signed_real(p, c["wrap_x"], c["wrap_h"]), c["wrap_z"])
    with pytest.raises(ValueError, match="encodable signed range"):
        P.convolve_signed_real(p, np.full(64, 32769), np.zeros(64))


# ------------------------------------------------------------------ quantize

def test_quantize_golden(golden):
    q = golden("quantize")
    for tag, (bits, sc) in {"s5": (5, SIG_SCALE), "s6": (6, 128.0), "s8": (8, 8.0)}.items():
        spec = P.QuantSpec(bits, sc)
        for k in ("x", "ties", "exact", "special"):
            v, cnt = P.quantize_real(q[k], spec)
            assert v.dtype == np.int64
            assert np.array_equal(v, q[f"{tag}_{k}_q"]), (tag, k)
            assert cnt == int(q[f"{tag}_{k}_c"]), (tag, k)


def test_encode_decode_arrays():
    f = P.FermatParams(4)
    v = np.array([-32768, -1, 0, 1, 32768])
    assert np.array_equal(P.encode_signed_array(v, f), [32769, 65536, 0, 1, 32768])
    assert np.array_equal(P.decode_signed_array([32769, 65536, 0, 1, 32768, 100000], f),
                          [-32768, -1, 0, 1, 32768, 34463])
    with pytest.raises(ValueError):
        P.encode_signed_array([40000], f)


# ----------------------------------------------------------------------- CDC

@pytest.fixture(params=("shift", "tc", "umma"))
def cdc_kernel(request):
    """Run a CDC test through every kernel: the shift-add butterflies and the
    split-integer matrix form on mma.sync (tc) and on tcgen05 (umma), the latter two
    for int8 planes (cdc.set_cdc_kernel)."""
    from paper_2405_04253_b200 import cdc as cdc_mod
    prev = cdc_mod.set_cdc_kernel(request.param)
    yield request.param
    cdc_mod.set_cdc_kernel(prev)


def _c2_engine():
    cfg = P.LinkConfig(n_symbols=2 ** 18, z_km=75.0, snr_db=(20.0,), pol_rotation_deg=0.0,
                       dgd_symbols=0.0, iq_skew_samples=0.0, seed=1)
    return P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())


def test_cdc_engine_constants(golden, digests):
    a = golden("cdc")
    eng = _c2_engine()
    assert np.array_equal(eng.tap_re, a["tap_re"]) and np.array_equal(eng.tap_im, a["tap_im"])
    assert np.array_equal(eng.taps, a["taps_float"])
    assert np.array_equal(eng._b_plus, a["b_plus"]) and np.array_equal(eng._b_minus, a["b_minus"])
    d = digests["cdc"]
    assert eng.budget.bound == d["c2_budget_bound"] and eng.tap_scale == d["c2_tap_scale"]
    assert eng.output_scale == d["c2_output_scale"]
    assert eng.support_warning == d["c2_support_warning"]


def test_cdc_config2_full(golden, digests, cdc_kernel):
    """BASELINE config 2 (2^19 samples, 75 km, 20 dB) bit-exact vs the reference."""
    a = golden("cdc")
    eng = _c2_engine()
    P.COUNTER.reset()
    with P.COUNTER.enabled_ctx():
        yr, yi = eng.process_int(a["c2_xr"].astype(np.int64), a["c2_xi"].astype(np.int64))
        assert P.COUNTER.total("cdc-fnt") == digests["cdc"]["c2_counter"]
    assert yr.dtype == np.int64
    assert sha(yr) == digests["cdc"]["c2_yr"] and sha(yi) == digests["cdc"]["c2_yi"]
    # int8 input path gives the same bits
    yr8, yi8 = eng.process_int(a["c2_xr"], a["c2_xi"])
    assert np.array_equal(yr8, yr) and np.array_equal(yi8, yi)
    y = eng.process(a["c2_xr"], a["c2_xi"])
    assert y.dtype == np.complex128 and sha(y) == digests["cdc"]["c2_process"]


def test_cdc_float64_quantize_on_load_config2(digests):
    """Config 2's float front-end samples (oracle/linkgen_np, the reference's link
    model; its quantized samples are pinned to the reference's) fed as float64 and
    quantized inside the CDC's load (in_dtype F64): outputs equal the reference's
    quantize_real + process_int bit for bit, and the clip count equals quantize_real's
    (fixedpoint.py:51-60, linksim.py:289-291), for the full stream and for range shards."""
    import torch
    import oracle.linkgen_np as G
    from paper_2405_04253_b200.stream import CdcBank
    link, c = G.config2_float()
    eng = _c2_engine()
    bank = CdcBank(eng)
    c0 = c[0]
    n = c0.size
    xr = torch.from_numpy(np.ascontiguousarray(c0.real)[None]).cuda()
    xi = torch.from_numpy(np.ascontiguousarray(c0.imag)[None]).cuda()
    yr = torch.empty((1, n), dtype=torch.int64, device="cuda")
    yi = torch.empty_like(yr)
    clip = torch.zeros(1, dtype=torch.int64, device="cuda")
    bank.run(xr, xi, yr=yr, yi=yi, in_spec=eng.sig_spec, in_clipped=clip)
    assert sha(yr[0].cpu().numpy()) == digests["cdc"]["c2_yr"]
    assert sha(yi[0].cpu().numpy()) == digests["cdc"]["c2_yi"]
    want = O.quantize_real(c0.real, link.sig_scale, 15)[1] + O.quantize_real(c0.imag, link.sig_scale, 15)[1]
    assert int(clip.item()) == want > 0
    # three range shards (each fed its input window): same outputs, clip counts add up
    clip.zero_()
    cuts = [0, 123_457, 300_001, n]
    for a, b in zip(cuts[:-1], cuts[1:]):
        lo, hi = max(0, (a + 16) // 32 * 32 - 32), min(n, ((b - 1 + 16) // 32) * 32 + 32)
        sr = torch.empty((1, b - a), dtype=torch.int32, device="cuda")
        si = torch.empty_like(sr)
        bank.run(xr[:, lo:hi], xi[:, lo:hi], length=n, x_first=lo, out_first=a, out_count=b - a,
                 yr=sr, yi=si, in_spec=eng.sig_spec, in_clipped=clip)
        assert np.array_equal(sr[0].cpu().numpy(), yr[0, a:b].cpu().numpy())
        assert np.array_equal(si[0].cpu().numpy(), yi[0, a:b].cpu().numpy())
    assert int(clip.item()) >= want  # block-aligned shards may share one boundary block


def test_cdc_float64_quantize_on_load_edges():
    """Ties at +-(k + 1/2), clipping values, signed zeros, NaN and ragged lengths /
    unaligned windows: the fused quantize-on-load equals the separate quantize_real
    kernel followed by the int8 CDC (both product paths), and matches the CPU oracle
    where numpy's result is defined (no NaN)."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    bank = CdcBank(eng)
    spec = eng.sig_spec
    rng = np.random.default_rng(17)
    for L in (1, 31, 33, 4097, 70_001):
        x = rng.normal(0.0, 1.3, (2, 2, L + 3))
        k = rng.integers(-20, 21, (2, 2, L + 3)) + 0.5
        ties = rng.random((2, 2, L + 3)) < 0.2
        x[ties] = k[ties] / spec.scale * (1 + 0 * k[ties])
        x[..., :2] = [[[0.0, -0.0], [1e300, -1e300]], [[np.nan, 0.0], [3.2, -3.2]]]
        off = int(rng.integers(0, 3))
        xr = torch.from_numpy(np.ascontiguousarray(x[:, 0])).cuda()[:, off:off + L]
        xi = torch.from_numpy(np.ascontiguousarray(x[:, 1])).cuda()[:, off:off + L]
        yr = torch.empty((2, L), dtype=torch.int32, device="cuda")
        yi = torch.empty_like(yr)
        clip = torch.zeros(1, dtype=torch.int64, device="cuda")
        bank.run(xr, xi, yr=yr, yi=yi, in_spec=spec, in_clipped=clip)
        qr = np.stack([P.quantize_real(xr[s].cpu().numpy(), spec)[0] for s in range(2)])
        qi = np.stack([P.quantize_real(xi[s].cpu().numpy(), spec)[0] for s in range(2)])
        nclip = sum(P.quantize_real(t[s].cpu().numpy(), spec)[1] for t in (xr, xi) for s in range(2))
        assert int(clip.item()) == nclip, L
        rr = torch.empty_like(yr)
        ri = torch.empty_like(yr)
        bank.run(torch.from_numpy(qr.astype(np.int8)).cuda(), torch.from_numpy(qi.astype(np.int8)).cuda(),
                 yr=rr, yi=ri)
        assert torch.equal(rr, yr) and torch.equal(ri, yi), L
        for s in range(2):
            fr, fi = xr[s].cpu().numpy(), xi[s].cpu().numpy()
            ok = ~(np.isnan(fr) | np.isnan(fi))
            if ok.all():
                orr, ori = O.cdc_direct(eng.tap_re, eng.tap_im, O.quantize_real(fr, spec.scale, 15)[0],
                                        O.quantize_real(fi, spec.scale, 15)[0])
                assert np.array_equal(yr[s].cpu().numpy(), orr) and np.array_equal(yi[s].cpu().numpy(), ori)


@pytest.mark.parametrize("kernel", ["umma", "tc"])
def test_cdc_matrix_forms_equal_shift_add_on_odd_windows(kernel):
    """The tensor-core forms against the shift-add kernel on odd output ranges, odd
    input windows and int8 views at every byte misalignment (TMA-eligible and
    vector-staged windows), with the fused requantization and decimation statistics
    and with plain int16 / int32 outputs."""
    import torch
    from paper_2405_04253_b200 import cdc as cdc_mod
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    spec = eng.sig_spec
    rng = np.random.default_rng(29)
    L = 40_000
    base_r = torch.from_numpy(rng.integers(-15, 16, (3, L + 64)).astype(np.int8)).cuda()
    base_i = torch.from_numpy(rng.integers(-15, 16, (3, L + 64)).astype(np.int8)).cuda()

    def run(name, mis, a, b):
        prev = cdc_mod.set_cdc_kernel(name)
        try:
            bank = CdcBank(eng)
            lo = max(0, (a + 16) // 32 * 32 - 32 - 7)
            hi = min(L, ((b - 1 + 16) // 32) * 32 + 32 + 5)
            xr = base_r[:, mis + lo:mis + hi]
            xi = base_i[:, mis + lo:mis + hi]
            outs = {}
            for od in (torch.int16, torch.int32):
                yr = torch.empty((3, b - a), dtype=od, device="cuda")
                yi = torch.empty_like(yr)
                bank.run(xr, xi, length=L, x_first=lo, out_first=a, out_count=b - a, yr=yr, yi=yi)
                outs[str(od)] = (yr.cpu(), yi.cpu())
            qr = torch.zeros((3, b - a + 64), dtype=torch.int8, device="cuda")
            qi = torch.zeros_like(qr)
            acc = torch.zeros((3 * 8,), dtype=torch.int64, device="cuda")
            qo = 0 if mis % 4 == 0 else 1  # aligned q planes take the vectorised epilogue
            bank.run(xr, xi, length=L, x_first=lo, out_first=a, out_count=b - a,
                     qr=qr[:, qo:], qi=qi[:, qo:], q_spec=spec, decim_acc=acc)
            # decimation statistics as integers: S2 and S4 = l3 2^64 + l2 2^32 + l1 (the
            # kernels may distribute carries differently across the 32-bit limbs)
            a64 = acc.cpu().numpy().astype(np.uint64).reshape(-1, 4)
            s4 = [int(r[3]) * 2 ** 64 + int(r[2]) * 2 ** 32 + int(r[1]) for r in a64]
            outs["q"] = (qr.cpu(), qi.cpu(), torch.tensor([int(r[0]) for r in a64]))
            outs["s4"] = (s4,)
            return outs
        finally:
            cdc_mod.set_cdc_kernel(prev)

    for mis in (0, 1, 2, 3, 16):
        for a, b in ((0, L), (33, 20_001), (4097, 39_999), (1, 2)):
            ref, got = run("shift", mis, a, b), run(kernel, mis, a, b)
            for key in ref:
                for r, g in zip(ref[key], got[key]):
                    same = (r == g) if isinstance(r, list) else torch.equal(r, g)
                    assert same, (kernel, mis, a, b, key)


def test_cdc_edges(golden, cdc_kernel):
    a = golden("cdc")
    eng = _c2_engine()
    for L in (0, 1, 2, 15, 16, 17, 31, 32, 33, 63, 64, 65, 97, 1000, 4097):
        r, i = eng.process_int(a[f"len{L}_xr"], a[f"len{L}_xi"])
        assert np.array_equal(r, a[f"len{L}_yr"]) and np.array_equal(i, a[f"len{L}_yi"]), L
    for tag in ("sat", "wide"):
        r, i = eng.process_int(a[f"{tag}_xr"], a[f"{tag}_xi"])
        assert np.array_equal(r, a[f"{tag}_yr"]) and np.array_equal(i, a[f"{tag}_yi"]), tag
    br, bi = eng.process_block(a["blk_r"], a["blk_i"])
    assert np.array_equal(br, a["blk_out_r"]) and np.array_equal(bi, a["blk_out_i"])
    with pytest.raises(ValueError, match="encodable"):
        eng.process_int(np.full(10, 40000), np.zeros(10))


def test_cdc_more_streams_than_one_grid_dimension(cdc_kernel):
    """70 000 short streams in one call (the launcher splits grid.y at 65 535)."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    rng = np.random.default_rng(9)
    S, L = 70_000, 96
    xr = rng.integers(-15, 16, (S, L)).astype(np.int8)
    xi = rng.integers(-15, 16, (S, L)).astype(np.int8)
    yr = torch.empty((S, L), dtype=torch.int32, device="cuda")
    yi = torch.empty_like(yr)
    CdcBank(eng).run(torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda(), length=L, yr=yr, yi=yi)
    for s in (0, 65534, 65535, 65536, S - 1):
        orr, oi = O.cdc_process_int(eng.tap_re, eng.tap_im, xr[s], xi[s])
        assert np.array_equal(yr[s].cpu().numpy(), orr) and np.array_equal(yi[s].cpu().numpy(), oi), s


def test_cdc_int8_full_range_vs_oracle(cdc_kernel):
    """int8 planes over their whole range (the kernel's carry-free first stages
    assume |x_r +- 2^8 x_i| <= 32896) and wrapping outputs, against the oracle."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    rng = np.random.default_rng(8)
    S, L = 3, 50_003
    xr = rng.integers(-128, 128, (S, L)).astype(np.int8)
    xi = rng.integers(-128, 128, (S, L)).astype(np.int8)
    xr[0, :64] = -128
    xi[0, :64] = -128
    xr[1, :64] = 127
    xi[1, :64] = -128
    yr = torch.empty((S, L), dtype=torch.int32, device="cuda")
    yi = torch.empty_like(yr)
    CdcBank(eng).run(torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda(), length=L, yr=yr, yi=yi)
    for s in range(S):
        orr, oi = O.cdc_process_int(eng.tap_re, eng.tap_im, xr[s], xi[s])
        assert np.array_equal(yr[s].cpu().numpy(), orr), s
        assert np.array_equal(yi[s].cpu().numpy(), oi), s


def test_cdc_tc_unrepresentable_residue():
    """Tap spectra chosen so that s = u+ + u- hits 32640 on every bin of one block: the
    one residue two signed bytes cannot hold in the tensor-core form (corrected after
    the MMAs, tests/test_tc_math.py); both kernels against the numpy oracle."""
    import torch
    from paper_2405_04253_b200 import cdc as cdc_mod
    from paper_2405_04253_b200.stream import CdcBank
    from oracle import np_port as N
    F = 65537
    eng = _c2_engine()
    rng = np.random.default_rng(21)
    S, L = 2, 4096
    xr = rng.integers(-128, 128, (S, L)).astype(np.int8)
    xi = rng.integers(-128, 128, (S, L)).astype(np.int8)
    blk = 40  # window of block 40 = samples [32 * 40 - 32, 32 * 40 + 32)
    wr = xr[0, 32 * blk - 32: 32 * blk + 32].astype(np.int64)
    wi = xi[0, 32 * blk - 32: 32 * blk + 32].astype(np.int64)
    ap = (N.transform(N.CDC64, N._enc(wr, F)) + 256 * N.transform(N.CDC64, N._enc(wi, F))) % F
    bp = np.array([32640 * pow(int(a), -1, F) % F if a else 1 for a in ap], dtype=np.int64)
    bm = np.zeros(64, dtype=np.int64)
    eng._b_plus, eng._b_minus, eng._taps_c = bp, bm, None
    want = [N.cdc_process_int(xr[s].astype(np.int64), xi[s].astype(np.int64), bp, bm, 32) for s in range(S)]
    for kern in ("tc", "umma", "shift"):
        prev = cdc_mod.set_cdc_kernel(kern)
        try:
            yr = torch.empty((S, L), dtype=torch.int32, device="cuda")
            yi = torch.empty_like(yr)
            CdcBank(eng).run(torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda(), length=L, yr=yr, yi=yi)
        finally:
            cdc_mod.set_cdc_kernel(prev)
        for s in range(S):
            assert np.array_equal(yr[s].cpu().numpy(), want[s][0]), (kern, s)
            assert np.array_equal(yi[s].cpu().numpy(), want[s][1]), (kern, s)


@pytest.mark.parametrize("ties", ("engine", "mixed"))
def test_cdc_fused_requantization_tie_tables(cdc_kernel, ties):
    """The fused int8 requantization (linksim.py:404 via quantize_real) against a numpy
    restatement on the kernel's own int32 outputs: with the engine's tie table (every
    tie rounds away: the kernels' shift-only fast form) and with a table whose even
    ties round down (the general form with the table lookup)."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    bank = CdcBank(eng)
    rng = np.random.default_rng(17)
    S, L = 2, 40_004
    xr = rng.integers(-16, 16, (S, L)).astype(np.int8)
    xi = rng.integers(-16, 16, (S, L)).astype(np.int8)
    dxr, dxi = torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda()
    y32r = torch.empty((S, L), dtype=torch.int32, device="cuda")
    y32i = torch.empty_like(y32r)
    bank.run(dxr, dxi, yr=y32r, yi=y32i)
    orig = bank._exact_requant
    tie = {}

    def patched(io, q_spec):
        orig(io, q_spec)
        if ties == "mixed":
            for j in range(0, int(q_spec.max_int) + 1, 2):
                io.q_tie[j] = min(j, int(q_spec.max_int))
        tie["k"] = io.q_shift
        tie["t"] = [int(io.q_tie[j]) for j in range(int(q_spec.max_int) + 1)]

    bank._exact_requant = patched
    qr = torch.empty((S, L), dtype=torch.int8, device="cuda")
    qi = torch.empty_like(qr)
    y16r = torch.empty((S, L), dtype=torch.int16, device="cuda")
    y16i = torch.empty_like(y16r)
    spec = eng.sig_spec
    bank.run(dxr, dxi, yr=y16r, yi=y16i, qr=qr, qi=qi, q_spec=spec)
    k, t, qmax = tie["k"], np.array(tie["t"]), int(spec.max_int)
    assert k == 7 and (ties == "engine") == all(t[j] == min(j + 1, qmax) for j in range(qmax + 1))

    def want(y):
        a = np.abs(y.astype(np.int64))
        base, rem, half = a >> k, a & ((1 << k) - 1), 1 << (k - 1)
        q = base + (rem > half)
        q = np.where(rem == half, t[np.minimum(base, qmax)], q)
        q = np.minimum(q, qmax)
        return np.where(y < 0, -q, q).astype(np.int8)

    for got, y in ((qr, y32r), (qi, y32i)):
        yy = y.cpu().numpy()
        assert np.array_equal(got.cpu().numpy(), want(yy))
    assert np.array_equal(y16r.cpu().numpy(), y32r.cpu().numpy().astype(np.int16))
    assert np.array_equal(y16i.cpu().numpy(), y32i.cpu().numpy().astype(np.int16))


def test_cdc_fused_statistics_full_range(cdc_kernel):
    """The fused decimation statistics (S2 = sum |y|^2, S4 = sum |y|^4 per stream and
    output parity) and the int8 requantization at the int16 extremes: full-range int8
    inputs, whose outputs wrap over the whole residue range, against numpy on the
    kernel's own int16 outputs; streams of odd and ragged lengths."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    bank = CdcBank(eng)
    rng = np.random.default_rng(23)
    for S, L in ((3, 70_001), (2, 4099), (1, 33)):
        xr = rng.integers(-128, 128, (S, L)).astype(np.int8)
        xi = rng.integers(-128, 128, (S, L)).astype(np.int8)
        xr[0, : min(L, 4096)] = -128
        xi[0, : min(L, 4096)] = 127 if S > 1 else -128
        dxr, dxi = torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda()
        y16r = torch.empty((S, L), dtype=torch.int16, device="cuda")
        y16i = torch.empty_like(y16r)
        qr = torch.empty((S, L), dtype=torch.int8, device="cuda")
        qi = torch.empty_like(qr)
        acc = torch.zeros((S * 8,), dtype=torch.int64, device="cuda")
        bank.run(dxr, dxi, yr=y16r, yi=y16i)
        bank.run(dxr, dxi, qr=qr, qi=qi, q_spec=eng.sig_spec, decim_acc=acc)
        yr = y16r.cpu().numpy().astype(np.int64)
        yi = y16i.cpu().numpy().astype(np.int64)
        assert np.abs(yr).max() >= 32000  # the wrap reaches the extremes
        a64 = acc.cpu().numpy().astype(np.uint64).reshape(S, 2, 4)
        for s in range(S):
            for ph in range(2):
                m2 = yr[s, ph::2] ** 2 + yi[s, ph::2] ** 2
                w = [int(x) for x in a64[s, ph]]
                assert w[0] == int(m2.sum()), (S, L, s, ph)
                assert w[3] * 2 ** 64 + w[2] * 2 ** 32 + w[1] == sum(int(x) ** 2 for x in m2), (S, L, s, ph)
        k, qmax = 7, int(eng.sig_spec.max_int)
        for got, y in ((qr, yr), (qi, yi)):
            q = np.minimum((np.abs(y) + (1 << (k - 1))) >> k, qmax)
            assert np.array_equal(got.cpu().numpy(), np.where(y < 0, -q, q).astype(np.int8))


@pytest.mark.parametrize("tag,cfg", [
    ("t33", dict(z_km=25.0, fs_hz=80e9, n_taps=33)),
    ("z0", dict(z_km=0.0, fs_hz=80e9, n_taps=32)),
    ("t17", dict(z_km=10.0, fs_hz=80e9, n_taps=17)),
    ("t1", dict(z_km=5.0, fs_hz=80e9, n_taps=1)),
])
def test_cdc_other_tap_designs(golden, tag, cfg, cdc_kernel):
    a = golden("cdc")
    eng = P.FntCdcEngine(P.CdcConfig(**cfg), P.QuantSpec(5, 8.0))
    assert np.array_equal(eng.tap_re, a[f"{tag}_tap_re"]) and eng.tap_scale == float(a[f"{tag}_scale"])
    r, i = eng.process_int(a[f"{tag}_xr"], a[f"{tag}_xi"])
    assert np.array_equal(r, a[f"{tag}_yr"]) and np.array_equal(i, a[f"{tag}_yi"])


def test_cdc_budget_error():
    with pytest.raises(P.BudgetError):
        P.FntCdcEngine(P.CdcConfig(z_km=0.0, fs_hz=80e9, n_taps=32), P.QuantSpec(12, 8.0))


def test_cdc_bank_ranges_match_full_stream(cdc_kernel):
    """Range shards with the 15/16-sample halo reproduce the full stream
    (SURVEY 8e), through the device-resident multi-stream API."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    bank = CdcBank(eng)
    rng = np.random.default_rng(11)
    S, L = 3, 100_003
    xr = rng.integers(-15, 16, (S, L)).astype(np.int8)
    xi = rng.integers(-15, 16, (S, L)).astype(np.int8)
    dxr, dxi = torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda()
    yr = torch.empty((S, L), dtype=torch.int32, device="cuda")
    yi = torch.empty_like(yr)
    bank.run(dxr, dxi, yr=yr, yi=yi)
    full_r, full_i = yr.cpu().numpy(), yi.cpu().numpy()
    for s in range(S):
        orr, ori = O.cdc_direct(eng.tap_re, eng.tap_im, xr[s], xi[s])
        assert np.array_equal(full_r[s], orr) and np.array_equal(full_i[s], ori)
    # 4 uneven shards, each fed only its inputs [a - 48, b + 48) (block-aligned halo)
    cuts = [0, 17_000, 50_001, 77_777, L]
    for a, b in zip(cuts[:-1], cuts[1:]):
        lo, hi = max(0, (a + 16) // 32 * 32 - 32), min(L, ((b - 1 + 16) // 32) * 32 + 32)
        sr = torch.empty((S, b - a), dtype=torch.int32, device="cuda")
        si = torch.empty_like(sr)
        bank.run(dxr[:, lo:hi].contiguous(), dxi[:, lo:hi].contiguous(), length=L, x_first=lo,
                 out_first=a, out_count=b - a, yr=sr, yi=si)
        assert np.array_equal(sr.cpu().numpy(), full_r[:, a:b])
        assert np.array_equal(si.cpu().numpy(), full_i[:, a:b])
    # a shard missing part of its halo is rejected before launch
    with pytest.raises(ValueError, match="needed"):
        bank.run(dxr[:, 1000:2000].contiguous(), dxi[:, 1000:2000].contiguous(), length=L,
                 x_first=1000, out_first=1000, out_count=1000, yr=sr, yi=si)


# ----------------------------------------------------------------------- AEQ

AEQ_MODES = (0, 1)  # FNTGPU_AEQ_FWD_FNT, FNTGPU_AEQ_FWD_DIRECT


@pytest.fixture(params=("warp", "pol"))
def aeq_kernel(request):
    """Every AEQ test runs through both stream layouts: one warp per stream
    (k_aeq.cu) and two warps per stream, one per polarization (k_aeq_pol.cu)."""
    from paper_2405_04253_b200 import aeq as A
    prev = A.set_aeq_kernel(request.param)
    yield request.param
    A.set_aeq_kernel(prev)


def _aeq(mu=1e-4, forward=0):
    cfg = P.AeqConfig(block_n=32, l_taps=16, mu=mu, sig_spec=P.QuantSpec(5, SIG_SCALE))
    return P.FntAeq(cfg, forward=forward)


@pytest.mark.parametrize("forward", AEQ_MODES)
@pytest.mark.parametrize("tag", ["a", "b"])
def test_aeq_link_golden(golden, tag, forward, aeq_kernel):
    g = golden("aeq")
    eq = _aeq(forward=forward)
    cfg = P.LinkConfig()
    y = eq.process(g[f"{tag}_q"], adapt=True, mu_schedule=cfg.mu_schedule())
    assert np.array_equal(y, g[f"{tag}_y"])
    assert np.array_equal(eq.w, g[f"{tag}_w"])
    assert np.array_equal(eq.taps.w_int, g[f"{tag}_wint"])
    assert np.array_equal(eq.history, g[f"{tag}_hist"])
    assert np.array_equal(np.array(eq.err_trace), g[f"{tag}_err"])
    assert eq.saturations == int(g[f"{tag}_sat"])
    assert eq.symbols_processed == g[f"{tag}_q"].shape[1] // 16 * 16


@pytest.mark.parametrize("forward", AEQ_MODES)
def test_aeq_saturation_noadapt_streaming(golden, forward, aeq_kernel):
    g = golden("aeq")
    eq = _aeq(mu=0.05, forward=forward)
    y = eq.process(g["c_q"])
    assert np.array_equal(y, g["c_y"]) and np.array_equal(eq.w, g["c_w"])
    assert np.array_equal(eq.taps.w_int, g["c_wint"]) and eq.saturations == int(g["c_sat"])
    assert np.array_equal(np.array(eq.err_trace), g["c_err"])
    eq = _aeq(forward=forward)
    P.COUNTER.reset()
    with P.COUNTER.enabled_ctx():
        y = eq.process(g["d_q"], adapt=False)
        assert P.COUNTER.total("aeq-fnt") == 65536
    assert np.array_equal(y, g["d_y"]) and eq.err_trace == []
    assert np.array_equal(eq.history, g["d_hist"])
    eq = _aeq(forward=forward)
    sched = lambda i: 0.0 if (i // 16) % 5 == 3 else 3e-3  # noqa: E731
    q = g["e_q"]
    y1 = eq.process(q[:, :16 * 77], mu_schedule=sched)
    y2 = eq.process(q[:, 16 * 77:], mu_schedule=sched)
    assert np.array_equal(y1, g["e_y1"]) and np.array_equal(y2, g["e_y2"])
    assert np.array_equal(eq.w, g["e_w"]) and np.array_equal(eq.taps.w_int, g["e_wint"])
    assert np.array_equal(np.array(eq.err_trace), g["e_err"])


def test_aeq_single_block_api(golden, aeq_kernel):
    g = golden("aeq")
    eq = _aeq()
    y, xb = eq.equalize_block(g["f_x"])
    assert np.array_equal(y, g["f_y"]) and np.array_equal(xb, g["f_xblk"])
    eq.update_taps(xb, y, mu=0.01)
    assert np.array_equal(eq.w, g["f_w"])
    y2, xb2 = eq.equalize_block(g["f_xblk2"][:, 16:])
    assert np.array_equal(y2, g["f_y2"]) and np.array_equal(xb2, g["f_xblk2"])


@pytest.mark.parametrize("forward", AEQ_MODES)
def test_aeq_nan_and_inf_step_size(golden, forward, aeq_kernel):
    """NaN and inf mu blocks (reference fixture aeq_nan.npz): NaN / inf float taps,
    14-bit taps -16383 and not counted as saturations (numpy's INT64_MIN cast), through
    FntAeq (single stream) and the multi-stream kernel's fast path."""
    import torch
    from paper_2405_04253_b200.stream import AeqBank
    g = golden("aeq_nan")
    eq = _aeq(mu=1e-4, forward=forward)
    mu = g["mu"]
    y = eq.process(g["x"], adapt=True, mu_schedule=lambda i: mu[i // 16])
    assert np.array_equal(y, g["y"])
    assert np.array_equal(eq.w, g["w"], equal_nan=True)
    assert np.array_equal(eq.taps.w_int, g["w_int"]) and eq.saturations == int(g["sat"])
    assert np.array_equal(np.array(eq.err_trace), g["err"], equal_nan=True)
    cfg = P.LinkConfig().aeq_config()
    cfg.sig_spec = P.QuantSpec(5, SIG_SCALE)
    bank = AeqBank(cfg, 3, forward=forward)
    x = torch.from_numpy(np.stack([g["x"]] * 3).astype(np.int8)).cuda()
    nb = g["x"].shape[1] // 16
    yd = torch.empty((3, 4, 16 * nb), dtype=torch.float64, device="cuda")
    err = torch.empty((3, nb), dtype=torch.float64, device="cuda")
    bank.run_planar(x, nb, yd, mu_blocks=torch.from_numpy(mu).cuda(), err=err)
    st = bank.read_state()
    for s in range(3):
        assert np.array_equal(yd[s].cpu().numpy(), g["y"])
        assert np.array_equal(err[s].cpu().numpy(), g["err"], equal_nan=True)
        assert np.array_equal(np.array(st[s].w).reshape(4, 4, 16), g["w"], equal_nan=True)
        assert np.array_equal(np.array(st[s].w_int).reshape(4, 4, 16), g["w_int"])
        assert int(st[s].saturations) == int(g["sat"])


@pytest.mark.parametrize("forward", AEQ_MODES)
def test_aeq_wide_inputs_match_oracle(forward, aeq_kernel):
    """|x| up to 2^15: per-group residues wrap mod F exactly as the reference's."""
    rng = np.random.default_rng(3)
    x = rng.integers(-32768, 32769, (4, 16 * 40))
    eq = _aeq(forward=forward)
    y = eq.process(x, adapt=False)
    oq = O.Aeq(SIG_SCALE)
    assert np.array_equal(y, oq.process(x, adapt=False))
    x = rng.integers(-300, 301, (4, 16 * 40))
    eq = _aeq(mu=1e-6, forward=forward)
    oq = O.Aeq(SIG_SCALE, mu=1e-6)
    assert np.array_equal(eq.process(x), oq.process(x))
    assert np.array_equal(eq.w, oq.w)


@pytest.mark.parametrize("forward", AEQ_MODES)
def test_aeq_int8_extremes_vs_oracle(forward, aeq_kernel):
    """int8 inputs over the whole int8 range, -128 included (the update's x / sig_scale
    for every int8 value), adapting, against the oracle: y, w, w_int and err_trace."""
    rng = np.random.default_rng(29)
    x = rng.integers(-128, 128, (4, 16 * 48))
    x[:, ::7] = -128
    x[1, 5::11] = 127
    eq = _aeq(mu=1e-7, forward=forward)
    oq = O.Aeq(SIG_SCALE, mu=1e-7)
    assert np.array_equal(eq.process(x), oq.process(x))
    assert np.array_equal(eq.w, oq.w)
    assert np.array_equal(eq.taps.w_int, oq.w_int)
    assert np.array_equal(np.asarray(eq.err_trace), np.asarray(oq.err_trace))


def test_aeq_bank_many_streams_vs_oracle(aeq_kernel):
    """The multi-stream kernel (one warp per stream) against the oracle on
    independent random streams with the LinkConfig gear-shift schedule."""
    import torch
    from paper_2405_04253_b200.stream import AeqBank
    cfg = P.LinkConfig().aeq_config()
    S, nb = 37, 300
    rng = np.random.default_rng(21)
    x = rng.integers(-15, 16, (S, 4, 16 * nb)).astype(np.int8)
    mu = O.mu_blocks(nb, mu1=2e-3, mu2=1e-4, gear_symbols=2000)
    for forward in AEQ_MODES:
        bank = AeqBank(cfg, S, forward=forward)
        y = torch.empty((S, 4, 16 * nb), dtype=torch.float64, device="cuda")
        err = torch.empty((S, nb), dtype=torch.float64, device="cuda")
        bank.run_planar(torch.from_numpy(x).cuda(), nb, y, mu_blocks=torch.from_numpy(mu).cuda(), err=err)
        yh, eh = y.cpu().numpy(), err.cpu().numpy()
        st = bank.read_state()
        for s in (0, 1, 17, 36):
            oq = O.Aeq(cfg.sig_spec.scale, mu=cfg.mu)
            oy = oq.process(x[s].astype(np.int64), mu_blocks=mu)
            assert np.array_equal(yh[s], oy), (forward, s)
            assert np.array_equal(eh[s], np.array(oq.err_trace))
            assert np.array_equal(np.array(st[s].w).reshape(4, 4, 16), oq.w)


@pytest.mark.parametrize("forward", AEQ_MODES)
def test_aeq_wide_then_narrow_calls_vs_oracle(forward, aeq_kernel):
    """A call with wide inputs leaves an out-of-int8 history; the next call with
    int8 inputs (DP4A direct form) must fall back for that history exactly."""
    rng = np.random.default_rng(46)
    eq = _aeq(mu=1e-4, forward=forward)
    oq = O.Aeq(SIG_SCALE, mu=1e-4)
    for x in (rng.integers(-3000, 3001, (4, 16 * 40)), rng.integers(-15, 16, (4, 16 * 40)),
              rng.integers(-15, 16, (4, 16 * 40))):
        y = eq.process(x.astype(np.int64), adapt=True)
        oy = oq.process(x.astype(np.int64))
        assert np.array_equal(y, oy)
    assert np.array_equal(eq.w, oq.w) and np.array_equal(eq.history, oq.history)


@pytest.mark.parametrize("forward", AEQ_MODES)
def test_aeq_bank_wide_int32_inputs_vs_oracle(forward, aeq_kernel):
    """int32 planar inputs up to |x| = 2^15 (group convolutions wrap mod F4 and are
    decoded one by one, as in the reference) through the multi-stream kernel's fast
    path (per-block mu, err_trace), against the oracle."""
    import torch
    from paper_2405_04253_b200.stream import AeqBank
    cfg = P.LinkConfig().aeq_config()
    S, nb = 5, 120
    rng = np.random.default_rng(44)
    x = rng.integers(-32768, 32769, (S, 4, 16 * nb)).astype(np.int32)
    mu = O.mu_blocks(nb, mu1=2e-3, mu2=1e-4, gear_symbols=800)
    bank = AeqBank(cfg, S, forward=forward)
    y = torch.empty((S, 4, 16 * nb), dtype=torch.float64, device="cuda")
    err = torch.empty((S, nb), dtype=torch.float64, device="cuda")
    bank.run_planar(torch.from_numpy(x).cuda(), nb, y, mu_blocks=torch.from_numpy(mu).cuda(), err=err)
    st = bank.read_state()
    for s in range(S):
        oq = O.Aeq(cfg.sig_spec.scale, mu=cfg.mu)
        oy = oq.process(x[s].astype(np.int64), mu_blocks=mu)
        assert np.array_equal(y[s].cpu().numpy(), oy), (forward, s)
        assert np.array_equal(err[s].cpu().numpy(), np.array(oq.err_trace))
        assert np.array_equal(np.array(st[s].w).reshape(4, 4, 16), oq.w)
        assert int(st[s].saturations) == int(oq.saturations)


@pytest.mark.parametrize("forward", AEQ_MODES)
@pytest.mark.parametrize("case", ["bursts", "big_taps", "mu_zero", "int32"])
def test_aeq_stream_sum_switching_vs_oracle(case, forward, aeq_kernel):
    """The FNT forward sums the four input streams before the inverse transform only
    when an exact range test passes (max |x| <= 16 over the block window and the
    tap-digit mass bound, k_aeq.cu fused_ok); otherwise it decodes per (s, t, group)
    like the reference. Blocks switch between the two forms within a stream:
    amplitude bursts past 16 (int8), taps driven to saturation by a large mu (the
    digit bound fails), and fixed taps (mu = 0). The DIRECT forward skips its
    per-group decodes on the same max |x| <= 16 test."""
    import torch
    from paper_2405_04253_b200.stream import AeqBank
    cfg = P.LinkConfig().aeq_config()
    S, nb = 6, 240
    rng = np.random.default_rng(61)
    x = rng.integers(-15, 16, (S, 4, 16 * nb))
    if case == "int32":  # 32-bit input rows: small blocks take the stream sum, wide ones not
        for s in range(S):
            for b in rng.choice(nb, nb // 5, replace=False):
                x[s, :, 16 * b:16 * b + 16] = rng.integers(-40000, 40001, (4, 16))
        mu = O.mu_blocks(nb, mu1=2e-3, mu2=1e-4, gear_symbols=1600)
    elif case == "bursts":
        for s in range(S):
            for b in rng.choice(nb, nb // 4, replace=False):
                a = int(rng.choice([16, 17, 40, 127]))
                t = int(rng.integers(0, 4))
                x[s, t, 16 * b:16 * b + 16] = rng.integers(-a, a + 1, 16)
        mu = O.mu_blocks(nb, mu1=2e-3, mu2=1e-4, gear_symbols=1600)
    elif case == "big_taps":
        mu = O.mu_blocks(nb, mu1=0.05, mu2=2e-3, gear_symbols=1600)
    else:
        mu = np.zeros(nb)
    x = x.astype(np.int32 if case == "int32" else np.int8)
    bank = AeqBank(cfg, S, forward=forward)
    y = torch.empty((S, 4, 16 * nb), dtype=torch.float64, device="cuda")
    err = torch.empty((S, nb), dtype=torch.float64, device="cuda")
    bank.run_planar(torch.from_numpy(x).cuda(), nb, y, mu_blocks=torch.from_numpy(mu).cuda(), err=err)
    yh, eh = y.cpu().numpy(), err.cpu().numpy()
    st = bank.read_state()
    for s in range(S):
        oq = O.Aeq(cfg.sig_spec.scale, mu=cfg.mu)
        oy = oq.process(x[s].astype(np.int64), mu_blocks=mu)
        assert np.array_equal(yh[s], oy), (case, forward, s)
        assert np.array_equal(eh[s], np.array(oq.err_trace)), (case, s)
        assert np.array_equal(np.array(st[s].w).reshape(4, 4, 16), oq.w), (case, s)
        assert np.array_equal(np.array(st[s].w_int).reshape(4, 4, 16), oq.w_int), (case, s)
        assert int(st[s].saturations) == int(oq.saturations), (case, s)
    if case == "big_taps":
        assert max(int(st[s].saturations) for s in range(S)) > 0


@pytest.mark.parametrize("case", [
    dict(radii=[0.6, 1.3]),                                   # 2 rings: general path
    dict(radii=[0.4, 0.9, 1.5], tap_scale=4096.0),            # 3 rings: fast path, other thresholds
    dict(radii=[0.1, 0.3, 0.5, 0.8, 1.0, 1.3, 1.6, 2.2]),     # 8 rings
    dict(no_err=True),                                        # 16QAM rings without err_trace
])
def test_aeq_bank_other_parameters_vs_oracle(case, aeq_kernel):
    """The equalizer kernel's general (runtime-parameter) path and its compile-time
    fast path with other rings / tap scales, against the oracle."""
    import torch
    from paper_2405_04253_b200.stream import AeqBank
    kw = {"radii": case["radii"]} if "radii" in case else {}
    cfg = P.AeqConfig(block_n=32, l_taps=16, mu=1e-4, sig_spec=P.QuantSpec(5, SIG_SCALE),
                      tap_scale=case.get("tap_scale", 8192.0), **kw)
    S, nb = 9, 200
    rng = np.random.default_rng(33)
    x = rng.integers(-15, 16, (S, 4, 16 * nb)).astype(np.int8)
    mu = O.mu_blocks(nb, mu1=2e-3, mu2=1e-4, gear_symbols=1600)
    bank = AeqBank(cfg, S)
    y = torch.empty((S, 4, 16 * nb), dtype=torch.float64, device="cuda")
    err = None if case.get("no_err") else torch.empty((S, nb), dtype=torch.float64, device="cuda")
    bank.run_planar(torch.from_numpy(x).cuda(), nb, y, mu_blocks=torch.from_numpy(mu).cuda(), err=err)
    yh = y.cpu().numpy()
    st = bank.read_state()
    for s in (0, 4, 8):
        oq = O.Aeq(SIG_SCALE, tap_scale=cfg.tap_scale, mu=cfg.mu, radii=cfg.radii)
        oy = oq.process(x[s].astype(np.int64), mu_blocks=mu)
        assert np.array_equal(yh[s], oy), s
        if err is not None:
            assert np.array_equal(err.cpu().numpy()[s], np.array(oq.err_trace))
        assert np.array_equal(np.array(st[s].w).reshape(4, 4, 16), oq.w)
        assert int(st[s].saturations) == int(oq.saturations)


# ------------------------------------------------------- CDC -> AEQ glue chain

def test_chain_matches_reference_glue(golden, cdc_kernel, aeq_kernel):
    """CDC (fused requantization + decimation statistics) -> phase -> AEQ on the
    75 km / 45 deg link of fixture b: phase, requantized AEQ input and the AEQ
    outputs equal the reference's rx_frontend + run_single glue."""
    import torch
    from paper_2405_04253_b200.stream import CdcAeqChain
    g = golden("aeq")
    cfg = P.LinkConfig(n_symbols=2 ** 14, z_km=75.0, snr_db=(18.0,), pol_rotation_deg=45.0,
                       dgd_symbols=0.0, iq_skew_samples=0.0, seed=6)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    q = g["b_cdc_q"]  # (pol, re/im, L) int8 front-end samples
    L = q.shape[-1]
    xr = torch.from_numpy(np.ascontiguousarray(q[:, 0])).cuda()
    xi = torch.from_numpy(np.ascontiguousarray(q[:, 1])).cuda()
    chain = CdcAeqChain(eng, cfg.aeq_config(), 1, L, cfg.sig_spec(), cfg.mu_schedule(),
                        keep_cdc_int=True)
    chain.run(xr, xi)
    assert int(chain.phase.cpu()[0]) == int(g["b_phase"])
    ph = int(g["b_phase"])
    qa = np.stack([chain.qr[0, ph:L:2].cpu().numpy(), chain.qi[0, ph:L:2].cpu().numpy(),
                   chain.qr[1, ph:L:2].cpu().numpy(), chain.qi[1, ph:L:2].cpu().numpy()])
    assert np.array_equal(qa, g["b_q"].astype(np.int8))
    y = chain.y[0].cpu().numpy()
    assert np.array_equal(y, g["b_y"])
    assert np.array_equal(chain.err[0].cpu().numpy(), g["b_err"])
    y0 = eng.process(q[0, 0], q[0, 1])
    assert np.array_equal(y0[:2048], g["b_cdc_y0_head"])


@pytest.mark.parametrize("case", [
    dict(),                                                   # the link config (16QAM rings)
    dict(tap_scale=4096.0),
    dict(tap_scale=1000.5, sig=3.3),
    dict(radii=[0.7, 1.3]),
    dict(radii=[0.1, 0.2, 0.5, 0.9, 1.0, 1.4, 2.0, 3.0]),
    dict(radii=[1.0, 1.0, 2.0]),                              # duplicate ring: never chosen
])
def test_aeq_division_and_ring_shortcuts(case):
    """The kernel's y = y_int / D (reciprocal + one correction FMA) equals IEEE division
    for EVERY int32 numerator, and the threshold ring decision equals sqrt + first
    argmin (fntgpu_aeq_selfcheck)."""
    from paper_2405_04253_b200.aeq import aeq_selfcheck
    cfg = P.AeqConfig(block_n=32, l_taps=16, sig_spec=P.QuantSpec(5, case.get("sig", SIG_SCALE)),
                      tap_scale=case.get("tap_scale", float(1 << 13)),
                      **({"radii": case["radii"]} if "radii" in case else {}))
    assert aeq_selfcheck(cfg) == (0, 0)


def test_randomized_differential_vs_oracle():
    """A short run of tools/fuzz_parity.py (fixed seed): random AEQ states / inputs /
    step sizes through both layouts and forwards, random CDC designs and lengths."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("fuzz_parity", ROOT / "tools" / "fuzz_parity.py")
    fz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fz)
    rng = np.random.default_rng(2405)
    stats = {}
    for _ in range(150):
        u = rng.random()
        (fz.aeq_case if u < 0.5 else fz.cdc_case if u < 0.62 else fz.cdc_bank_case if u < 0.74
         else fz.chain_case if u < 0.84 else fz.transform_case if u < 0.94 else fz.host_case)(rng, stats)
    assert sum(stats.values()) == 150


def test_cdc_float64_persistent_many_items():
    """The persistent float64 CDC (several items per CTA, each next window prefetched
    by TMA while the current one is transformed) over 3 streams x ~2^20 samples,
    aligned and unaligned views (bulk and synchronous staging mixed), equals the
    separate quantize_real + int8 CDC, clip count included."""
    import torch
    from paper_2405_04253_b200.stream import CdcBank
    eng = _c2_engine()
    bank = CdcBank(eng)
    spec = eng.sig_spec
    rng = np.random.default_rng(29)
    L = (1 << 20) + 77
    for off in (0, 1):
        x = rng.normal(0.0, 1.6, (2, 3, L + 2))
        xr = torch.from_numpy(x[0]).cuda()[:, off:off + L]
        xi = torch.from_numpy(x[1]).cuda()[:, off:off + L]
        yr = torch.empty((3, L), dtype=torch.int16, device="cuda")
        yi = torch.empty_like(yr)
        clip = torch.zeros(1, dtype=torch.int64, device="cuda")
        bank.run(xr, xi, yr=yr, yi=yi, in_spec=spec, in_clipped=clip)
        q = [np.stack([P.quantize_real(t[s].cpu().numpy(), spec)[0] for s in range(3)]) for t in (xr, xi)]
        nclip = sum(P.quantize_real(t[s].cpu().numpy(), spec)[1] for t in (xr, xi) for s in range(3))
        assert int(clip.item()) == nclip > 0
        rr = torch.empty_like(yr)
        ri = torch.empty_like(yr)
        bank.run(torch.from_numpy(q[0].astype(np.int8)).cuda(), torch.from_numpy(q[1].astype(np.int8)).cuda(),
                 yr=rr, yi=ri)
        assert torch.equal(rr, yr) and torch.equal(ri, yi), off
