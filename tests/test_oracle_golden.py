"""Pin the CPU oracle (oracle/) to the reference's own outputs before it is
trusted as the checker for GPU parity (tests/golden/ was produced by the
unmodified reference, see tests/golden/make_golden.py)."""

import json

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, SIG_SCALE, sha

PLANS = ("mod17", "aeq32", "cdc64")


@pytest.mark.parametrize("name", PLANS)
def test_plan_tables_match_reference(name):
    ref = json.loads((GOLDEN / "plans.json").read_text())[name]
    p = O.Plan.named(name)
    assert p.code == 0
    assert p.F == ref["F"] and p.n == ref["n"] and p.alpha == ref["alpha"]


@pytest.mark.parametrize("name", PLANS)
def test_transforms(golden, name):
    g = golden("transforms")
    p = O.Plan.named(name)
    for k, suf in (("x", ""), ("xs", "_xs"), ("ext", "_ext")):
        assert np.array_equal(O.fnt(p, g[f"{name}_{k}"]), g[f"{name}_fnt{suf}"])
        assert np.array_equal(O.ifnt(p, g[f"{name}_{k}"]), g[f"{name}_ifnt{suf}"])
    assert np.array_equal(O.fnt(p, g[f"{name}_x3"]), g[f"{name}_fnt3"])


def test_selftest_vectors(golden, digests):
    g = golden("selftest")
    p17 = O.Plan.named("mod17")
    assert np.array_equal(O.fnt(p17, [1, 0, 0, 0, 0, 0, 0, 0]), g["delta_fnt"])
    assert np.array_equal(g["pair_fnt"], [2, 3, 5, 9, 0, 16, 14, 10])
    assert np.array_equal(O.fnt(p17, [1, 1, 0, 0, 0, 0, 0, 0]), g["pair_fnt"])
    assert np.array_equal(O.ifnt(p17, g["pair_fnt"]), g["pair_ifnt"])
    for name in PLANS:
        p = O.Plan.named(name)
        assert np.array_equal(O.ifnt(p, O.fnt(p, g[f"rt_{name}_x"])), g[f"rt_{name}_y"])
    assert digests["selftest"]["sqrt2"] == 4080


@pytest.mark.parametrize("name", PLANS)
def test_convolutions(golden, name):
    c = golden("convolution")
    p = O.Plan.named(name)
    F = p.F
    xr, xi, yr, yi = (c[f"{name}_{k}"] for k in ("xr", "xi", "yr", "yi"))
    assert np.array_equal(O.cyclic_real(p, xr % F, yr[0] % F), c[f"{name}_real_bcast"])
    assert np.array_equal(O.cyclic_real(p, xr % F, yr % F), c[f"{name}_real"])
    zr, zi = O.cyclic_complex(p, xr % F, xi % F, yr % F, yi % F)
    assert np.array_equal(zr, c[f"{name}_cplx_re"]) and np.array_equal(zi, c[f"{name}_cplx_im"])


def test_config1_direct_cyclic(golden, digests):
    """C1: bit-exact against direct cyclic convolution (BASELINE config 1) and
    the reference's full-size digest."""
    c = golden("convolution")
    p = O.Plan.named("cdc64")
    rng = np.random.default_rng(0)
    x = rng.integers(-16, 16, (16384, 64))
    h = rng.integers(-32, 32, (16384, 64))
    z = O.cyclic_real(p, x % p.F, h % p.F)
    assert sha(z) == digests["convolution"]["c1_cyclic_real"]
    assert np.array_equal(z[:256], c["c1_z_head"])
    # O(N^2) direct cyclic convolution mod F on a slice
    k = np.arange(64)
    for b in range(0, 16384, 4093):
        d = np.array([(x[b] * h[b][(m - k) % 64]).sum() % p.F for m in range(64)])
        assert np.array_equal(z[b], d)


def test_quantize(golden):
    q = golden("quantize")
    for tag, (bits, sc) in {"s5": (5, SIG_SCALE), "s6": (6, 128.0), "s8": (8, 8.0)}.items():
        for k in ("x", "ties", "exact", "special"):
            v, cnt = O.quantize_real(q[k], sc, (1 << (bits - 1)) - 1)
            assert np.array_equal(v, q[f"{tag}_{k}_q"]), (tag, k)
            assert cnt == int(q[f"{tag}_{k}_c"])


def test_cdc_c2_and_edges(golden, digests):
    a = golden("cdc")
    yr, yi = O.cdc_process_int(a["tap_re"], a["tap_im"], a["c2_xr"], a["c2_xi"])
    assert sha(yr) == digests["cdc"]["c2_yr"] and sha(yi) == digests["cdc"]["c2_yi"]
    dr, di = O.cdc_direct(a["tap_re"], a["tap_im"], a["c2_xr"], a["c2_xi"])
    assert np.array_equal(dr, yr) and np.array_equal(di, yi)
    for L in (0, 1, 2, 15, 16, 17, 31, 32, 33, 63, 64, 65, 97, 1000, 4097):
        r, i = O.cdc_process_int(a["tap_re"], a["tap_im"], a[f"len{L}_xr"], a[f"len{L}_xi"])
        assert np.array_equal(r, a[f"len{L}_yr"]) and np.array_equal(i, a[f"len{L}_yi"]), L
    for tag in ("sat", "wide"):
        r, i = O.cdc_process_int(a["tap_re"], a["tap_im"], a[f"{tag}_xr"], a[f"{tag}_xi"])
        assert np.array_equal(r, a[f"{tag}_yr"]) and np.array_equal(i, a[f"{tag}_yi"])
        r2, i2 = O.cdc_direct(a["tap_re"], a["tap_im"], a[f"{tag}_xr"], a[f"{tag}_xi"])
        assert np.array_equal(r2, r) and np.array_equal(i2, i)
    for tag in ("t33", "z0", "t17", "t1"):
        r, i = O.cdc_process_int(a[f"{tag}_tap_re"], a[f"{tag}_tap_im"], a[f"{tag}_xr"], a[f"{tag}_xi"])
        assert np.array_equal(r, a[f"{tag}_yr"]) and np.array_equal(i, a[f"{tag}_yi"]), tag


@pytest.mark.parametrize("tag", ["a", "b"])
def test_aeq_link_streams(golden, tag):
    g = golden("aeq")
    q = g[f"{tag}_q"].astype(np.int64)
    eq = O.Aeq(SIG_SCALE, mu=1e-4)
    y = eq.process(q, mu_blocks=O.mu_blocks(q.shape[1] // 16))
    assert np.array_equal(y, g[f"{tag}_y"])
    assert np.array_equal(eq.w, g[f"{tag}_w"])
    assert np.array_equal(eq.w_int, g[f"{tag}_wint"])
    assert np.array_equal(eq.history, g[f"{tag}_hist"])
    assert np.array_equal(np.array(eq.err_trace), g[f"{tag}_err"])
    assert eq.saturations == int(g[f"{tag}_sat"])


def test_aeq_saturating_and_streaming(golden):
    g = golden("aeq")
    eq = O.Aeq(SIG_SCALE, mu=0.05)
    y = eq.process(g["c_q"].astype(np.int64))
    assert np.array_equal(y, g["c_y"]) and np.array_equal(eq.w_int, g["c_wint"])
    assert eq.saturations == int(g["c_sat"]) > 0
    eq = O.Aeq(SIG_SCALE)
    y = eq.process(g["d_q"].astype(np.int64), adapt=False)
    assert np.array_equal(y, g["d_y"]) and eq.err_trace == []
    eq = O.Aeq(SIG_SCALE)
    sched = lambda i: 0.0 if (i // 16) % 5 == 3 else 3e-3  # noqa: E731
    q = g["e_q"].astype(np.int64)
    y1 = eq.process(q[:, :16 * 77], mu_blocks=[sched(16 * b) for b in range(77)])
    y2 = eq.process(q[:, 16 * 77:], mu_blocks=[sched(16 * b) for b in range(200 - 77)])
    assert np.array_equal(y1, g["e_y1"]) and np.array_equal(y2, g["e_y2"])
    assert np.array_equal(eq.w, g["e_w"]) and np.array_equal(np.array(eq.err_trace), g["e_err"])


def test_aeq_single_block_api(golden):
    g = golden("aeq")
    eq = O.Aeq(SIG_SCALE, mu=1e-4)
    y, xb = eq.equalize_block(g["f_x"])
    assert np.array_equal(y, g["f_y"]) and np.array_equal(xb, g["f_xblk"])
    eq.update_taps(xb, y, 0.01)
    assert np.array_equal(eq.w, g["f_w"])
    y2, xb2 = eq.equalize_block(np.zeros((4, 16), np.int64) + 0)
    assert xb2.shape == (4, 32)


def test_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(9)
    for n in (1, 7, 8, 9, 31, 32, 100, 128, 129, 1000, 4097, 1 << 16):
        a = rng.standard_normal(n)
        assert O.pairwise_sum(a) == float(np.add.reduce(a))


def test_oracle_aeq_nan_and_inf_step_size(golden):
    """A NaN and an inf mu block (reference fixture aeq_nan.npz): the float taps turn
    NaN / inf and the 14-bit taps clip to -16383 uncounted, as numpy's cast does."""
    g = golden("aeq_nan")
    oq = O.Aeq(SIG_SCALE, mu=1e-4)
    y = oq.process(g["x"], mu_blocks=g["mu"])
    assert np.array_equal(y, g["y"])
    assert np.array_equal(oq.w, g["w"], equal_nan=True)
    assert np.array_equal(oq.w_int, g["w_int"]) and oq.saturations == int(g["sat"])
    assert np.array_equal(np.array(oq.err_trace), g["err"], equal_nan=True)
