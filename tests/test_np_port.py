"""Pin the numpy restatement used as the timed CPU baseline (oracle/np_port.py)
to the reference's golden fixtures, so the baseline measures the same work."""

import numpy as np

import oracle.np_port as N
from conftest import SIG_SCALE, sha


def test_np_transform_and_cdc(golden, digests):
    g = golden("transforms")
    assert np.array_equal(N.transform(N.CDC64, g["cdc64_x"]), g["cdc64_fnt"])
    assert np.array_equal(N.transform(N.AEQ32, g["aeq32_x"], True), g["aeq32_ifnt"])
    a = golden("cdc")
    bp, bm = N.cdc_spectra(a["tap_re"], a["tap_im"])
    assert np.array_equal(bp, a["b_plus"]) and np.array_equal(bm, a["b_minus"])
    yr, yi = N.cdc_process_int(a["c2_xr"].astype(np.int64), a["c2_xi"].astype(np.int64), bp, bm, 32)
    assert sha(yr) == digests["cdc"]["c2_yr"] and sha(yi) == digests["cdc"]["c2_yi"]


def test_np_aeq_and_chain(golden):
    g = golden("aeq")
    eq = N.NpAeq(SIG_SCALE)
    mu = np.where(np.arange(g["a_q"].shape[1] // 16) * 16 < 20000, 2e-3, 1e-4)
    y = eq.process(g["a_q"], mu_blocks=mu)
    assert np.array_equal(y, g["a_y"]) and np.array_equal(eq.w, g["a_w"])
    assert np.array_equal(np.array(eq.err_trace), g["a_err"])
    a = golden("cdc")
    q = g["b_cdc_q"].astype(np.int64)
    mu = np.where(np.arange(q.shape[-1] // 32) * 16 < 20000, 2e-3, 1e-4)
    y, eq = N.chain(q[:, 0], q[:, 1], a["tap_re"], a["tap_im"], 32, SIG_SCALE * 128.0, SIG_SCALE, mu)
    assert np.array_equal(y, g["b_y"])
