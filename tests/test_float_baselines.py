"""The float comparators (not on the FNT path) against the reference's own outputs
(tests/golden/float.npz): the per-symbol TD-AEQ kernel reproduces the reference's
numba kernel bit for bit; the GPU FD/TD CDC (cuFFT / conv1d, library code) agree
to float64 rounding."""

import numpy as np
import pytest

import paper_2405_04253_b200 as P


@pytest.mark.gpu
def test_td_aeq_float_matches_reference(golden):
    g = golden("float")
    cfg = P.LinkConfig()
    y, w = P.td_aeq_float(g["xa"], cfg.aeq_config(), mu_schedule=cfg.mu_schedule())
    assert np.array_equal(y, g["ya"]) and np.array_equal(w, g["wa"])


@pytest.mark.gpu
@pytest.mark.parametrize("fn,key", [("fd_cdc_float", "fd"), ("td_cdc_float", "td")])
def test_float_cdc_on_gpu_matches_reference(golden, fn, key):
    g = golden("float")
    cfg = P.LinkConfig(n_symbols=2 ** 18, z_km=75.0, snr_db=(20.0,), pol_rotation_deg=0.0,
                       dgd_symbols=0.0, iq_skew_samples=0.0, seed=1)
    y = getattr(P, fn)(g["x"], cfg.cdc_config("fnt"))
    ref = g[key]
    assert y.shape == ref.shape
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
