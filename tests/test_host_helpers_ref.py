"""The drop-in scalar helpers of fermat.py and the host-side pieces of fixedpoint.py
(budget, tap split, quantized blocks) against the unmodified reference, when it is
present (this build container; skipped elsewhere): values, dtypes, reprs and error
messages."""

import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2405_04253_b200 as P
from paper_2405_04253_b200 import fermat as PF

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not (REF / "fntdsp").is_dir(), reason="reference not present")


def err(f, *a):
    try:
        f(*a)
    except Exception as e:  # noqa: BLE001
        return (type(e).__name__, str(e))
    return None


def test_host_helpers_equal_reference():
    sys.path.insert(0, str(REF))
    try:
        import fntdsp.fermat as RF
        import fntdsp.fixedpoint as R
    finally:
        sys.path.remove(str(REF))
    rng = np.random.default_rng(0)

    w = rng.integers(-16383, 16384, 1000)
    a = P.split_taps(w); b = R.split_taps(w)
    assert np.array_equal(a.high, b.high) and np.array_equal(a.low, b.low) and np.array_equal(a.recombined(), b.recombined())
    assert a.high.dtype == b.high.dtype and a.recombined().dtype == b.recombined().dtype
    assert np.array_equal(P.recombine(a.high, a.low), R.recombine(b.high, b.low))
    for cm in (False, True):
        for mags in ([1,2,3], [0], [], rng.integers(-40,40,33)):
            x = P.check_overflow(mags, P.QuantSpec(5, 8.0), P.FermatParams(4), cm)
            y = R.check_overflow(mags, R.QuantSpec(5, 8.0), RF.FermatParams(4), cm)
            assert (x.bound, x.limit, x.passed, x.margin, str(x), repr(x)) == (y.bound, y.limit, y.passed, y.margin, str(y), repr(y)), (str(x), str(y))
    for bw in (2, 5, 6, 14, 31):
        assert P.QuantSpec(bw, 1.0).max_int == R.QuantSpec(bw, 1.0).max_int
    for bad in ((1, 1.0), (5, 0.0), (5, -1.0), (5, float('nan'))):
        assert err(P.QuantSpec, *bad) == err(R.QuantSpec, *bad), bad
    assert err(P.split_taps, [16384]) == err(R.split_taps, [16384])
    qb = P.QuantizedBlock(np.zeros(3), np.zeros(3), P.QuantSpec(5, 8.0), 2)
    rb = R.QuantizedBlock(np.zeros(3), np.zeros(3), R.QuantSpec(5, 8.0), 2)
    assert qb.clip_fraction == rb.clip_fraction and np.array_equal(P.dequantize(qb), R.dequantize(rb))
    qb1 = P.QuantizedBlock(np.arange(3), None, P.QuantSpec(5, 8.0)); rb1 = R.QuantizedBlock(np.arange(3), None, R.QuantSpec(5, 8.0))
    assert np.array_equal(P.dequantize(qb1), R.dequantize(rb1)) and qb1.clip_fraction == rb1.clip_fraction
    for t in range(5):
        p = PF.FermatParams(t); q = RF.FermatParams(t)
        assert (p.b, p.F, p.half) == (q.b, q.F, q.half)
        assert PF.for_modulus(p.F) == p and PF.for_modulus(float(p.F)) == p
        F = p.F
        for v in list(range(0, min(F*F, 5000), 7)) + [F*F-1, F*F-2, F-1, F]:
            if v < F * F: assert PF.reduce(v, p) == RF.reduce(v, q)
        vals = range(-5, F + 5) if F < 300 else [*range(-5, 300), *rng.integers(0, F, 1500).tolist(), F - 1, F, F + 1]
        for a_ in vals:
            for bb in range(-3, F+3, max(1, F//7)):
                assert PF.add(a_, bb, p) == RF.add(a_, bb, q) and PF.sub(a_, bb, p) == RF.sub(a_, bb, q)
            assert PF.neg(a_, p) == RF.neg(a_, q)
            if 0 <= a_ < F:
                assert PF.decode_signed(a_, p) == RF.decode_signed(a_, q)
                for s in range(-70, 70):
                    assert PF.mul_pow2(a_, s, p) == RF.mul_pow2(a_, s, q)
        for v in range(-p.half, p.half + 1, max(1, p.half // 50)):
            assert PF.encode_signed(v, p) == RF.encode_signed(v, q)
        assert err(PF.sqrt2, p) == err(RF.sqrt2, q)
        if p.b >= 4: assert PF.sqrt2(p) == RF.sqrt2(q)
    for bad in (5, -1):
        assert err(PF.FermatParams, bad) == err(RF.FermatParams, bad)
    for F in (65536, 7):
        assert err(PF.for_modulus, F) == err(RF.for_modulus, F)
    assert err(PF.encode_signed, 40000, PF.FermatParams(4)) == err(RF.encode_signed, 40000, RF.FermatParams(4))



def test_linksim_helpers_equal_reference():
    sys.path.insert(0, str(REF))
    try:
        import fntdsp.linksim as R
    finally:
        sys.path.remove(str(REF))
    import paper_2405_04253_b200.linksim as L
    rng = np.random.default_rng(1)
    for _ in range(1500):
        n = rng.integers(2, 8)
        snrs = rng.uniform(10, 25, n)
        bers = 10 ** rng.uniform(-6, -1, n)
        if rng.random() < 0.2:
            bers[rng.integers(0, n)] = 0.0
        if rng.random() < 0.1:
            bers[:] = 3.8e-3
        assert err(L.fec_crossing_snr, snrs, bers) == err(R.fec_crossing_snr, snrs, bers)
        try:
            assert L.fec_crossing_snr(snrs, bers) == R.fec_crossing_snr(snrs, bers)
        except ValueError:
            pass
    for ber in (0.0, -1.0, 1e-9, 1e-3, 0.2, 0.49, 0.5):
        assert err(L._q_factor_db, ber) == err(R._q_factor_db, ber)
        if 0 < ber < 0.5:
            assert L._q_factor_db(ber) == R._q_factor_db(ber)
    for bits in (3, 5, 8):
        for lf in (0.5, 0.8, 1.0):
            assert (L.LinkConfig(sig_bits=bits, load_fraction=lf).sig_scale
                    == R.LinkConfig(sig_bits=bits, load_fraction=lf).sig_scale)
    pts = list(zip((14, 16, 18, 20), (1e-2, 5e-3, 2e-3, 1e-4)))
    rows = [L.Metrics(s, x, y, 0, 0, 0, 0, 0, True) for s in ("fnt", "float") for x, y in pts]
    rrows = [R.Metrics(s, x, y, 0, 0, 0, 0, 0, True) for s in ("fnt", "float") for x, y in pts]
    assert L.penalty_at_fec(rows, "fnt", "float") == R.penalty_at_fec(rrows, "fnt", "float")


def test_cdc_aeq_host_helpers_equal_reference(tmp_path, monkeypatch):
    """Tap design, quantization scale, tap files, the RDE error and the MIMO tap
    object, bit for bit (quantize runs on the GPU in the product; the reference's numpy
    quantizer stands in for it here, its own parity is a GPU test)."""
    sys.path.insert(0, str(REF))
    try:
        import fntdsp.aeq as RA
        import fntdsp.cdc as RC
        import fntdsp.fixedpoint as RF
    finally:
        sys.path.remove(str(REF))
    import paper_2405_04253_b200.aeq as A
    import paper_2405_04253_b200.cdc as C
    monkeypatch.setattr(C, "quantize", lambda taps, spec: RF.quantize(taps, RF.QuantSpec(spec.bit_width, spec.scale)))
    for z in (0.0, 25.0, 75.0, 1000.0):
        for nt in (1, 5, 32, 33):
            for fs in (80e9, 64e9):
                a = C.CdcConfig(z_km=z, fs_hz=fs, n_taps=nt)
                b = RC.CdcConfig(z_km=z, fs_hz=fs, n_taps=nt)
                assert a.accumulated_dispersion == b.accumulated_dispersion
                assert C.required_taps(a) == RC.required_taps(b)
                ta, tb = C.design_cd_taps(a), RC.design_cd_taps(b)
                assert ta.dtype == tb.dtype and np.array_equal(ta.view(np.float64), tb.view(np.float64))
                if z:
                    qa, qb = C.quantize_taps(ta, 6), RC.quantize_taps(tb, 6)
                    assert all(np.array_equal(x, y) for x, y in zip(qa[:2], qb[:2])) and qa[2] == qb[2]
                    C.save_taps(tmp_path / "a", *qa)
                    RC.save_taps(tmp_path / "b", *qb)
                    assert (tmp_path / "a").read_text() == (tmp_path / "b").read_text()
                    la, lb = C.load_taps(tmp_path / "a"), RC.load_taps(tmp_path / "b")
                    assert all(np.array_equal(x, y) for x, y in zip(la[:2], lb[:2])) and la[2] == lb[2]
    rng = np.random.default_rng(3)
    radii = RA.qam16_radii()
    assert np.array_equal(A.qam16_radii(), radii)
    for _ in range(50):
        yi, yq = rng.normal(0, 1, (2, 4, 16))
        assert np.array_equal(A.rde_error(yi, yq, radii), RA.rde_error(yi, yq, radii))
    for l_taps, spike in ((16, 8192), (8, 100)):
        a, b = A.RvMimoTaps.center_spike(l_taps, spike), RA.RvMimoTaps.center_spike(l_taps, spike)
        assert all(np.array_equal(getattr(a, k), getattr(b, k)) for k in ("w_int", "high", "low"))
