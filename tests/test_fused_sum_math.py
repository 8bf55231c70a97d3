"""CPU checks of the arithmetic behind the FNT-AEQ's transform-domain stream sum
(paper_2405_04253_b200/csrc/k_aeq.cu: pack_taps, fused_ok, fused_forward).

The kernel sums the four input streams' products before the inverse transform
only when an exact range test passes; these tests restate the identities it
relies on in numpy and check them exhaustively or on random worst cases. The GPU
parity tests (tests/test_gpu_parity.py) check the kernel itself."""

import numpy as np

F4 = 65537
W_MAX = 16383  # TAP_MAG_MAX (aeq.py:26)


def pack_bal(w):
    """k_aeq.cu pack_taps<true>: p = w 2^16 - a (2^22 - 1), a = (w + 32) >> 6."""
    w = np.asarray(w, dtype=np.int64)
    a = (w + 32) >> 6
    return ((w * 65536 - a * 4194303) & 0xFFFFFFFF).astype(np.uint32)


def unpack_group(p, g):
    """k_aeq.cu unpack_group: g = 0 -> low half sign-extended, 1 -> (p + 2^15) >> 16."""
    p = np.asarray(p, dtype=np.uint32).astype(np.int64)
    if g == 0:
        lo = p & 0xFFFF
        return np.where(lo >= 0x8000, lo - 0x10000, lo)
    v = (p + 0x8000) & 0xFFFFFFFF
    v = np.where(v >= 1 << 31, v - (1 << 32), v)
    return v >> 16


def ref_groups(w):
    """split_taps (fixedpoint.py:111-121): sign * (|w| >> 7), sign * (|w| & 127)."""
    w = np.asarray(w, dtype=np.int64)
    s = np.sign(w)
    m = np.abs(w)
    return s * (m >> 7), s * (m & 127)


def dec(r):
    """decode_signed (fermat.py:130-133) of a residue mod F4."""
    r = np.mod(r, F4)
    return np.where(r > 32768, r - F4, r)


def test_balanced_digits_all_taps():
    w = np.arange(-W_MAX, W_MAX + 1)
    p = pack_bal(w)
    a, b = unpack_group(p, 0), unpack_group(p, 1)
    assert np.array_equal(64 * a + b, w)
    assert b.min() == -32 and b.max() == 31
    assert np.abs(a).max() == 256
    hi, lo = ref_groups(w)
    assert np.array_equal(128 * hi + lo, w) and np.abs(hi).max() == 127 and np.abs(lo).max() == 127


def _conv_valid(taps, xb):
    """Outputs 16..31 of the 32-point cyclic convolution of 16 taps with a 32-sample
    window: y[m] = sum_k taps[k] x[16 + m - k] (aeq.py:118-144, probe t15)."""
    return np.array([sum(int(taps[k]) * int(xb[16 + m - k]) for k in range(16)) for m in range(16)])


def test_stream_sum_equals_reference_decode_under_the_range_test():
    """With max|x| <= 16 and the digit-mass bound, 64 dec(sum_t conv a) +
    dec(sum_t conv b) equals the reference's sum over t of 128 dec(conv hi) +
    dec(conv lo) -- including adversarial taps near the bound."""
    rng = np.random.default_rng(3)
    for trial in range(60):
        if trial % 3 == 0:  # large taps: the a-digit mass near its limit
            w = rng.integers(-W_MAX, W_MAX + 1, (4, 16))
            w[:, rng.random(16) < 0.8] //= 64
        else:
            w = rng.integers(-3000, 3001, (4, 16))
        x = rng.integers(-16, 17, (4, 32))
        amax = int(np.abs(x).max())
        a = (w + 32) >> 6
        b = w - 64 * a
        fused_ok = amax <= 16 and int(np.abs(a).sum()) * amax <= 32768
        hi, lo = ref_groups(w)
        ref = sum(128 * dec(_conv_valid(hi[t], x[t])) + dec(_conv_valid(lo[t], x[t])) for t in range(4))
        exact = sum(_conv_valid(w[t], x[t]) for t in range(4))
        assert np.array_equal(ref, exact)  # condition (1): the reference decodes are exact
        if fused_ok:
            ya = sum(_conv_valid(a[t], x[t]) for t in range(4))
            yb = sum(_conv_valid(b[t], x[t]) for t in range(4))
            assert np.abs(yb).max() <= 32768 and np.abs(ya).max() <= 32768
            assert np.array_equal(64 * dec(ya) + dec(yb), ref)


def test_range_test_is_needed():
    """Without the bound the stream sum can wrap mod F4 where the reference's
    per-stream decodes do not (why the kernel keeps the reference form as fallback)."""
    w = np.full((4, 16), 64 * 256 - 1)  # a = 256, b = -1
    x = np.full((4, 32), 16)
    a = (w + 32) >> 6
    ya = sum(_conv_valid(a[t], x[t]) for t in range(4))
    assert np.abs(ya).max() > 32768
    assert not np.array_equal(dec(ya), ya)
