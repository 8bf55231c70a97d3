"""CPU restatement of the tensor-core (split-integer matrix) form of the FNT-CDC
(paper_2405_04253_b200/csrc/k_cdc.cu: k_cdc64_umma, k_cdc64_tc).

The kernel runs the 64-point forward FNT and the pruned inverse as int8 matrix
products on the tensor cores (mma.sync m16n8k32, exact int32 accumulation): every
matrix entry is a 64th root of unity mod F4 split into two 8-bit limbs, the
forward spectra are reduced mod F4 and multiplied by the tap spectra b+- on the
CUDA cores exactly like the reference (cdc.py:141-156), and the products are split
into two signed 8-bit limbs for the inverse. These tests restate that algorithm in
numpy (limb tables, accumulator bounds, the one residue two signed bytes cannot
hold and its correction) and check it bit-exactly against the oracle's shift-add
FNT path, which is pinned to the reference (tests/test_np_port.py)."""

import numpy as np

from oracle import np_port as npp

F = 65537
ALPHA = 4080                 # cdc64 root: sqrt(2) mod F4 (fnt.py, plan cdc64)
N = 64
HOP = 32
N_INV = pow(N, -1, F)
C_RE = F - (1 << 15)         # cdc.py:152-153
C_IM = F - (1 << 7)
W_OFF = 32896                # w = (u + 32896) mod F: s8 limbs are the bytes of w ^ 0x80


def limbs_u8s8(t):
    """Residue t -> (t1 in [0, 255], t0 in [-128, 127]) with 256 t1 + t0 == t mod F.
    256 t1 + t0 spans [-128, 65407]: every residue but 65408 (== -129), which is not
    a 64th root of unity, so every transform matrix entry has a representation."""
    t = np.asarray(t, dtype=np.int64) % F
    v = np.where(t > 65407, t - F, t)
    assert not np.any(v < -128), "residue 65408 has no (u8, s8) representation"
    t0 = ((v + 128) & 255) - 128
    t1 = (v - t0) >> 8
    assert t1.min() >= 0 and t1.max() <= 255 and t0.min() >= -128 and t0.max() <= 127
    return t1, t0


def root_table():
    return np.array([pow(ALPHA, e, F) for e in range(N)], dtype=np.int64)


E_RE, E_IM = 50, 34          # c_re N^-1 = alpha^50, c_im N^-1 = alpha^34 (checked below)


def forward_matrix():
    """T[k, n] = alpha^(nk): the forward FNT-64 of one real plane (fnt.py:106-109)."""
    k = np.arange(N)[:, None]
    n = np.arange(N)[None, :]
    return root_table()[(n * k) % N]


def inverse_matrices():
    """M_re[m, k], M_im[m, k] for the kept outputs m in [32, 64):
    z_re = c_re IFNT(s), z_im = c_im IFNT(d) with s = u+ + u-, d = u+ - u- (cdc.py:152-155)."""
    m = np.arange(HOP, N)[:, None]
    k = np.arange(N)[None, :]
    R = root_table()
    return R[(E_RE - m * k) % N], R[(E_IM - m * k) % N]


def roots():
    return set(root_table().tolist())


def tap_betas(bp, bm):
    """Per-bin constants of the transform-domain combination: with A+- = X_r +- 2^8 X_i
    (cdc.py:148-149), s = A+ b+ + A- b- = X_r beta1 + X_i beta2 and
    d = A+ b+ - A- b- = X_r beta3 + X_i beta4."""
    bp = np.asarray(bp, dtype=np.int64)
    bm = np.asarray(bm, dtype=np.int64)
    return ((bp + bm) % F, 256 * (bp - bm) % F, (bp - bm) % F, 256 * (bp + bm) % F)


def split_s8(w):
    """w = (value + 32896) mod F in [0, 65536] -> signed bytes (v1, v0) = bytes of w ^ 0x80,
    256 v1 + v0 == value, except w == 65536 (bytes wrap: represents value + 1)."""
    v0 = ((w & 255) ^ 0x80).astype(np.int64)
    v1 = (((w >> 8) & 255) ^ 0x80).astype(np.int64)
    return np.where(v1 >= 128, v1 - 256, v1), np.where(v0 >= 128, v0 - 256, v0), w == 65536


def tc_blocks(win_r, win_i, bp, bm, stats=None):
    """Split-integer matrix form of cdc.py:141-156 for windows (B, 64) of int8 samples,
    as k_cdc64_umma and k_cdc64_tc compute it. Returns decoded (z_re, z_im) (B, 32) of the kept outputs."""
    xr = np.asarray(win_r, dtype=np.int64)
    xi = np.asarray(win_i, dtype=np.int64)
    t1, t0 = limbs_u8s8(forward_matrix())
    P1r, P0r = xr @ t1.T, xr @ t0.T                                     # s8 x u8, s8 x s8
    P1i, P0i = xi @ t1.T, xi @ t0.T
    for P in (P1r, P0r, P1i, P0i):
        assert np.abs(P).max() <= 64 * 128 * 255
    Xr = 256 * P1r + P0r                                                # FNT(x_r) mod F
    Xi = 256 * P1i + P0i
    assert np.abs(Xr).max() < 2 ** 30 and np.abs(Xi).max() < 2 ** 30
    b1, b2, b3, b4 = tap_betas(bp, bm)
    S = Xr * b1 + Xi * b2                                               # 64-bit (IMAD.WIDE) sums
    D = Xr * b3 + Xi * b4
    assert np.abs(S).max() < 2 ** 47 and np.abs(D).max() < 2 ** 47
    ws = (S + W_OFF) % F
    wd = (D + W_OFF) % F
    s1, s0, fs = split_s8(ws)
    d1, d0, fd = split_s8(wd)
    if stats is not None:
        stats["flagged"] = stats.get("flagged", 0) + int(fs.sum() + fd.sum())
    Mre, Mim = inverse_matrices()
    out = []
    for v1, v0, flag, M in ((s1, s0, fs, Mre), (d1, d0, fd, Mim)):
        i1, i0 = limbs_u8s8(M)
        Q11 = v1 @ i1.T
        Qmid = v1 @ i0.T + v0 @ i1.T
        Q00 = v0 @ i0.T
        z = 256 * Qmid + Q00 - Q11                                      # 65536 == -1 mod F
        assert np.abs(z).max() < 2 ** 30
        z = z - flag.astype(np.int64) @ M.T                             # flagged bins carried value + 1
        r = z % F
        out.append(np.where(r <= (F - 1) // 2, r, r - F))               # decode_signed (fermat.py:131-133)
    return out[0], out[1]


def tc_process_int(xr, xi, bp, bm, n_taps, stats=None):
    L = len(xr)
    nb = -(-(L + HOP) // HOP)
    pad = np.zeros((2, HOP + nb * HOP + HOP), dtype=np.int64)
    pad[0, HOP:HOP + L] = xr
    pad[1, HOP:HOP + L] = xi
    win = np.lib.stride_tricks.sliding_window_view(pad, N, axis=1)[:, ::HOP][:, :nb]
    zr, zi = tc_blocks(win[0], win[1], bp, bm, stats)
    c = n_taps // 2
    return zr.reshape(-1)[c:c + L], zi.reshape(-1)[c:c + L]


def test_matrix_entries_are_roots_with_limbs():
    R = roots()
    assert len(R) == N
    assert (C_RE * N_INV) % F == pow(ALPHA, E_RE, F) and (C_IM * N_INV) % F == pow(ALPHA, E_IM, F)
    assert set(np.unique(forward_matrix()).tolist()) <= R
    for M in inverse_matrices():
        assert set(np.unique(M).tolist()) <= R
    # every root has a (u8, s8) limb pair; s8 x s8 and u8 x u8 would each miss one
    limbs_u8s8(np.array(sorted(R)))
    assert pow(ALPHA, 7, F) == 32640 and 32768 in R and F - 1 in R


def test_tc_form_matches_shift_add_fnt_cdc():
    rng = np.random.default_rng(11)
    taps_r = rng.integers(-31, 32, 32)
    taps_i = rng.integers(-31, 32, 32)
    bp, bm = npp.cdc_spectra(taps_r, taps_i)
    for lo, hi, L in ((-16, 16, 5000), (-128, 128, 3001)):
        xr = rng.integers(lo, hi, L)
        xi = rng.integers(lo, hi, L)
        st = {}
        got = tc_process_int(xr, xi, bp, bm, 32, st)
        want = npp.cdc_process_int(xr, xi, bp, bm, 32)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_unrepresentable_residue_is_corrected():
    """Force s[k] == 32640 (w = 65536, the one residue two signed bytes cannot hold) on
    many bins and check the corrected output against the shift-add path."""
    rng = np.random.default_rng(5)
    B = 64
    win_r = rng.integers(-128, 128, (B, N))
    win_i = rng.integers(-128, 128, (B, N))
    T = forward_matrix()
    Xr0 = (win_r[0] @ T.T) % F
    Xi0 = (win_i[0] @ T.T) % F
    # b- = 0 and b+ chosen so that s = A+ b+ = 32640 on block 0 wherever A+ != 0
    Ap = (Xr0 + 256 * Xi0) % F
    bp = np.array([32640 * pow(int(a), -1, F) % F if a else 1 for a in Ap], dtype=np.int64)
    bm = np.zeros(N, dtype=np.int64)
    st = {}
    zr, zi = tc_blocks(win_r, win_i, bp, bm, st)
    assert st["flagged"] >= N - 1
    Xr = npp.transform(npp.CDC64, npp._enc(win_r, F))
    Xi = npp.transform(npp.CDC64, npp._enc(win_i, F))
    up = (((Xr + 256 * Xi) % F) * bp) % F
    um = (((Xr - 256 * Xi) % F) * bm) % F
    wr = npp._dec((npp.transform(npp.CDC64, (up + um) % F, True) * C_RE) % F, F)[:, HOP:]
    wi = npp._dec((npp.transform(npp.CDC64, (up - um) % F, True) * C_IM) % F, F)[:, HOP:]
    assert np.array_equal(zr, wr) and np.array_equal(zi, wi)


def test_tc_form_extreme_windows():
    """Windows at the int8 extremes (all -128, all 127, alternating) and the largest tap
    spectra: the accumulator bounds asserted inside tc_blocks hold at the worst case and
    the outputs still match the shift-add FNT path."""
    rng = np.random.default_rng(23)
    bp = rng.integers(0, F, N)
    bm = rng.integers(0, F, N)
    bp[:4] = F - 1
    bm[:4] = 32768
    wins = [np.full(N, -128), np.full(N, 127), np.where(np.arange(N) % 2, 127, -128),
            np.where(np.arange(N) < 32, -128, 127)]
    win_r = np.array([w for w in wins for _ in wins])
    win_i = np.array([v for _ in wins for v in wins])
    zr, zi = tc_blocks(win_r, win_i, bp, bm)
    Xr = npp.transform(npp.CDC64, npp._enc(win_r, F))
    Xi = npp.transform(npp.CDC64, npp._enc(win_i, F))
    up = (((Xr + 256 * Xi) % F) * bp) % F
    um = (((Xr - 256 * Xi) % F) * bm) % F
    wr = npp._dec((npp.transform(npp.CDC64, (up + um) % F, True) * C_RE) % F, F)[:, HOP:]
    wi = npp._dec((npp.transform(npp.CDC64, (up - um) % F, True) * C_IM) % F, F)[:, HOP:]
    assert np.array_equal(zr, wr) and np.array_equal(zi, wi)
