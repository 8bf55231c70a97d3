"""oracle/linkgen_np.py (numpy restatement of the reference's link model,
linksim.py:105-291) regenerates the reference's own quantized front-end samples
bit for bit: config 2 (both planes), config 3 at one SNR point and config-5 links,
against digests the unmodified reference produced (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import oracle.linkgen_np as G
from conftest import sha


def test_config2_inputs_match_reference(digests):
    _, _, _, fe = G.config2()
    xr, xi = fe[0]
    assert sha(np.asarray(xr).astype(np.int8)) == digests["cdc"]["c2_xr"]
    assert sha(np.asarray(xi).astype(np.int8)) == digests["cdc"]["c2_xi"]


@pytest.mark.parametrize("link", [0, 63])
def test_config5_inputs_match_reference(digests, link):
    _, _, _, fe = G.config5(link)
    q = np.stack([np.stack([xr, xi]) for xr, xi in fe]).astype(np.int8)
    assert sha(q) == digests["c5"][str(link)]["q_in"]


def test_config3_inputs_match_reference(digests):
    _, _, _, fe = G.config3(24.0)
    got = [sha(np.stack([a, b]).astype(np.int8)) for a, b in fe]
    assert got == digests["c3"]["24.0"]["q_in"]
