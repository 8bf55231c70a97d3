"""LinkConfig.mu_schedule (linksim.py:82-83) as a GearSchedule: the same values as the
reference's lambda per symbol index, the vectorized per-block table FntAeq uses, and
the lambda's late binding to the config's fields."""

import numpy as np

import paper_2405_04253_b200 as P
from paper_2405_04253_b200.aeq import mu_block_array


def test_gear_schedule_matches_reference_lambda():
    cfg = P.LinkConfig(z_km=75.0)
    sch = cfg.mu_schedule()
    ref = lambda i: cfg.mu1 if i < cfg.gear_symbols else cfg.mu2  # noqa: E731 (linksim.py:83)
    for i in (0, 1, cfg.gear_symbols - 1, cfg.gear_symbols, 10 ** 7):
        assert sch(i) == ref(i)
    for nb in (0, 1, 1249, 1250, 1251, 16384):
        assert np.array_equal(mu_block_array(nb, 16, sch, 1.0),
                              np.array([float(ref(16 * b)) for b in range(nb)]))
    cfg.mu1, cfg.gear_symbols = 5e-3, 160          # the lambda reads the fields late
    assert sch(159) == 5e-3 and sch(160) == cfg.mu2
    assert np.array_equal(mu_block_array(12, 16, sch, 1.0), np.array([5e-3] * 10 + [cfg.mu2] * 2))
    cfg.mu2 = None                                  # non-numeric: per-block calls, config mu
    assert np.array_equal(mu_block_array(12, 16, sch, 7.0), np.array([5e-3] * 10 + [7.0] * 2))
