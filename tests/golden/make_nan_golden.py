"""Golden AEQ run of the unmodified reference with a NaN and an inf step size
(aeq.py:148-170: the float taps become NaN / inf, numpy casts rint(NaN) to INT64_MIN,
which is not counted and clips to -16383). Run in the build container:

    python tests/golden/make_nan_golden.py
"""

import sys
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import fntdsp  # noqa: E402

HERE = Path(__file__).resolve().parent
SIG = 8.94427190999916


def main():
    warnings.simplefilter("ignore")
    rng = np.random.default_rng(5)
    x = rng.integers(-15, 16, (4, 16 * 40))
    mu = np.full(40, 2e-3)
    mu[7] = np.nan
    mu[20] = np.inf
    eq = fntdsp.FntAeq(fntdsp.AeqConfig(mu=1e-4, sig_spec=fntdsp.QuantSpec(5, SIG)))
    y = eq.process(x, adapt=True, mu_schedule=lambda i: mu[i // 16])
    np.savez_compressed(HERE / "aeq_nan.npz", x=x, mu=mu, y=y, w=eq.w, w_int=eq.taps.w_int,
                        sat=eq.saturations, err=np.array(eq.err_trace))
    print("saturations", eq.saturations, "w_int[0,0,:4]", eq.taps.w_int[0, 0, :4])


if __name__ == "__main__":
    main()
