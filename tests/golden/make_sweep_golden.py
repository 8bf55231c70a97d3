"""Golden output of the reference CLI's `sweep` (cli.py:239-267) on a small link
config, for tests/test_cli.py::test_cli_sweep_matches_reference. Run in the build
container (needs /root/reference):

    python tests/golden/make_sweep_golden.py

The config is one whose every point the reference completes (its receiver rarely
converges -- SURVEY finding 4 -- and `sweep` raises on a BER of 0.5): 20 km,
2^16 symbols, SNR 15 and 22 dB, schemes fnt and float, seed 77. The CLI runs with
the working directory at a scratch dir and relative paths, because the manifest
digest and the summary line contain them."""

import json
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
INI = """[link]
n_symbols = 65536
z_km = 20.0
snr_db = 15.0,22.0
schemes = fnt,float
seed = 77
"""


def main():
    with tempfile.TemporaryDirectory() as d:
        Path(d, "link.ini").write_text(INI)
        r = subprocess.run([sys.executable, "-m", "fntdsp.cli", "sweep", "--config", "link.ini",
                            "--out-dir", "sweep_out"], cwd=d, capture_output=True, text=True,
                           env={"PYTHONPATH": "/root/reference/pkg/src", "PATH": "/usr/bin:/bin"})
        out = {"ini": INI, "argv": ["sweep", "--config", "link.ini", "--out-dir", "sweep_out"],
               "rc": r.returncode, "stdout": r.stdout,
               "csv": Path(d, "sweep_out", "sweep.csv").read_text(),
               "summary": Path(d, "sweep_out", "summary.txt").read_text()}
    (HERE / "sweep.json").write_text(json.dumps(out, indent=1))
    print(out["stdout"], out["csv"])


if __name__ == "__main__":
    main()
