"""bench.py contract smoke tests on the GPU box: one JSON line with the required
keys at N=1, and the torchrun multi-rank path (2 ranks sharing the single GPU,
FNT_BENCH_BACKEND=gloo for the rank reductions) exits 0 with rank 0 printing."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches"}


def _json_line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--links", "128", "--symbols", "32768", "--steps", "1",
                        "--warmup", "1", "--no-cpu", "--no-sub"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["roofline"]["frac"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] == 4 and d["parity"]["all_equal"]
    assert d["e2e"]["dropin_api"]["value"] > 0
    assert d["link_quality"]["links"] == 128


@pytest.mark.slow
def test_bench_torchrun_two_ranks():
    env = dict(os.environ, FNT_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
           "--links", "64", "--symbols", "32768", "--steps", "1", "--warmup", "1", "--no-cpu",
           "--no-e2e", "--no-alt", "--no-sub"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    # the 64 links are split 32 + 32 (strong scaling); rank 0 checked its links vs the oracle
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["links_per_gpu"] == 32 and d["config"]["links_total"] == 64
    assert d["link_quality"]["links"] == 64  # both ranks' links, reduced over the group
    assert d["parity"]["all_equal"]
