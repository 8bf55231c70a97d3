#!/usr/bin/env python3
"""FNT-CDC + FNT-AEQ throughput on B200 (BASELINE.json metric).

Headline workload (default): BASELINE config 5 -- 4096 independent dual-pol
PDM-16QAM links of 2^18 symbols at 2 sps (L = 2^19 complex samples per
polarization), 75 km, per-link Haar Jones rotation and SNR ~ U[16, 22] dB,
generated on device (paper_2405_04253_b200.linkgen; Philox streams keyed by
global link index, so every shard holds the same links at any GPU count;
statistically equivalent to the reference generator, not bitwise). Under
torchrun the 4096 links are split across ranks (sharding.link_shards: 512 per
GPU at N = 8) -- strong scaling, no collective on the data path (NCCL only
reduces the timing maximum and the sample count).

One step = the whole receiver chain over the rank's links with inputs resident
in HBM: FNT-CDC on both polarizations (fused requantization + exact decimation
statistics) -> decimation phase (with its tie guard) -> adaptive FNT-AEQ (fresh
state per link, LinkConfig gear-shift mu schedule). Inputs (8.6 GB at N = 1)
exceed L2 (126 MB), so no L2 flush is needed between steps.

Metric: Gsamples/s = complex samples per polarization, summed over
polarizations and links, per second (whole job, all ranks).

Also in the line (each measured here, on the same box):
  roofline   dominant kernel against the measured INT32 peak, SURVEY 8(d) op
             convention (AEQ: 23872 ALG INT ops per 16-symbol block; the
             tap-spectrum refresh, 15360 ops per block, reported separately)
  parity     2 of the timed links re-run through the CPU oracle, bit-exact
  e2e        all of the rank's links through the host-buffer chain
             (stream.HostChain, 512-link slabs, H2D + D2H every step) and the
             reference-style per-link drop-in API (numpy in / out)
  c4, c1, c3 BASELINE configs 4 (2^31-sample CDC), 1 (API-path convolution) and
             the per-stream latency regime of config 3 (6 links x 2^20 symbols)
  cpu_baseline  the reference algorithm (oracle/np_port, pinned to the
             reference's outputs) on the box's host cores, bounded sample

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "FNT-CDC+AEQ Gsamples/s"
UNIT = "Gsamples/s"
PROFILES = ROOT / "profiles"

# Algorithmic work per unit (SURVEY 8(d) convention): radix-2 butterfly = 6 INT ops,
# general residue product = 6, modular aux op = 2, plain add/shift = 1.
CDC_INT_OPS_PER_BLOCK = 4 * 192 * 6 + 128 * 6 + 256 * 2     # 5888 per 64-block = 184 / sample
CDC_TC_MACS_PER_BLOCK = 2 * 2 * 64 * 64 + 2 * 4 * 32 * 64      # int8 MACs per block, matrix forms
# AEQ per 16-symbol block: 4 FNT-32 + 32 IFNT-32 (2880 butterflies) + 1024 products + 448 plain
AEQ_INT_OPS_PER_BLOCK = (4 + 32) * 80 * 6 + 1024 * 6 + 448     # 23872
AEQ_TAP_REFRESH_OPS_PER_BLOCK = 32 * 80 * 6                    # 15360: 32 tap-spectrum FNT-32s
AEQ_INT_OPS_PER_BLOCK_DIRECT = 2 * 4096 + 448                  # 8640 (exact time-domain MIMO FIR)
AEQ_FP64_OPS_PER_BLOCK = 2 * 4096 + 256 * 4 + 64 * 2 + 32 * 12  # gradient + update + y + rde ~ 9728
C1_OPS_PER_ELEMENT = 60                                        # 3 FNT-64 + products, per element


def allreduce(vals, op: str) -> list:
    """Reduce floats over ranks (device tensors under NCCL, CPU tensors under gloo)."""
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.tolist()


def measured_peaks() -> dict:
    peaks = {}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        peaks.update(json.loads(p.read_text()))
    q = PROFILES / "int_peaks_r01.json"
    if q.exists():
        d = json.loads(q.read_text())
        peaks["int_tops"] = d["mixed_iadd_imad"]["Tinst_per_s"]
        peaks["fp64_tinst"] = d["fp64_dadd"]["Tinst_per_s"]
        peaks["int_source"] = "measured: profiles/int_peaks_r01.json (tools/int_peaks.cu)"
    else:
        peaks["int_tops"] = 36.0
        peaks["fp64_tinst"] = 18.3
        peaks["int_source"] = "fallback constants"
    peaks.setdefault("hbm_gbs", 6650.0)
    return peaks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU side

def _cpu_task(args):
    """One config-5 link through the numpy restatement of the reference chain
    (np_port.chain). The link's inputs are the reference's own link model
    (oracle/linkgen_np.config5, bit-identical to linksim.py's generator) at the
    sample's symbol count; only the chain is timed."""
    link, n_sym, tap_re, tap_im, n_taps, out_scale, sig_scale, mu = args
    import oracle.linkgen_np as G
    import oracle.np_port as N
    _, _, _, fe = G.config5(link, n_symbols=n_sym)
    xr2 = np.stack([fe[0][0], fe[1][0]])
    xi2 = np.stack([fe[0][1], fe[1][1]])
    t0 = time.perf_counter()
    N.chain(xr2, xi2, tap_re, tap_im, n_taps, out_scale, sig_scale, mu)
    return time.perf_counter() - t0


def run_cpu_baseline(engine, cfg, n_sym: int, cores: int, rounds: int | None = None,
                     seconds: float = 20.0) -> dict:
    """Time the reference algorithm (numpy port) on all host cores: one config-5
    link of n_sym symbols per task, one process per core, ~`seconds` of wall time."""
    from concurrent.futures import ProcessPoolExecutor
    import oracle.np_port  # noqa: F401  (checker / baseline only)
    hop = 16
    nb = n_sym // hop
    mu = np.where(np.arange(nb) * hop < cfg.gear_symbols, cfg.mu1, cfg.mu2)
    mk = lambda i: (i, n_sym, engine.tap_re, engine.tap_im, cfg.n_cdc_taps,  # noqa: E731
                    engine.output_scale, cfg.sig_scale, mu)
    with ProcessPoolExecutor(max_workers=cores) as ex:
        list(ex.map(_cpu_task, [mk(i) for i in range(cores)]))  # warm the workers' imports
        busy, r = 0.0, 0
        t0 = time.perf_counter()
        # rounds of one link per core until ~20 s of wall time (or the requested count)
        while (r < rounds) if rounds is not None else (time.perf_counter() - t0 < seconds and r < 400):
            busy += sum(ex.map(_cpu_task, [mk(cores * (r + 1) + i) for i in range(cores)]))
            r += 1
        rounds = r
        wall = time.perf_counter() - t0
    # samples / (chain time per core) with all cores busy; the per-link input
    # generation (the reference's numpy link model) is not part of the timed chain
    n_samples = rounds * cores * 2 * (2 * n_sym)
    value = n_samples / (busy / cores) / 1e9
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"{rounds * cores} config-5 links (reference link model, oracle/linkgen_np) x "
                       f"2 pols x {2 * n_sym} samples (2^{int(math.log2(n_sym))} symbols) through "
                       f"oracle/np_port.chain (numpy restatement of the reference's CDC -> glue -> "
                       f"AEQ, pinned to reference fixtures; calibration against the unmodified "
                       f"reference in profiles/port_calibration_r02.json), one process per core, "
                       f"{wall:.1f} s wall"),
            "wall_s": wall}


def impl_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = _link_cfg(args)
    cores = os.cpu_count() or 1
    eng = _HostEngine(cfg)
    n_sym = args.cpu_symbols
    if args.config == "c4":
        import oracle.np_port as N
        eng._b_plus, eng._b_minus = N.cdc_spectra(eng.tap_re, eng.tap_im)
        t0 = time.perf_counter()
        vals = [run_cpu_cdc_baseline(eng, 1 << 20, cores) for _ in range(args.steps)]
        wall = time.perf_counter() - t0
        v = float(np.mean([x["value"] for x in vals]))
        print(json.dumps({
            "impl": "reference", "metric": "FNT-CDC Gsamples/s (config 4)", "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": "C4 throughput-scale FNT-CDC, CPU sample: %d streams x 2^20 "
                                   "samples per round" % cores},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}))
        return
    for _ in range(args.warmup and 1):
        run_cpu_baseline(eng, cfg, n_sym, cores, rounds=1)
    # each step a bounded sample: the whole --steps K run stays within ~2 minutes
    per_step = max(3.0, 120.0 / max(args.steps, 1))
    t0 = time.perf_counter()
    vals = [run_cpu_baseline(eng, cfg, n_sym, cores, seconds=per_step) for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    v = float(np.mean([x["value"] for x in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic (the reference's link model, oracle/linkgen_np config 5)",
        "config": {"workload": ("C5 many-channel FNT-CDC+FNT-AEQ, CPU sample: config-5 links "
                                "(75 km, Haar Jones, SNR U[16,22] dB) of 2^%d symbols, one link per "
                                "core per round, ~20 s per step" % int(math.log2(n_sym))),
                   "symbols_per_link": n_sym, "samples_per_pol": 2 * n_sym,
                   "cores": cores, "full_config_links": args.links,
                   "note": "throughput per sample is independent of the link count and length "
                           "(the per-link work is linear in the samples): the same metric"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": ("the reference is pure numpy (no native build); its algorithm is timed through "
                 "oracle/np_port.py, a numpy restatement pinned to the reference's golden outputs "
                 "and calibrated against the unmodified reference on the same link "
                 "(profiles/port_calibration_r02.json)"),
    }
    print(json.dumps(line))


class _HostEngine:
    """Tap constants computed on the host exactly as FntCdcEngine does, for the
    CPU-only reference arm (no GPU needed)."""

    def __init__(self, cfg):
        from paper_2405_04253_b200.cdc import design_cd_taps
        import oracle
        c = cfg.cdc_config("fnt")
        taps = design_cd_taps(c)
        max_int = (1 << (c.tap_bits - 1)) - 1
        peak = max(np.abs(taps.real).max(), np.abs(taps.imag).max())
        scale = 2.0 ** math.floor(math.log2(max_int / peak))
        self.tap_re, _ = oracle.quantize_real(taps.real, scale, max_int)
        self.tap_im, _ = oracle.quantize_real(taps.imag, scale, max_int)
        self.tap_scale = scale
        self.output_scale = cfg.sig_scale * scale


def _cdc_cpu_task(args):
    xr, xi, bp, bm = args
    import oracle.np_port as N
    t0 = time.perf_counter()
    N.cdc_process_int(xr, xi, bp, bm, 32)
    return time.perf_counter() - t0


def run_cpu_cdc_baseline(eng, n: int, cores: int) -> dict:
    """Reference-algorithm CDC (numpy restatement) on all host cores, ~20 s of CPU
    work, on 5-bit front-end samples of the reference's link model."""
    from concurrent.futures import ProcessPoolExecutor
    import oracle.linkgen_np as G
    _, _, _, fe = G.config5(0, n_symbols=n // 2)
    xr, xi = fe[0]
    tasks = [(xr, xi, eng._b_plus, eng._b_minus) for _ in range(cores)]
    with ProcessPoolExecutor(max_workers=cores) as ex:
        per = max(ex.map(_cdc_cpu_task, tasks))
        rounds = max(1, int(round(20.0 / max(per * cores, 1e-3))))
        t0 = time.perf_counter()
        for _ in range(rounds):
            list(ex.map(_cdc_cpu_task, tasks))
        wall = time.perf_counter() - t0
    return {"value": rounds * cores * n / wall / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"{rounds * cores} streams x {n} complex samples (reference link model) "
                       f"through oracle/np_port.cdc_process_int (numpy restatement of the "
                       f"reference's FntCdcEngine.process_int), one process per core, "
                       f"{wall:.1f} s wall")}


# ------------------------------------------------------------------ GPU side

def _link_cfg(args):
    from paper_2405_04253_b200.linksim import LinkConfig
    return LinkConfig(n_symbols=args.symbols, z_km=75.0, pol_rotation_deg=0.0, dgd_symbols=0.0,
                      iq_skew_samples=0.0, seed=4)


def _sync_all(world):
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()


def _config_dict(args, world, n_local, first):
    return {"workload": ("C5 many-channel FNT-CDC+FNT-AEQ: %d dual-pol PDM-16QAM links x 2^%d "
                         "symbols x 2 sps split over %d GPU(s), 75 km SSMF, Haar Jones, SNR "
                         "U[16,22] dB, 5-bit I/Q, 6-bit CDC taps (N=64 sqrt2 FNT), 4x4 FNT-AEQ "
                         "(N=32) gear-shift mu")
                        % (args.links, int(math.log2(args.symbols)), world),
            "links_total": args.links, "links_per_gpu": n_local, "rank0_links": [first, n_local],
            "symbols": args.symbols, "samples_per_pol": 2 * args.symbols,
            "aeq_forward": args.forward, "aeq_kernel": args.aeq_kernel,
            "cdc_kernel": {"tc": "k_cdc64_tc (mma.sync split-integer FNT)",
                           "umma": "k_cdc64_umma (tcgen05 split-integer FNT)",
                           "shift": "k_cdc64 (shift-add butterflies)"}.get(
                               args.cdc_kernel, "auto (k_cdc64, shift-add butterflies)"),
            "parallelism": f"links sharded over {world} GPU(s) (sharding.link_shards), no collective",
            "l2": "inputs (int8 I/Q, %.1f GB/GPU) exceed the 126 MB L2; no flush needed"
                  % (4 * n_local * 2 * args.symbols / 1e9)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--links", type=int, default=4096, help="config-5 links in the whole job")
    ap.add_argument("--symbols", type=int, default=1 << 18)
    ap.add_argument("--forward", default="fnt", choices=["fnt", "direct"])
    ap.add_argument("--cpu-symbols", type=int, default=1 << 13)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the c4 / c1 / c3 sub-objects")
    ap.add_argument("--config", default="c5", choices=["c5", "c4"],
                    help="c5: many-channel CDC+AEQ chain (headline); c4: throughput-scale CDC")
    ap.add_argument("--c4-samples", type=int, default=1 << 31, help="C4 samples per polarization")
    ap.add_argument("--no-alt", action="store_true", help="skip the direct-forward / layout / CDC-kernel A/B")
    ap.add_argument("--no-quality", action="store_true", help="skip the on-device BER/EVM scoring")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timing oracle check")
    ap.add_argument("--aeq-kernel", default="auto", choices=["auto", "warp", "pol"],
                    help="FNT-AEQ stream layout: one warp per stream, two warps per stream (one per "
                         "polarization), or auto (the split form below 4 streams per SM)")
    ap.add_argument("--cdc-kernel", default="auto", choices=["auto", "umma", "tc", "shift"],
                    help="FNT-CDC kernel: auto (shift-add butterflies), or the split-integer matrix "
                         "form on tcgen05 (umma) / mma.sync (tc)")
    args = ap.parse_args()
    if args.impl == "reference":
        impl_reference(args)
        return

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; FNT_BENCH_BACKEND=gloo lets several ranks share a GPU for a
    # functional smoke test of the multi-rank path (reductions on CPU tensors)
    backend = os.environ.get("FNT_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2405_04253_b200 import cdc as cdc_mod
    from paper_2405_04253_b200 import aeq as aeq_mod
    cdc_mod.set_cdc_kernel(args.cdc_kernel)
    aeq_mod.set_aeq_kernel(args.aeq_kernel)

    if args.config == "c4":
        line = run_c4(args, world, rank, local)
    else:
        line = run_c5(args, world, rank, local)
        if not args.no_sub:
            torch.cuda.empty_cache()
            line["c4"] = run_c4(args, world, rank, local, sub=True)
            torch.cuda.empty_cache()
            if world == 1:
                line["c1"] = run_c1(args)
                line["c3"] = run_c3(args)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


AEQ_KERNEL_NAMES = {"warp": "k_aeq_process", "pol": "k_aeq_pol"}
AEQ_POL_AUTO_PER_SM = 4  # k_aeq.cu use_pol_kernel


def _aeq_layout(args, n_streams: int) -> str:
    """The AEQ stream layout fntgpu_aeq_process runs (k_aeq.cu use_pol_kernel)."""
    if args.aeq_kernel != "auto":
        return args.aeq_kernel
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return "pol" if n_streams < AEQ_POL_AUTO_PER_SM * sms else "warp"


def _ncu_traffic(name: str, world: int, full_size: bool):
    """Per-launch DRAM bytes (ncu --set full) of the committed capture, when it was
    taken at this configuration; else None."""
    path = PROFILES / name
    if world != 1 or not full_size or not path.exists():
        return None
    try:
        return json.loads(path.read_text()).get("per_launch_dram_bytes", {})
    except Exception:
        return None


def run_c5(args, world, rank, local) -> dict:
    import torch
    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200 import _lib
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.sharding import link_shards
    from paper_2405_04253_b200.stream import CdcAeqChain, decimation_phase

    cfg = _link_cfg(args)
    fwd = _lib.AEQ_FWD_DIRECT if args.forward == "direct" else _lib.AEQ_FWD_FNT
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    L = 2 * args.symbols
    first, n_local = link_shards(args.links, world)[rank]
    gen = DeviceLinkGenerator(args.symbols, z_km=cfg.z_km, sig_scale=cfg.sig_scale)
    xr, xi, sidx = gen.generate(n_local, seed=4, first_link=first, symbols=True)
    chain = CdcAeqChain(eng, cfg.aeq_config(), n_local, L, cfg.sig_spec(), cfg.mu_schedule(),
                        forward=fwd)
    torch.cuda.synchronize()

    ev = []

    def step(record: bool):
        s = torch.cuda.current_stream()
        if not record:
            chain.run(xr, xi)
            return
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        chain.aeq.reset()
        chain.acc.zero_()
        e[0].record(s)
        chain.cdc.run(xr, xi, length=L, qr=chain.qr, qi=chain.qi, q_spec=chain.sig_spec,
                      decim_acc=chain.acc)
        e[1].record(s)
        decimation_phase(chain.acc, chain.n_links, L, chain.phase, chain.gap)
        chain.check_ties(xr, xi)  # tie guard (a small device-to-host read each step)
        e[2].record(s)
        chain.aeq.run_decim(chain.qr, chain.qi, chain.phase, chain.n_blocks, chain.y,
                            adapt=True, mu_blocks=chain.mu_blocks, err=chain.err)
        e[3].record(s)
        ev.append(e)

    for _ in range(args.warmup):
        step(False)
    _sync_all(world)
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    _sync_all(world)
    t_start.record()
    for _ in range(args.steps):
        step(True)
    t_end.record()
    _sync_all(world)
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    cdc_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    ph_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    aeq_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    samples_rank = args.steps * n_local * 2 * L
    if world > 1:
        ms_max = allreduce([ms], "max")[0]
        samples_all = allreduce([float(samples_rank)], "sum")[0]
    else:
        ms_max, samples_all = ms, float(samples_rank)
    value = samples_all / (ms_max * 1e-3) / 1e9
    ok = bool(torch.isfinite(chain.y).all().item())

    peaks = measured_peaks()
    cdc_name = {"tc": "k_cdc64_tc", "umma": "k_cdc64_umma"}.get(args.cdc_kernel, "k_cdc64")
    aeq_name = (AEQ_KERNEL_NAMES[_aeq_layout(args, n_local)] if fwd == _lib.AEQ_FWD_FNT
                else "k_aeq_process")
    n_blk_cdc = 2 * n_local * (L // 32 + 1)
    n_blk_aeq = n_local * chain.n_blocks
    cdc_tops = n_blk_cdc * CDC_INT_OPS_PER_BLOCK / (cdc_ms * 1e-3) / 1e12
    aeq_int = AEQ_INT_OPS_PER_BLOCK if fwd == _lib.AEQ_FWD_FNT else AEQ_INT_OPS_PER_BLOCK_DIRECT
    aeq_tops = n_blk_aeq * aeq_int / (aeq_ms * 1e-3) / 1e12
    refresh_tops = (n_blk_aeq * AEQ_TAP_REFRESH_OPS_PER_BLOCK / (aeq_ms * 1e-3) / 1e12
                    if fwd == _lib.AEQ_FWD_FNT else 0.0)
    aeq_fp64 = n_blk_aeq * AEQ_FP64_OPS_PER_BLOCK / (aeq_ms * 1e-3) / 1e12
    cdc_bytes = 2 * n_local * L * (2 + 2)  # int8 I/Q in, int8 requantized I/Q out
    aeq_bytes = n_local * (4 * 32 * chain.n_blocks + 4 * 16 * chain.n_blocks * 8 + 8 * chain.n_blocks)
    traffic = _ncu_traffic("ncu_summary_r02.json", world, n_local == 4096)
    kernels = {
        cdc_name: {"ms": cdc_ms, "bound": "int", "achieved": cdc_tops, "peak": peaks["int_tops"],
                   "unit": "Tops/s", "frac": cdc_tops / peaks["int_tops"],
                   "alg_ops_per_launch": n_blk_cdc * CDC_INT_OPS_PER_BLOCK,
                   "hbm_gbs": cdc_bytes / (cdc_ms * 1e-3) / 1e9},
        aeq_name: {"ms": aeq_ms, "bound": "int", "achieved": aeq_tops, "peak": peaks["int_tops"],
                   "unit": "Tops/s", "frac": aeq_tops / peaks["int_tops"],
                   "alg_ops_per_block": aeq_int, "alg_ops_per_launch": n_blk_aeq * aeq_int,
                   "convention": ("SURVEY 8(d): 4 FNT-32 + 32 IFNT-32 + 1024 products + 448 plain "
                                  "= 23872 ALG INT ops per 16-symbol block" if fwd == _lib.AEQ_FWD_FNT
                                  else "exact time-domain FIR: 8640 ALG INT ops per block"),
                   "tap_refresh": {"alg_ops_per_block": AEQ_TAP_REFRESH_OPS_PER_BLOCK,
                                   "achieved": refresh_tops, "unit": "Tops/s",
                                   "note": "32 tap-spectrum FNT-32s per block (the taps change "
                                           "every adapting block), outside the 8(d) numerator"},
                   "with_refresh_frac": (aeq_tops + refresh_tops) / peaks["int_tops"],
                   "fp64": {"achieved": aeq_fp64, "unit": "T FP64 inst/s", "peak": peaks["fp64_tinst"],
                            "frac": aeq_fp64 / peaks["fp64_tinst"],
                            "ops_per_block": AEQ_FP64_OPS_PER_BLOCK},
                   "int_plus_fp64_issue_frac": ((aeq_tops + refresh_tops) / peaks["int_tops"]
                                                + aeq_fp64 / peaks["fp64_tinst"]),
                   "block_us": aeq_ms * 1e3 / chain.n_blocks,
                   "hbm_gbs": aeq_bytes / (aeq_ms * 1e-3) / 1e9},
        "k_decim_phase": {"ms": ph_ms, "note": "incl. the tie guard's device-to-host read"},
    }
    if cdc_name != "k_cdc64":
        tmacs = n_blk_cdc * CDC_TC_MACS_PER_BLOCK / (cdc_ms * 1e-3)
        int8_peak = 2.0 * peaks.get("bf16_tflops", 2250.0)
        kernels[cdc_name]["tensor"] = {"achieved": 2.0 * tmacs / 1e12, "peak": int8_peak,
                                       "unit": "Tops/s (int8)", "frac": 2.0 * tmacs / 1e12 / int8_peak}
    dom = aeq_name if aeq_ms >= cdc_ms else cdc_name
    kd = kernels[dom]
    roofline = {"bound": kd["bound"], "kernel": dom, "achieved": kd["achieved"], "peak": kd["peak"],
                "unit": kd["unit"], "frac": kd["frac"],
                "traffic": traffic.get(dom) if traffic else None,
                "traffic_note": ("ncu dram read+write bytes per launch, profiles/ncu_summary_r02.json"
                                 if traffic else "no ncu capture at this shard size"),
                "peak_source": peaks["int_source"],
                "step_share": kd["ms"] / (cdc_ms + ph_ms + aeq_ms),
                "kernels": kernels,
                "hbm": {"achieved_gbs": (cdc_bytes + aeq_bytes) / ((cdc_ms + aeq_ms) * 1e-3) / 1e9,
                        "peak_gbs": peaks["hbm_gbs"]}}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32 (Z/(2^32-1) residues) + f64",
        "data": "synthetic (on-device 16QAM link model, Philox streams keyed by global link index)",
        "config": _config_dict(args, world, n_local, first),
        "roofline": roofline, "clocks": clk, "gpu_launches": 4 * args.steps,
        "outputs_finite": ok, "tie_guard_resolved": len(chain.resolved),
    }

    if not args.no_parity and rank == 0:
        line["parity"] = c5_parity(chain, xr, xi, eng, cfg, sorted({0, n_local - 1}))

    if not args.no_alt:
        line["pipelined"] = run_pipelined(args, eng, cfg, xr, xi, fwd, world, n_local, samples_all,
                                          chain)

    if not args.no_quality:
        from paper_2405_04253_b200 import metrology as M
        bers, evms, oks = [], [], []
        for c0 in range(0, n_local, 32):
            c1 = min(n_local, c0 + 32)
            sym, bits = gen.tx_reference(sidx[c0:c1])
            b, e, o = M.align_and_count(M.aeq_to_pols(chain.y[c0:c1]), sym, bits,
                                        cfg.discard_symbols)
            bers.append(b)
            evms.append(e)
            oks.append(o)
        bers, evms, oks = np.concatenate(bers), np.concatenate(evms), np.concatenate(oks)
        # whole-job figures: the ranks' sums and minimum gathered over the process
        # group (results only, after the timed region -- the one collective besides the
        # timing maximum)
        tot = [float(bers.sum()), float(bers.size), float(evms[oks].sum()), float(oks.sum())]
        low = [-float(bers.min())]
        if world > 1:
            tot, low = allreduce(tot, "sum"), allreduce(low, "max")
        line["link_quality"] = {
            "links": int(tot[1]), "ber_mean": tot[0] / tot[1], "ber_min": -low[0],
            "evm_db_mean": tot[2] / tot[3] if tot[3] else None,
            "aligned_fraction": tot[3] / tot[1],
            "note": "BER/EVM of every link of the job computed on the GPU (metrology."
                    "align_and_count; per-rank sums reduced over the process group); high BER "
                    "at 75 km reproduces the reference's behaviour (SURVEY finding 4)"}

    if not args.no_alt:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)

        def timed_steps():
            chain.run(xr, xi)
            _sync_all(world)
            ev.clear()
            a.record()
            for _ in range(args.steps):
                step(True)
            b.record()
            torch.cuda.synchronize()
            ms_ = a.elapsed_time(b)
            return allreduce([ms_], "max")[0] if world > 1 else ms_

        if fwd == _lib.AEQ_FWD_FNT:
            # the exact-equivalent time-domain forward (same bits) on the same resident data
            chain.aeq.prm.forward = _lib.AEQ_FWD_DIRECT
            ms_alt = timed_steps()
            line["aeq_forward_direct"] = {
                "value": samples_all / (ms_alt * 1e-3) / 1e9, "unit": UNIT,
                "ms_per_step": ms_alt / args.steps,
                "aeq_ms": float(np.mean([e[2].elapsed_time(e[3]) for e in ev])),
                "note": "same chain with the AEQ forward as an exact time-domain integer FIR "
                        "(bit-identical outputs, tests/test_gpu_parity.py); headline uses the FNT forward"}
            chain.aeq.prm.forward = _lib.AEQ_FWD_FNT
            # the other AEQ stream layout on the same data
            other = "k_aeq_process" if aeq_name == "k_aeq_pol" else "k_aeq_pol"
            chain.aeq.prm.kernel = 1 if other == "k_aeq_process" else 2
            ms_o = timed_steps()
            line["aeq_layouts"] = {
                aeq_name + "_ms": aeq_ms,
                other + "_ms": float(np.mean([e[2].elapsed_time(e[3]) for e in ev])),
                "other_value": samples_all / (ms_o * 1e-3) / 1e9,
                "note": "k_aeq_process: one warp per stream (throughput form); k_aeq_pol: two warps "
                        "per stream, one per polarization (latency form); identical outputs"}
            chain.aeq.prm.kernel = 0
        line["cdc_kernels"] = time_cdc_kernels(
            lambda: chain.cdc.run(xr, xi, length=L, qr=chain.qr, qi=chain.qi,
                                  q_spec=chain.sig_spec, decim_acc=chain.acc),
            args.steps, world)

    if not args.no_e2e:
        y_dev = chain.y
        del chain
        torch.cuda.empty_cache()
        line["e2e"] = run_e2e(args, eng, cfg, xr, xi, fwd, world, n_local)
        del y_dev
        if rank == 0:
            line["e2e"]["dropin_api"] = run_dropin(eng, cfg, xr, xi,
                                                   threads=min(16, os.cpu_count() or 1))

    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = run_cpu_baseline(eng, cfg, args.cpu_symbols, os.cpu_count() or 1)
    return line


def run_pipelined(args, eng, cfg, xr, xi, fwd, world, n_local, samples_all, chain) -> dict:
    """The same K steps as a steady-state pipeline (stream.PipelinedChain): step k + 1's
    CDC + decimation phase on its own CUDA stream overlapping step k's AEQ, two sets
    of intermediate buffers; each step is still the whole chain over every link.
    The outputs of the last step are compared with the plain chain's."""
    import torch
    from paper_2405_04253_b200.stream import PipelinedChain
    L = 2 * args.symbols
    pc = PipelinedChain(eng, cfg.aeq_config(), n_local, L, cfg.sig_spec(), cfg.mu_schedule(),
                        forward=fwd)
    for _ in range(max(2, args.warmup)):
        pc(xr, xi)
    pc.join()
    _sync_all(world)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        pc(xr, xi)
    pc.join()
    b.record()
    _sync_all(world)
    ms = a.elapsed_time(b)
    if world > 1:
        ms = allreduce([ms], "max")[0]
    same = bool(torch.equal(pc.y, chain.y) and torch.equal(pc.err, chain.err))
    del pc
    return {"value": samples_all / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms / args.steps,
            "outputs_equal_plain_chain": same,
            "how": "stream.PipelinedChain: CDC + phase of step k+1 (own CUDA stream) overlapping the "
                   "AEQ of step k (high-priority stream), double-buffered requantized planes; "
                   "timed over the same K steps, first CDC and last AEQ included"}


def c5_parity(chain, xr, xi, eng, cfg, links) -> dict:
    """Bench-data parity: links of the timed run (their on-device generated inputs)
    through the CPU oracle of the whole chain, compared bit-exactly with the GPU's
    phase, AEQ outputs and err_trace of the last timed step."""
    import oracle as O
    t0 = time.perf_counter()
    res = {}
    for l in links:
        fe = [(xr[2 * l + p].cpu().numpy().astype(np.int64), xi[2 * l + p].cpu().numpy().astype(np.int64))
              for p in range(2)]
        ph, y, oq = O.chain_link(eng.tap_re, eng.tap_im, eng.output_scale, cfg.sig_scale, fe,
                                 cfg.mu1, cfg.mu2, cfg.gear_symbols)
        res[str(l)] = bool(int(chain.phase[l].item()) == ph
                           and np.array_equal(chain.y[l].cpu().numpy(), y)
                           and np.array_equal(chain.err[l].cpu().numpy(), np.array(oq.err_trace)))
    return {"links": res, "all_equal": all(res.values()), "wall_s": time.perf_counter() - t0,
            "how": "oracle.chain_link (C restatement of process_int, decimation phase, quantize_real, "
                   "FntAeq; pinned to reference fixtures) on the links' timed inputs"}


def time_cdc_kernels(run, reps: int, world: int) -> dict:
    """Device time of one CDC launch with each kernel (shift-add butterflies and the
    tensor-core matrix forms), on the launching stream, max over ranks."""
    import torch
    from paper_2405_04253_b200 import cdc as cdc_mod
    out = {}
    prev = cdc_mod.set_cdc_kernel("shift")
    try:
        for name in ("shift", "umma", "tc"):
            cdc_mod.set_cdc_kernel(name)
            run()
            torch.cuda.synchronize()
            s = torch.cuda.current_stream()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(reps):
                run()
            b.record(s)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            if world > 1:
                ms = allreduce([ms], "max")[0]
            out[name + "_ms"] = ms
    finally:
        cdc_mod.set_cdc_kernel(prev)
    out["speedup_tc"] = out["shift_ms"] / out["tc_ms"]
    out["speedup_umma"] = out["shift_ms"] / out["umma_ms"]
    out["note"] = ("k_cdc64: radix-sqrt2 shift-add butterflies (auto); k_cdc64_umma / k_cdc64_tc: "
                   "forward FNT-64 and pruned inverse as split-integer int8 matrix products on "
                   "tcgen05 (UTCIMMA, TMEM accumulators) / mma.sync (IMMA.16832). Bit-identical "
                   "outputs (tests/test_gpu_parity.py)")
    return out


def run_e2e(args, eng, cfg, xr, xi, fwd, world, n_local) -> dict:
    """End to end through the host-buffer chain: every one of the rank's links per
    step, pinned host int8 I/Q -> H2D -> CDC -> phase -> AEQ -> D2H float64 y +
    err_trace, in 512-link slabs (stream.HostChain; each slab's outputs land in the
    chain's pinned output buffer, which the next slab reuses)."""
    import torch
    from paper_2405_04253_b200.stream import HostChain
    L = 2 * args.symbols
    slab = min(512, n_local)
    hx_r = torch.empty((2 * n_local, L), dtype=torch.int8, pin_memory=True)
    hx_i = torch.empty((2 * n_local, L), dtype=torch.int8, pin_memory=True)
    hx_r.copy_(xr)
    hx_i.copy_(xi)
    slabs = [(a, min(n_local, a + slab)) for a in range(0, n_local, slab)]
    chains = {slab: HostChain(eng, cfg.aeq_config(), slab, L, cfg.sig_spec(), cfg.mu_schedule(),
                              forward=fwd)}
    last = slabs[-1][1] - slabs[-1][0]
    if last not in chains:  # a short last slab runs through its own chain
        chains[last] = HostChain(eng, cfg.aeq_config(), last, L, cfg.sig_spec(), cfg.mu_schedule(),
                                 forward=fwd)

    def one_step():
        for a, b in slabs:
            chains[b - a](hx_r[2 * a:2 * b], hx_i[2 * a:2 * b])

    def join():
        for h in chains.values():
            h.join()

    one_step()
    join()
    _sync_all(world)
    steps = max(1, min(args.steps, 3))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        one_step()
    join()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        ms = allreduce([ms], "max")[0]
    samples = steps * args.links * 2 * L
    h2d = sum(chains[b_ - a_].h2d_bytes for a_, b_ in slabs)
    d2h = sum(chains[b_ - a_].d2h_bytes for a_, b_ in slabs)
    del chains, hx_r, hx_i
    # the PCIe roofline of this box: a pinned 1 GiB device-to-host copy
    pin = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    pin.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(4):
        pin.copy_(dev, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    d2h_peak = 4 * (1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9
    del pin, dev
    d2h_gbs = d2h / (ms / steps * 1e-3) / 1e9
    return {"value": samples / (ms * 1e-3) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": ms / steps, "steps": steps, "links_per_gpu": n_local,
            "pcie": {"d2h_gbs": d2h_gbs, "d2h_peak_gbs": d2h_peak, "frac": d2h_gbs / d2h_peak,
                     "note": "the step moves the float64 outputs back over PCIe; peak = pinned 1 GiB "
                             "device-to-host copy measured in this run (H2D runs concurrently)"},
            "path": "paper_2405_04253_b200.stream.HostChain over every link of the job in %d-link "
                    "slabs: pinned host int8 I/Q -> H2D -> CDC -> phase -> AEQ -> D2H float64 y + "
                    "err_trace, every step; copies pipelined with the kernels over 3 CUDA streams"
                    % slab}


def run_dropin(eng, cfg, xr, xi, n_links: int = 2, threads: int = 0) -> dict:
    """The reference-facing drop-in API on numpy arrays, one link after another, as a
    reference user calls it (cdc.py:165-180, linksim.py:249-308, aeq.py:172-190):
    FntCdcEngine.process on both polarizations, the decimation phase and the
    requantization of the decimated I/Q (quantize_real), FntAeq.process."""
    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200.stream import reference_phase
    L = xr.shape[1]
    n_data = max(n_links, 3 * threads)
    data = [[(xr[2 * l + p].cpu().numpy().astype(np.int64), xi[2 * l + p].cpu().numpy().astype(np.int64))
             for p in range(2)] for l in range(n_data)]
    spec = cfg.sig_spec()

    def one(fe):
        streams = [eng.process(a, b) for a, b in fe]
        ph = reference_phase(streams)
        dec = [s[ph::2] for s in streams]
        q = np.stack([P.quantize_real(v, spec)[0] for v in (dec[0].real, dec[0].imag,
                                                            dec[1].real, dec[1].imag)])
        eq = P.FntAeq(cfg.aeq_config())
        return eq.process(q, adapt=True, mu_schedule=cfg.mu_schedule())

    one(data[0])  # warm-up (plans, allocations)
    t0 = time.perf_counter()
    for fe in data[:n_links]:
        one(fe)
    wall = time.perf_counter() - t0
    out = {"value": n_links * 2 * L / wall / 1e9, "unit": UNIT, "links": n_links,
           "ms_per_link": 1e3 * wall / n_links,
           "path": "FntCdcEngine.process x 2 pols -> decimation phase -> quantize_real -> "
                   "FntAeq.process (numpy in / out, one link at a time; each call moves its "
                   "arrays over PCIe)"}
    if threads > 1:
        # the same per-link calls from `threads` host threads, one engine per thread
        # (the reference's threading convention): each thread's calls run on its own
        # CUDA stream (_lib.api_stream), so the links' latency-bound AEQs overlap
        from concurrent.futures import ThreadPoolExecutor
        local = threading.local()

        def work(fe):
            if not hasattr(local, "eng"):
                local.eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
            streams = [local.eng.process(a, b) for a, b in fe]
            ph = reference_phase(streams)
            dec = [s[ph::2] for s in streams]
            q = np.stack([P.quantize_real(v, spec)[0] for v in (dec[0].real, dec[0].imag,
                                                                dec[1].real, dec[1].imag)])
            eq = P.FntAeq(cfg.aeq_config())
            return eq.process(q, adapt=True, mu_schedule=cfg.mu_schedule())

        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(work, data[:threads]))  # warm-up: per-thread streams, engines
            t0 = time.perf_counter()
            list(ex.map(work, data))
            wall_t = time.perf_counter() - t0
        out["threads"] = {"value": len(data) * 2 * L / wall_t / 1e9, "unit": UNIT,
                          "links": len(data), "threads": threads,
                          "ms_per_link": 1e3 * wall_t / len(data),
                          "path": "the same calls from a thread pool, one CDC engine and one "
                                  "FntAeq per link per thread, per-thread CUDA streams"}
    return out


# ------------------------------------------------------------------ config 4

def run_c4(args, world, rank, local, sub: bool = False) -> dict:
    """BASELINE config 4: one dual-pol stream of 2^31 complex samples per
    polarization, FNT-CDC range-sharded across ranks (strong scaling) with the
    overlap-save halo read from each rank's input window (sharding.py); no
    data-path collective. Inputs are generated on device in independent 2^22-sample
    segments, each keyed by its GLOBAL segment index, so a rank's window holds the
    same samples at any GPU count."""
    import torch
    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.sharding import cdc_range_shards
    from paper_2405_04253_b200.stream import CdcBank, HostCdc

    cfg = P.LinkConfig(z_km=75.0, seed=3)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    bank = CdcBank(eng)
    L = args.c4_samples
    sh = cdc_range_shards(L, world, n_taps=cfg.n_cdc_taps)[rank]
    xr, xi = c4_window(sh.x_first, sh.x_count, cfg.sig_scale)
    yr = torch.empty((2, sh.out_count), dtype=torch.int16, device="cuda")
    yi = torch.empty_like(yr)
    torch.cuda.synchronize()

    def step():
        bank.run(xr, xi, length=L, x_first=sh.x_first, out_first=sh.out_first,
                 out_count=sh.out_count, yr=yr, yi=yi)

    for _ in range(args.warmup):
        step()
    _sync_all(world)
    clocks = ClockSampler(local)
    clocks.start()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step()
    b.record()
    _sync_all(world)
    clk = clocks.stop()
    ms = a.elapsed_time(b)
    ms_max = allreduce([ms], "max")[0] if world > 1 else ms
    samples = 2 * L  # both polarizations of the whole stream, all ranks
    value = args.steps * samples / (ms_max * 1e-3) / 1e9
    peaks = measured_peaks()
    per_launch_ms = ms / args.steps
    n_blocks = 2 * (sh.out_count // 32 + 2)
    achieved = n_blocks * CDC_INT_OPS_PER_BLOCK / (per_launch_ms * 1e-3) / 1e12
    hbm_bytes = 2 * sh.x_count * 2 + 2 * sh.out_count * 4  # int8 I/Q in, int16 I/Q out
    hbm_gbs = hbm_bytes / (per_launch_ms * 1e-3) / 1e9
    kname = {"tc": "k_cdc64_tc", "umma": "k_cdc64_umma"}.get(args.cdc_kernel, "k_cdc64")
    tr = _ncu_traffic("ncu_summary_r02_c4.json", world, L == 1 << 31)
    line = {
        "metric": "FNT-CDC Gsamples/s (config 4)", "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32 (Z/(2^32-1) residues)", "data": "synthetic (on-device 16QAM link model)",
        "config": {"workload": "C4 throughput-scale FNT-CDC: one dual-pol stream of %d complex "
                               "samples per pol, 75 km taps, range-sharded over %d GPU(s) with the "
                               "overlap-save halo" % (L, world),
                   "samples_per_pol": L, "shard_out": [sh.out_first, sh.out_count],
                   "cdc_kernel": kname,
                   "l2": "inputs (%.1f GB) exceed L2" % (hbm_bytes / 1e9)},
        "roofline": {"bound": "int", "kernel": kname, "achieved": achieved,
                     "peak": peaks["int_tops"], "unit": "Tops/s",
                     "frac": achieved / peaks["int_tops"],
                     "traffic": tr.get(kname) if tr else None,
                     "peak_source": peaks["int_source"],
                     "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks["hbm_gbs"],
                             "frac": hbm_gbs / peaks["hbm_gbs"]}},
        "clocks": clk, "gpu_launches": args.steps,
    }
    if not args.no_alt:
        line["cdc_kernels"] = time_cdc_kernels(step, args.steps, world)
    if not args.no_e2e:
        # host buffers through the C ABI: pinned int8 I/Q -> H2D -> CDC -> D2H int16 I/Q
        n = min(1 << 28, sh.out_count)
        hc = HostCdc(eng, 2, n)
        hx = torch.empty((2, n), dtype=torch.int8, pin_memory=True)
        hy = torch.empty((2, n), dtype=torch.int8, pin_memory=True)
        hx.copy_(xr[:, :n])
        hy.copy_(xi[:, :n])
        hc(hx, hy)
        hc.join()
        _sync_all(world)
        a.record()
        for _ in range(args.steps):
            hc(hx, hy)
        hc.join()
        b.record()
        torch.cuda.synchronize()
        ms_e = a.elapsed_time(b)
        if world > 1:
            ms_e = allreduce([ms_e], "max")[0]
        line["e2e"] = {"value": args.steps * 2 * n * world / (ms_e * 1e-3) / 1e9, "unit": UNIT,
                       "h2d_bytes_per_step": hc.h2d_bytes, "d2h_bytes_per_step": hc.d2h_bytes,
                       "path": "stream.HostCdc: pinned host int8 I/Q -> H2D -> fntgpu_cdc64_process "
                               "-> D2H int16 I/Q, %d samples x 2 pols per call, copies pipelined "
                               "with the range-sharded CDC over 3 CUDA streams" % n}
        del hc, hx, hy
    line["f64_input"] = c4_f64_variant(args, bank, eng, xr, xi, sh, L, world, peaks)
    if not sub and rank == 0 and world == 1 and not args.no_cpu:
        import oracle.np_port as N
        eng._b_plus, eng._b_minus = N.cdc_spectra(eng.tap_re, eng.tap_im)
        line["cpu_baseline"] = run_cpu_cdc_baseline(eng, 1 << 20, os.cpu_count() or 1)
    del xr, xi, yr, yi
    return line


def c4_f64_variant(args, bank, eng, xr, xi, sh, L, world, peaks) -> dict:
    """The CDC with float64 front-end samples quantized on load (in_dtype F64,
    fixedpoint.py:51-60 fused into the staging): 16 B of float64 I/Q in + 4 B of int16
    I/Q out per complex sample (SURVEY 8(d)'s 20 B/sample row), on the first 2^28
    samples per polarization of this rank's window. The floats are the window's
    5-bit samples plus uniform dither within +-0.45 LSB, divided by the signal scale
    (they quantize back to the same integers; the clip count is checked)."""
    import torch
    n = min(1 << 28, sh.x_count)
    g = torch.Generator(device="cuda").manual_seed(11)
    sc = float(eng.sig_spec.scale)
    fr = (xr[:, :n].double() + (torch.rand((2, n), generator=g, device="cuda", dtype=torch.float64) - 0.5) * 0.9) / sc
    fi = (xi[:, :n].double() + (torch.rand((2, n), generator=g, device="cuda", dtype=torch.float64) - 0.5) * 0.9) / sc
    out_n = max(0, min(n - 128, sh.out_count))  # inside the provided window with its halo
    yr = torch.empty((2, out_n), dtype=torch.int16, device="cuda")
    yi = torch.empty_like(yr)
    clip = torch.zeros(1, dtype=torch.int64, device="cuda")

    def step():
        bank.run(fr, fi, length=L, x_first=sh.x_first, out_first=sh.out_first, out_count=out_n,
                 yr=yr, yi=yi, in_spec=eng.sig_spec, in_clipped=clip)

    for _ in range(args.warmup):
        step()
    _sync_all(world)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    # the same range from the int8 planes gives the same outputs
    rr = torch.empty_like(yr)
    ri = torch.empty_like(yi)
    bank.run(xr[:, :n], xi[:, :n], length=L, x_first=sh.x_first, out_first=sh.out_first,
             out_count=out_n, yr=rr, yi=ri)
    same = bool(torch.equal(rr, yr) and torch.equal(ri, yi))
    n_blocks = 2 * (out_n // 32 + 2)
    tops = n_blocks * CDC_INT_OPS_PER_BLOCK / (ms * 1e-3) / 1e12
    byts = 2 * out_n * 20
    del fr, fi, yr, yi, rr, ri
    return {"value": 2 * out_n / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_launch": ms,
            "samples_per_pol": out_n, "alg_bytes_per_sample": 20,
            "hbm_gbs": byts / (ms * 1e-3) / 1e9, "hbm_frac": byts / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "int_tops": tops, "int_frac": tops / peaks["int_tops"],
            "equals_int8_path": same, "clip_count": int(clip.item()),
            "kernel": "k_cdc64_f64p (persistent; raw float64 windows prefetched by TMA, quantized on load from shared memory; shift-add butterflies)"}


def c4_window(x_first: int, x_count: int, sig_scale: float, seg: int = 1 << 22):
    """Samples [x_first, x_first + x_count) of the config-4 stream: independent
    2^22-sample link segments, segment j drawn from the Philox stream keyed by
    (seed 3, j) -- the same samples whatever range a rank owns."""
    import torch
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    s_lo, s_hi = x_first // seg, -(-(x_first + x_count) // seg)
    gen = DeviceLinkGenerator(seg // 2, z_km=75.0, sig_scale=sig_scale)
    xr = torch.empty((2, x_count), dtype=torch.int8, device="cuda")
    xi = torch.empty_like(xr)
    per = 8  # segments per generator group (keyed by the group's global index)
    for g0 in range(s_lo - s_lo % per, s_hi, per):
        g1 = min(s_hi, g0 + per)
        gr, gi = gen.generate(g1 - g0, seed=3, first_link=g0, chunk=per)
        gr = gr.view(g1 - g0, 2, seg).transpose(0, 1).reshape(2, (g1 - g0) * seg)
        gi = gi.view(g1 - g0, 2, seg).transpose(0, 1).reshape(2, (g1 - g0) * seg)
        a = max(g0 * seg, x_first)
        b = min(g1 * seg, x_first + x_count)
        xr[:, a - x_first:b - x_first] = gr[:, a - g0 * seg:b - g0 * seg]
        xi[:, a - x_first:b - x_first] = gi[:, a - g0 * seg:b - g0 * seg]
        del gr, gi
    return xr, xi


# ------------------------------------------------------------------ config 1 / 3

def run_c1(args) -> dict:
    """BASELINE config 1: 16384 blocks of 64 (5-bit signal, 6-bit per-block taps)
    through cyclic_convolve_real (cdc64 plan). Two numbers: the drop-in API call on
    numpy int64 arrays (host copies included, what a reference user calls) and the
    same kernel on device-resident buffers through the C ABI (looped, CUDA events)."""
    import torch
    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200 import _lib
    plan = P.default_plans()["cdc64"]
    rng = np.random.default_rng(0)
    x = rng.integers(-16, 16, (16384, 64))
    h = rng.integers(-32, 32, (16384, 64))
    z = P.cyclic_convolve_real(plan, P.encode_signed_array(x, plan.params),
                               P.encode_signed_array(h, plan.params))
    import oracle as O  # checker: the pinned C restatement
    ok = bool(np.array_equal(z, O.cyclic_real(O.Plan.named("cdc64"), x % 65537, h % 65537)))
    xe, he = P.encode_signed_array(x, plan.params), P.encode_signed_array(h, plan.params)
    reps = 50
    t0 = time.perf_counter()
    for _ in range(reps):
        P.cyclic_convolve_real(plan, xe, he)
    api_s = (time.perf_counter() - t0) / reps
    lib = _lib.load()
    dp = plan.device_plan()
    st = _lib.stream_handle()
    dx = torch.from_numpy(xe).cuda()
    dh = torch.from_numpy(he).cuda()
    dz = torch.empty_like(dx)
    run = lambda: lib.fntgpu_cyclic_convolve_real(dp.handle, dx.data_ptr(), dh.data_ptr(), 64,  # noqa: E731
                                                  dz.data_ptr(), 16384, 0, st)
    for _ in range(5):
        run()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(1000):
        run()
    b.record()
    torch.cuda.synchronize()
    loop_us = a.elapsed_time(b)  # ms for 1000 launches = us per launch (host launch rate bound)
    # the kernel alone: 100 launches captured in a CUDA graph, replayed 10 times (the
    # Python/ctypes launch loop above cannot issue a ~5 us kernel back to back)
    k_us, timing = loop_us, "1000 launches from a Python loop (CUDA events)"
    try:
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                gst = _lib.stream_handle()
                for _ in range(100):
                    lib.fntgpu_cyclic_convolve_real(dp.handle, dx.data_ptr(), dh.data_ptr(), 64,
                                                    dz.data_ptr(), 16384, 0, gst)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(10):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        k_us = a.elapsed_time(b)  # ms for 1000 graph-launched kernels = us per launch
        timing = "100 launches captured in a CUDA graph, replayed 10 times (CUDA events)"
    except Exception as e:  # noqa: BLE001 -- keep the loop number
        timing += f" (graph capture failed: {e})"
    n = 16384 * 64
    peaks = measured_peaks()
    tops = n * C1_OPS_PER_ELEMENT / (k_us * 1e-6) / 1e12
    return {"metric": "config-1 cyclic convolutions Gsamples/s", "unit": UNIT,
            "value": n / api_s / 1e9, "api_us_per_call": api_s * 1e6,
            "api_path": "P.cyclic_convolve_real(plan, x, h) on numpy int64 (16384, 64) residue "
                        "arrays: H2D of x and h, one fntgpu_cyclic_convolve_real launch, D2H of z",
            "kernel": {"us_per_launch": k_us, "gsamples_s": n / (k_us * 1e-6) / 1e9,
                       "alg_ops_per_element": C1_OPS_PER_ELEMENT, "achieved_tops": tops,
                       "int_frac": tops / peaks["int_tops"],
                       "hbm_gbs_int64": n * 24 / (k_us * 1e-6) / 1e9,
                       "timing": timing, "python_loop_us_per_launch": loop_us,
                       "note": "the API takes the reference's int64 arrays (24 B per element moved); "
                               "SURVEY 8(d)'s 6 B/element assumes int8 / int32 I/O"},
            "parity_vs_oracle": ok}


def run_c3(args) -> dict:
    """The per-stream latency regime of config 3: 6 dual-pol links of 2^20 symbols
    (SNR 14..24 dB) through the whole chain on one GPU -- each link's 16-symbol block
    recursion is sequential, so this measures per-stream latency."""
    import torch
    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.stream import CdcAeqChain, decimation_phase
    n_sym = 1 << 20
    cfg = P.LinkConfig(n_symbols=n_sym, z_km=75.0, pol_rotation_deg=0.0, dgd_symbols=0.0,
                       iq_skew_samples=0.0, seed=2)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    L = 2 * n_sym
    gen = DeviceLinkGenerator(n_sym, z_km=75.0, sig_scale=cfg.sig_scale)
    xr, xi = gen.generate(6, seed=2, snr_db=(14.0, 24.0), chunk=6)
    chain = CdcAeqChain(eng, cfg.aeq_config(), 6, L, cfg.sig_spec(), cfg.mu_schedule())
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def once():
        chain.aeq.reset()
        chain.acc.zero_()
        e[0].record()
        chain.cdc.run(xr, xi, length=L, qr=chain.qr, qi=chain.qi, q_spec=chain.sig_spec,
                      decim_acc=chain.acc)
        e[1].record()
        decimation_phase(chain.acc, 6, L, chain.phase, chain.gap)
        chain.check_ties(xr, xi)
        e[2].record()
        chain.aeq.run_decim(chain.qr, chain.qi, chain.phase, chain.n_blocks, chain.y, adapt=True,
                            mu_blocks=chain.mu_blocks, err=chain.err)
        e[3].record()
        torch.cuda.synchronize()
        return e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3]), e[0].elapsed_time(e[3])

    once()
    reps = 2
    t = np.array([once() for _ in range(reps)]).mean(axis=0)
    cdc_ms, aeq_ms, ms = (float(v) for v in t)
    res = {"metric": "config-3 shape chain Gsamples/s (per-stream latency regime)", "unit": UNIT,
           "value": 6 * 2 * L / (ms * 1e-3) / 1e9, "ms_per_step": ms, "cdc_ms": cdc_ms,
           "aeq_ms": aeq_ms, "aeq_block_us": aeq_ms * 1e3 / chain.n_blocks,
           "aeq_kernel": "k_aeq_pol (two warps per stream; auto)",
           "workload": "6 dual-pol links x 2^20 symbols (SNR 14..24 dB, 75 km), whole chain, one GPU"}
    chain.aeq.prm.kernel = 1  # the one-warp layout on the same data
    once()
    res["aeq_ms_one_warp_layout"] = float(np.mean([once()[1] for _ in range(reps)]))
    del chain, xr, xi
    return res


if __name__ == "__main__":
    main()
