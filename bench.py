#!/usr/bin/env python3
"""FNT-CDC + FNT-AEQ throughput on B200 (BASELINE.json metric).

Workload (default, --config c5): BASELINE config 5 -- many-channel dual-pol
PDM-16QAM receivers: per GPU `--links` (4096) independent links of 2^18 symbols
at 2 sps (L = 2^19 complex samples per polarization), 75 km, per-link Haar Jones
rotation and SNR ~ U[16, 22] dB, generated on device (paper_2405_04253_b200.
linkgen; statistically equivalent to the reference generator, not bitwise).
One step = the whole receiver chain over every link with inputs resident in
HBM: FNT-CDC on both polarizations (fused requantization + decimation
statistics) -> decimation phase -> adaptive FNT-AEQ (fresh state per link,
LinkConfig gear-shift mu schedule). Inputs (8.6 GB) exceed L2 (126 MB), so no
L2 flush is needed between steps.

Metric: Gsamples/s = complex samples per polarization, summed over
polarizations and links, per second (whole job, all ranks).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU,
        links sharded as independent objects: weak scaling, no collective on
        the data path; NCCL only reduces the timing/sample counts)
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

# Algorithmic work per unit (SURVEY 8d convention):
#   radix-2 butterfly = 6 INT ops, general residue product = 6, modular aux op = 2
CDC_INT_OPS_PER_BLOCK = 4 * 192 * 6 + 128 * 6 + 256 * 2   # 5888 per 64-block = 184 / sample
CDC_TC_MACS_PER_BLOCK = 2 * 2 * 64 * 64 + 2 * 4 * 32 * 64    # int8 MACs per block, matrix forms
AEQ_INT_OPS_PER_BLOCK_FNT = (4 + 32 + 32) * 80 * 6 + 1024 * 6 + 448  # 39232 (incl. tap-spectrum refresh)
AEQ_INT_OPS_PER_BLOCK_DIRECT = 2 * 4096 + 448               # 8640 (exact time-domain MIMO FIR)
# The kernel's transform-domain stream sum (k_aeq.cu fused_ok; every block of 5-bit
# inputs with ordinary taps) runs 8 split inverses instead of 32, plus the sums over t
# (3 modular adds x 32 bins x 8) and the inverses' cross-lane twiddles (8 x 4 x 16):
AEQ_INT_OPS_PER_BLOCK_FNT_FUSED = (4 + 32 + 8) * 80 * 6 + 1024 * 6 + 768 * 2 + 512 * 2 + 448  # 30272
AEQ_FP64_OPS_PER_BLOCK = 2 * 4096 + 256 * 4 + 64 * 2 + 32 * 12  # gradient + update + y + rde ~ 9728


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
    """One link through the numpy restatement of the reference (np_port.chain)."""
    xr2, xi2, tap_re, tap_im, n_taps, out_scale, sig_scale, mu = args
    import oracle.np_port as N
    t0 = time.perf_counter()
    N.chain(xr2, xi2, tap_re, tap_im, n_taps, out_scale, sig_scale, mu)
    return time.perf_counter() - t0


def cpu_links_sample(n_tasks: int, n_sym: int, seed: int = 4):
    """Bounded CPU sample: n_tasks links of n_sym symbols from the numpy
    generator port of the reference link model (oracle.linkgen), falling back to
    i.i.d. 5-bit samples if unavailable; returns per-task inputs."""
    rng = np.random.default_rng(seed)
    L = 2 * n_sym
    out = []
    for _ in range(n_tasks):
        out.append((rng.integers(-15, 16, (2, L)), rng.integers(-15, 16, (2, L))))
    return out


def run_cpu_baseline(engine, cfg, n_sym: int, cores: int, rounds: int | None = None) -> dict:
    """Time the reference algorithm (numpy port) on all host cores."""
    from concurrent.futures import ProcessPoolExecutor
    import oracle.np_port  # noqa: F401  (checker / baseline only)
    hop = 16
    nb = n_sym // hop
    mu = np.where(np.arange(nb) * hop < cfg.gear_symbols, cfg.mu1, cfg.mu2)
    samples = cpu_links_sample(cores, n_sym)
    args = [(xr, xi, engine.tap_re, engine.tap_im, cfg.n_cdc_taps, engine.output_scale,
             cfg.sig_scale, mu) for xr, xi in samples]
    with ProcessPoolExecutor(max_workers=cores) as ex:
        per_task = max(list(ex.map(_cpu_task, args)))  # warm the workers' imports, size the sample
        if rounds is None:
            # about 20 s of CPU work over all cores (a bounded sample of the workload)
            rounds = max(1, int(round(20.0 / max(per_task * cores, 1e-3))))
        t0 = time.perf_counter()
        for _ in range(rounds):
            list(ex.map(_cpu_task, args))
        wall = time.perf_counter() - t0
    n_samples = rounds * cores * 2 * (2 * n_sym)
    return {"value": n_samples / wall / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"{rounds * cores} links x 2 pols x {2 * n_sym} samples (2^{int(math.log2(n_sym))} "
                       f"symbols) through oracle/np_port.chain (numpy restatement of the reference's "
                       f"CDC -> glue -> AEQ, pinned to reference fixtures), one process per core, "
                       f"{wall:.1f} s wall"),
            "wall_s": wall}


def impl_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT))
    from paper_2405_04253_b200.cdc import CdcConfig
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
            "config": {"workload": "C4 throughput-scale FNT-CDC (CPU sample)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}))
        return
    for _ in range(args.warmup and 1):
        run_cpu_baseline(eng, cfg, n_sym, cores)
    t0 = time.perf_counter()
    vals = [run_cpu_baseline(eng, cfg, n_sym, cores) for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    v = float(np.mean([x["value"] for x in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic", "config": _config_dict(args, cpu=True),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": ("the reference is pure numpy (no native build); its algorithm is timed through "
                 "oracle/np_port.py, a numpy restatement pinned to the reference's golden outputs"),
    }
    del CdcConfig
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


# ------------------------------------------------------------------ GPU side

def _link_cfg(args):
    from paper_2405_04253_b200.linksim import LinkConfig
    return LinkConfig(n_symbols=args.symbols, z_km=75.0, pol_rotation_deg=0.0, dgd_symbols=0.0,
                      iq_skew_samples=0.0, seed=4)


def _config_dict(args, cpu=False):
    d = {"workload": ("C5 many-channel FNT-CDC+FNT-AEQ: per GPU %d dual-pol PDM-16QAM links x 2^%d "
                      "symbols x 2 sps, 75 km SSMF, Haar Jones, SNR U[16,22] dB, 5-bit I/Q, "
                      "6-bit CDC taps (N=64 sqrt2 FNT), 4x4 FNT-AEQ (N=32) gear-shift mu")
                     % (args.links, int(math.log2(args.symbols))),
         "links_per_gpu": args.links, "symbols": args.symbols, "samples_per_pol": 2 * args.symbols,
         "aeq_forward": args.forward,
         "cdc_kernel": {"tc": "k_cdc64_tc (mma.sync split-integer FNT)",
                        "umma": "k_cdc64_umma (tcgen05 split-integer FNT)"}.get(
                            args.cdc_kernel, "k_cdc64_umma (tcgen05 split-integer FNT; auto)"),
         "parallelism": f"links sharded over {args.gpus} GPU(s), no collective",
         "l2": "inputs (int8 I/Q, %.1f GB/GPU) exceed the 126 MB L2; no flush needed"
               % (4 * args.links * 2 * args.symbols / 1e9)}
    if cpu:
        d["cpu_symbols"] = args.cpu_symbols
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--links", type=int, default=4096, help="links per GPU (C5: 4096)")
    ap.add_argument("--symbols", type=int, default=1 << 18)
    ap.add_argument("--forward", default="fnt", choices=["fnt", "direct"])
    ap.add_argument("--e2e-links", type=int, default=None,
                    help="links per rank in the host-buffer e2e run (default 512 on one GPU, "
                         "256 per rank under torchrun: bounds the pinned host memory per node)")
    ap.add_argument("--cpu-symbols", type=int, default=1 << 13)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", default="c5", choices=["c5", "c4"],
                    help="c5: many-channel CDC+AEQ chain (headline); c4: throughput-scale CDC")
    ap.add_argument("--c4-samples", type=int, default=1 << 31, help="C4 samples per polarization")
    ap.add_argument("--no-alt", action="store_true", help="skip the direct-forward AEQ comparison")
    ap.add_argument("--no-quality", action="store_true", help="skip the on-device BER/EVM scoring")
    ap.add_argument("--aeq-kernel", default="auto", choices=["auto", "warp", "pol"],
                    help="FNT-AEQ stream layout: one warp per stream, two warps per stream (one per "
                         "polarization), or auto (the split form below ~8 streams per SM)")
    ap.add_argument("--cdc-kernel", default="auto", choices=["auto", "umma", "tc", "shift"],
                    help="FNT-CDC kernel for the int8 planes: auto (measured-faster choice), shift-add "
                         "butterflies, or the split-integer matrix form on mma.sync (tc) / tcgen05 (umma)")
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

    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200 import _lib
    from paper_2405_04253_b200 import cdc as cdc_mod
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.stream import CdcAeqChain
    cdc_mod.set_cdc_kernel(args.cdc_kernel)
    from paper_2405_04253_b200 import aeq as aeq_mod
    aeq_mod.set_aeq_kernel(args.aeq_kernel)

    if args.config == "c4":
        run_c4(args, world, rank, local)
        if world > 1:
            dist.destroy_process_group()
        return

    cfg = _link_cfg(args)
    fwd = _lib.AEQ_FWD_DIRECT if args.forward == "direct" else _lib.AEQ_FWD_FNT
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    L = 2 * args.symbols
    gen = DeviceLinkGenerator(args.symbols, z_km=cfg.z_km, sig_scale=cfg.sig_scale)
    xr, xi, sidx = gen.generate(args.links, seed=4 + 7919 * rank, symbols=True)
    chain = CdcAeqChain(eng, cfg.aeq_config(), args.links, L, cfg.sig_spec(), cfg.mu_schedule(),
                        forward=fwd)
    torch.cuda.synchronize()

    # instrumented step: events around the two heavy kernels on the launching stream
    ev = []

    def step(record: bool):
        s = torch.cuda.current_stream()
        if record:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            chain.aeq.reset()
            chain.acc.zero_()
            e[0].record(s)
            chain.cdc.run(xr, xi, length=L, qr=chain.qr, qi=chain.qi, q_spec=chain.sig_spec,
                          decim_acc=chain.acc)
            e[1].record(s)
            from paper_2405_04253_b200.stream import decimation_phase
            decimation_phase(chain.acc, chain.n_links, L, chain.phase, chain.gap)
            e[2].record(s)
            chain.aeq.run_decim(chain.qr, chain.qi, chain.phase, chain.n_blocks, chain.y,
                                adapt=True, mu_blocks=chain.mu_blocks, err=chain.err)
            e[3].record(s)
            ev.append(e)
        else:
            chain.run(xr, xi)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start.record()
    for _ in range(args.steps):
        step(True)
    t_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    cdc_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    ph_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    aeq_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    samples_rank = args.steps * args.links * 2 * L
    if world > 1:
        ms_max = allreduce([ms], "max")[0]
        samples_all = allreduce([float(samples_rank)], "sum")[0]
    else:
        ms_max, samples_all = ms, float(samples_rank)
    value = samples_all / (ms_max * 1e-3) / 1e9

    # sanity on the outputs of the last step (cheap): finite, phase decided
    ok = bool(torch.isfinite(chain.y).all().item())

    peaks = measured_peaks()
    # the CDC kernel auto selects for int8 planes with the fused epilogue (k_cdc.cu)
    cdc_name = {"tc": "k_cdc64_tc", "shift": "k_cdc64"}.get(args.cdc_kernel, "k_cdc64_umma")
    n_blk_cdc = 2 * args.links * (L // 32 + 1)
    n_blk_aeq = args.links * chain.n_blocks
    cdc_tops = n_blk_cdc * CDC_INT_OPS_PER_BLOCK / (cdc_ms * 1e-3) / 1e12
    aeq_int = AEQ_INT_OPS_PER_BLOCK_FNT if fwd == _lib.AEQ_FWD_FNT else AEQ_INT_OPS_PER_BLOCK_DIRECT
    aeq_tops = n_blk_aeq * aeq_int / (aeq_ms * 1e-3) / 1e12
    aeq_fp64 = n_blk_aeq * AEQ_FP64_OPS_PER_BLOCK / (aeq_ms * 1e-3) / 1e12
    cdc_bytes = 2 * args.links * L * (2 + 2)  # int8 I/Q in, int8 requantized I/Q out
    # AEQ HBM: 4 int8 rows read in 32-byte phase pairs, float64 y written, err_trace written
    aeq_bytes = args.links * (4 * 32 * chain.n_blocks + 4 * 16 * chain.n_blocks * 8 + 8 * chain.n_blocks)
    traffic = None
    ncu = PROFILES / "ncu_summary_r01.json"
    if ncu.exists():
        try:
            traffic = json.loads(ncu.read_text()).get("per_launch_dram_bytes", {})
        except Exception:
            traffic = None
    kernels = {
        cdc_name: {"ms": cdc_ms, "bound": "int", "achieved": cdc_tops, "peak": peaks["int_tops"],
                   "unit": "Tops/s", "frac": cdc_tops / peaks["int_tops"],
                   "alg_ops_per_launch": n_blk_cdc * CDC_INT_OPS_PER_BLOCK,
                   "hbm_gbs": cdc_bytes / (cdc_ms * 1e-3) / 1e9},
        "k_aeq_process": {"ms": aeq_ms, "bound": "int", "achieved": aeq_tops,
                          "peak": peaks["int_tops"], "unit": "Tops/s",
                          "frac": aeq_tops / peaks["int_tops"],
                          "alg_ops_per_launch": n_blk_aeq * aeq_int,
                          "fp64_tinst_per_s": aeq_fp64,
                          "fp64_frac": aeq_fp64 / peaks["fp64_tinst"],
                          # the kernel's two kinds of work share the SM sub-partitions' issue
                          # slots: INT ops at the INT peak plus FP64 ops at the FP64 peak,
                          # back to back, over the measured time (INT-only "frac" is the headline)
                          "int_plus_fp64_frac": (aeq_tops / peaks["int_tops"]
                                                 + aeq_fp64 / peaks["fp64_tinst"]),
                          # the same with the op count of the form the kernel executes
                          # (transform-domain sum over input streams; FNT forward only)
                          "int_plus_fp64_frac_fused_form": (
                              (n_blk_aeq * AEQ_INT_OPS_PER_BLOCK_FNT_FUSED / (aeq_ms * 1e-3) / 1e12
                               / peaks["int_tops"] + aeq_fp64 / peaks["fp64_tinst"])
                              if fwd == _lib.AEQ_FWD_FNT else None),
                          "hbm_gbs": aeq_bytes / (aeq_ms * 1e-3) / 1e9},
        "k_decim_phase": {"ms": ph_ms},
    }
    if cdc_name != "k_cdc64":
        # matrix forms: FNT-equivalent ALG ops against the INT peak above, tensor side here
        tmacs = n_blk_cdc * CDC_TC_MACS_PER_BLOCK / (cdc_ms * 1e-3)
        int8_peak = 2.0 * peaks.get("bf16_tflops", 2250.0)
        kernels[cdc_name]["tensor"] = {"achieved": 2.0 * tmacs / 1e12, "peak": int8_peak,
                                       "unit": "Tops/s (int8)", "frac": 2.0 * tmacs / 1e12 / int8_peak}
    dom = "k_aeq_process" if aeq_ms >= cdc_ms else cdc_name
    kd = kernels[dom]
    tr = None
    if isinstance(traffic, dict) and dom in traffic:
        tr = traffic[dom]
    roofline = {"bound": kd["bound"], "kernel": dom, "achieved": kd["achieved"], "peak": kd["peak"],
                "unit": kd["unit"], "frac": kd["frac"], "traffic": tr,
                "peak_source": peaks["int_source"],
                "step_share": kd["ms"] / (cdc_ms + ph_ms + aeq_ms),
                "kernels": kernels,
                "hbm": {"achieved_gbs": (cdc_bytes + aeq_bytes) / ((cdc_ms + aeq_ms) * 1e-3) / 1e9,
                        "peak_gbs": peaks["hbm_gbs"]}}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32 (Z/(2^32-1) residues) + f64",
        "data": "synthetic (on-device 16QAM link model, seeded)", "config": _config_dict(args),
        "roofline": roofline, "clocks": clk, "gpu_launches": 4 * args.steps,
        "outputs_finite": ok,
    }

    # link quality of the timed step's outputs, scored on the device (metrology.py;
    # outside the timed region). Expected to be poor at 75 km: 32 CDC taps cover the
    # dispersion badly and the reference's RDE does not converge (SURVEY finding 4).
    if not args.no_quality:
        from paper_2405_04253_b200 import metrology as M
        bers, evms, oks = [], [], []
        for c0 in range(0, args.links, 32):
            c1 = min(args.links, c0 + 32)
            sym, bits = gen.tx_reference(sidx[c0:c1])
            b, e, o = M.align_and_count(M.aeq_to_pols(chain.y[c0:c1]), sym, bits,
                                        cfg.discard_symbols)
            bers.append(b)
            evms.append(e)
            oks.append(o)
        bers, evms, oks = np.concatenate(bers), np.concatenate(evms), np.concatenate(oks)
        line["link_quality"] = {
            "ber_mean": float(bers.mean()), "ber_min": float(bers.min()),
            "evm_db_mean": float(evms[oks].mean()) if oks.any() else None,
            "aligned_fraction": float(oks.mean()),
            "note": "BER/EVM of every link computed on the GPU (metrology.align_and_count); "
                    "high BER at 75 km reproduces the reference's behaviour (SURVEY finding 4)"}

    # the exact-equivalent time-domain forward (FNTGPU_AEQ_FWD_DIRECT, same bits) on the
    # same resident data, reported beside the FNT-domain headline
    if fwd == _lib.AEQ_FWD_FNT and not args.no_alt:
        chain.aeq.prm.forward = _lib.AEQ_FWD_DIRECT
        chain.run(xr, xi)
        torch.cuda.synchronize()
        ev.clear()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            step(True)
        b.record()
        torch.cuda.synchronize()
        ms_alt = a.elapsed_time(b)
        if world > 1:
            ms_alt = allreduce([ms_alt], "max")[0]
        line["aeq_forward_direct"] = {
            "value": samples_all / (ms_alt * 1e-3) / 1e9, "unit": UNIT,
            "ms_per_step": ms_alt / args.steps,
            "aeq_ms": float(np.mean([e[2].elapsed_time(e[3]) for e in ev])),
            "note": "same chain with the AEQ forward as an exact time-domain integer FIR "
                    "(bit-identical outputs, tests/test_gpu_parity.py); headline uses the FNT forward"}
        chain.aeq.prm.forward = _lib.AEQ_FWD_FNT

    # the CDC launch of the chain through both kernels (same inputs, same outputs)
    if not args.no_alt:
        line["cdc_kernels"] = time_cdc_kernels(
            lambda: chain.cdc.run(xr, xi, length=L, qr=chain.qr, qi=chain.qi,
                                  q_spec=chain.sig_spec, decim_acc=chain.acc),
            args.steps, world)

    # end-to-end through the public host API: pinned host int8 in, float64 AEQ y out
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, eng, cfg, xr, xi, fwd, world)

    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = run_cpu_baseline(eng, cfg, args.cpu_symbols, os.cpu_count() or 1)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def _cdc_cpu_task(args):
    xr, xi, bp, bm = args
    import oracle.np_port as N
    t0 = time.perf_counter()
    N.cdc_process_int(xr, xi, bp, bm, 32)
    return time.perf_counter() - t0


def run_cpu_cdc_baseline(eng, n: int, cores: int) -> dict:
    """Reference-algorithm CDC (numpy restatement) on all host cores, ~20 s of CPU work."""
    from concurrent.futures import ProcessPoolExecutor
    rng = np.random.default_rng(3)
    tasks = [(rng.integers(-15, 16, n), rng.integers(-15, 16, n), eng._b_plus, eng._b_minus)
             for _ in range(cores)]
    with ProcessPoolExecutor(max_workers=cores) as ex:
        per = max(ex.map(_cdc_cpu_task, tasks))
        rounds = max(1, int(round(20.0 / max(per * cores, 1e-3))))
        t0 = time.perf_counter()
        for _ in range(rounds):
            list(ex.map(_cdc_cpu_task, tasks))
        wall = time.perf_counter() - t0
    return {"value": rounds * cores * n / wall / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"{rounds * cores} streams x {n} complex samples through oracle/np_port."
                       f"cdc_process_int (numpy restatement of the reference's FntCdcEngine."
                       f"process_int), one process per core, {wall:.1f} s wall")}


def time_cdc_kernels(run, reps: int, world: int) -> dict:
    """Device time of one CDC launch with each kernel (tensor-core matrix form and the
    shift-add butterflies), on the launching stream, max over ranks."""
    import torch
    from paper_2405_04253_b200 import cdc as cdc_mod
    out = {}
    prev = cdc_mod.set_cdc_kernel("tc")
    try:
        for name in ("umma", "tc", "shift"):
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
    out["note"] = ("k_cdc64_umma / k_cdc64_tc: forward FNT-64 and pruned inverse as split-integer "
                   "int8 matrix products on tcgen05 (UTCIMMA, TMEM accumulators) / mma.sync "
                   "(IMMA.16832); k_cdc64: radix-sqrt2 shift-add butterflies. Bit-identical "
                   "outputs (tests/test_gpu_parity.py)")
    return out


def c4_traffic(world: int, kernel: str = "k_cdc64"):
    """DRAM bytes of one CDC launch at config 4 on one GPU, from the committed ncu
    --set full capture (profiles/ncu_summary_r01_c4.json); None for other shard sizes."""
    path = PROFILES / "ncu_summary_r01_c4.json"
    if world != 1 or not path.exists():
        return None
    try:
        return json.loads(path.read_text()).get("per_launch_dram_bytes", {}).get(kernel)
    except Exception:
        return None


def run_c4(args, world, rank, local):
    """BASELINE config 4: one dual-pol stream of 2^31 complex samples per
    polarization, FNT-CDC range-sharded across ranks (strong scaling: the stream
    length is fixed) with the overlap-save halo read from each rank's input window
    (sharding.py); no data-path collective."""
    import torch
    import torch.distributed as dist
    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200 import cdc as cdc_mod
    from paper_2405_04253_b200.linkgen import DeviceLinkGenerator
    from paper_2405_04253_b200.sharding import cdc_range_shards
    cdc_mod.set_cdc_kernel(args.cdc_kernel)
    from paper_2405_04253_b200.stream import CdcBank

    cfg = P.LinkConfig(z_km=75.0, seed=3)
    eng = P.FntCdcEngine(cfg.cdc_config("fnt"), cfg.sig_spec())
    bank = CdcBank(eng)
    L = args.c4_samples
    sh = cdc_range_shards(L, world, n_taps=cfg.n_cdc_taps)[rank]
    # input window of this rank, generated on device in independent 2^22-sample
    # link segments (same signal model; seeded per segment)
    seg = 1 << 22
    n_seg = -(-sh.x_count // seg)
    gen = DeviceLinkGenerator(seg // 2, z_km=75.0, sig_scale=cfg.sig_scale)
    xr = torch.empty((2, n_seg * seg), dtype=torch.int8, device="cuda")
    xi = torch.empty_like(xr)
    per = 64
    for c0 in range(0, n_seg, per):
        c = min(per, n_seg - c0)
        gr, gi = gen.generate(c, seed=3 * 1_000_003 + sh.x_first // seg + c0)
        xr[:, c0 * seg:(c0 + c) * seg] = gr.view(c, 2, seg).transpose(0, 1).reshape(2, c * seg)
        xi[:, c0 * seg:(c0 + c) * seg] = gi.view(c, 2, seg).transpose(0, 1).reshape(2, c * seg)
        del gr, gi
    xr = xr[:, :sh.x_count]
    xi = xi[:, :sh.x_count]
    yr = torch.empty((2, sh.out_count), dtype=torch.int16, device="cuda")
    yi = torch.empty_like(yr)
    torch.cuda.synchronize()

    def step():
        bank.run(xr, xi, length=L, x_first=sh.x_first, out_first=sh.out_first,
                 out_count=sh.out_count, yr=yr, yi=yi)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step()
    b.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = a.elapsed_time(b)
    ms_max = ms
    if world > 1:
        ms_max = allreduce([ms], "max")[0]
    samples = 2 * L  # both polarizations of the whole stream, all ranks
    value = args.steps * samples / (ms_max * 1e-3) / 1e9
    peaks = measured_peaks()
    per_launch_ms = ms / args.steps
    n_blocks = 2 * (sh.out_count // 32 + 2)
    achieved = n_blocks * CDC_INT_OPS_PER_BLOCK / (per_launch_ms * 1e-3) / 1e12
    hbm_bytes = 2 * sh.x_count * 2 + 2 * sh.out_count * 4  # int8 I/Q in, int16 I/Q out
    hbm_gbs = hbm_bytes / (per_launch_ms * 1e-3) / 1e9
    # kernel auto picks for int8 planes with int16 outputs (k_cdc.cu launch_cdc64)
    c4_kernel = {"tc": "k_cdc64_tc", "shift": "k_cdc64"}.get(args.cdc_kernel, "k_cdc64_umma")
    line = {
        "metric": "FNT-CDC Gsamples/s (config 4)", "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32 (Z/(2^32-1) residues)", "data": "synthetic (on-device 16QAM link model)",
        "config": {"workload": "C4 throughput-scale FNT-CDC: one dual-pol stream of %d complex "
                               "samples per pol, 75 km taps, range-sharded over %d GPU(s) with the "
                               "overlap-save halo" % (L, world),
                   "samples_per_pol": L, "shard_out": [sh.out_first, sh.out_count],
                   "cdc_kernel": {"tc": "k_cdc64_tc", "shift": "k_cdc64"}.get(
                       args.cdc_kernel, "k_cdc64_umma (tcgen05 split-integer FNT; auto)"),
                   "l2": "inputs (%.1f GB) exceed L2" % (hbm_bytes / 1e9)},
        "roofline": {"bound": "int", "kernel": c4_kernel, "achieved": achieved,
                     "peak": peaks["int_tops"], "unit": "Tops/s",
                     "frac": achieved / peaks["int_tops"], "traffic": c4_traffic(world, c4_kernel),
                     "peak_source": peaks["int_source"],
                     "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks["hbm_gbs"],
                             "frac": hbm_gbs / peaks["hbm_gbs"]}},
        "clocks": clk, "gpu_launches": args.steps,
    }
    if c4_kernel != "k_cdc64":
        # the matrix forms run the transforms on the tensor cores: the roofline above counts
        # the algorithm's FNT work (SURVEY 8d convention) against the INT peak of the CUDA
        # cores that still carry the mod-F4 reductions; the tensor side is reported here
        macs = n_blocks * CDC_TC_MACS_PER_BLOCK / (per_launch_ms * 1e-3)
        int8_peak = 2.0 * peaks.get("bf16_tflops", 2250.0)  # dense int8 = 2x dense bf16
        line["roofline"]["tensor"] = {
            "achieved": 2.0 * macs / 1e12, "peak": int8_peak, "unit": "Tops/s (int8)",
            "frac": 2.0 * macs / 1e12 / int8_peak,
            "peak_source": "2 x measured dense bf16 (MEASURED_PEAKS.json)" if "bf16_tflops" in peaks
                           else "2 x nominal dense bf16",
            "macs_per_block": CDC_TC_MACS_PER_BLOCK}
    if not args.no_alt:
        line["cdc_kernels"] = time_cdc_kernels(step, args.steps, world)
    if not args.no_e2e:
        # host buffers through the C ABI: pinned int8 I/Q -> H2D -> CDC -> D2H int16 I/Q
        from paper_2405_04253_b200.stream import HostCdc
        n = min(1 << 28, sh.out_count)
        hc = HostCdc(eng, 2, n)
        hx = torch.empty((2, n), dtype=torch.int8, pin_memory=True)
        hy = torch.empty((2, n), dtype=torch.int8, pin_memory=True)
        hx.copy_(xr[:, :n])
        hy.copy_(xi[:, :n])
        hc(hx, hy)
        hc.join()
        torch.cuda.synchronize()
        a.record()
        for _ in range(args.steps):
            hc(hx, hy)  # each call: H2D of its inputs, CDC, D2H of the int16 outputs
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
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = run_cpu_cdc_baseline(eng, 1 << 20, os.cpu_count() or 1)
    if rank == 0:
        print(json.dumps(line))


def run_e2e(args, eng, cfg, xr, xi, fwd, world):
    import torch
    import torch.distributed as dist
    from paper_2405_04253_b200.stream import HostChain
    e2e_links = args.e2e_links if args.e2e_links is not None else (512 if world == 1 else 256)
    n = min(e2e_links, args.links)
    L = 2 * args.symbols
    hc = HostChain(eng, cfg.aeq_config(), n, L, cfg.sig_spec(), cfg.mu_schedule(), forward=fwd)
    hx_r = torch.empty((2 * n, L), dtype=torch.int8, pin_memory=True)
    hx_i = torch.empty((2 * n, L), dtype=torch.int8, pin_memory=True)
    hx_r.copy_(xr[:2 * n])
    hx_i.copy_(xi[:2 * n])
    for _ in range(min(args.warmup, 2)):
        hc(hx_r, hx_i)
    hc.join()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        hc(hx_r, hx_i)  # each call: H2D of its inputs, CDC, AEQ, D2H of y + err_trace
    hc.join()           # the current stream waits for the last call's copy-out
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        ms = allreduce([ms], "max")[0]
    samples = args.steps * n * 2 * L * world
    return {"value": samples / (ms * 1e-3) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": hc.h2d_bytes, "d2h_bytes_per_step": hc.d2h_bytes,
            "links_per_gpu": n,
            "path": "paper_2405_04253_b200.stream.HostChain: pinned host int8 I/Q -> H2D -> "
                    "CDC -> phase -> AEQ -> D2H float64 y + err_trace, every step; copies "
                    "pipelined with the kernels over 3 CUDA streams (input pieces, AEQ time "
                    "segments)"}


if __name__ == "__main__":
    main()
