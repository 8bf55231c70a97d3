#!/bin/bash
# A/B timing of libfntgpu variants: tools/ab_run.sh NAME... (build/ab/libfntgpu_NAME.so)
# Prints the per-kernel CUDA-event times bench.py measures for each variant.
for n in "$@"; do
  FNTGPU_LIB=build/ab/libfntgpu_$n.so python bench.py --no-cpu --no-e2e --no-quality --no-alt \
    --steps 3 --warmup 2 ${AB_ARGS} > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  python - "$n" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{n}.json"))
    k = d["roofline"].get("kernels", {})
    aeq = next((v.get("ms") for kk, v in k.items() if kk.startswith("k_aeq")), float("nan"))
    cdc = next((v.get("ms") for kk, v in k.items() if kk.startswith("k_cdc64")), float("nan"))
    print(f"{n:12s} step {d['ms_per_step']:8.2f} ms  value {d['value']:8.2f}  aeq {aeq:8.2f}  cdc {cdc:7.2f}  frac {d['roofline']['frac']:.3f}")
except Exception as e:
    print(n, "FAILED", e, open(f"gpurun_out/ab_{n}.err").read()[-500:])
PY
done
