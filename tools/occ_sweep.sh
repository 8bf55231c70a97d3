for L in 592 1184 1776 2368 2960; do
  python bench.py --no-cpu --no-e2e --no-quality --no-alt --steps 2 --warmup 2 --links $L > gpurun_out/occ_$L.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/occ_$L.json')); k=d['roofline']['kernels']; print($L, round(k['k_aeq_process']['ms'],2), round(k['k_cdc64']['ms'],2))"
done
FNTGPU_LIB=build/ab/libfntgpu_mb3.so python bench.py --no-cpu --no-e2e --no-quality --no-alt --steps 2 --warmup 2 --links 1776 > gpurun_out/occ_mb3.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/occ_mb3.json')); k=d['roofline']['kernels']; print('mb3@1776', round(k['k_aeq_process']['ms'],2))"
