# Round-end evidence (run on the GPU box from the repo root; outputs in gpurun_out/):
# ncu launch lists and full captures that profiles/ summarises (tools/ncu_summary.py).
# Each profiled command first runs once without ncu (it must exit 0).
set -x
C5="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-quality --no-alt --no-sub --no-parity"
C5S="python bench.py --links 512 --steps 2 --warmup 1 --no-cpu --no-e2e --no-quality --no-alt --no-sub --no-parity"
C4="python bench.py --config c4 --steps 2 --warmup 1 --no-cpu --no-e2e --no-alt"
$C5 > gpurun_out/p_c5.json 2> gpurun_out/p_c5.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(cdc64|aeq|decim)" -c 40 --csv \
      --log-file gpurun_out/launches_r02.csv $C5 > gpurun_out/ncu_launch.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_cdc64|k_aeq_process" -c 2 \
      -o gpurun_out/prof_r02 $C5 > gpurun_out/ncu_full.log 2>&1
$C5S > gpurun_out/p_c5s.json 2> gpurun_out/p_c5s.err && \
  ncu --set full --import-source on --clock-control none -k regex:"k_aeq_pol" -c 1 \
      -o gpurun_out/prof_r02_pol512 $C5S > gpurun_out/ncu_full_pol.log 2>&1
$C4 > gpurun_out/p_c4.json 2> gpurun_out/p_c4.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cdc64" -c 10 --csv \
      --log-file gpurun_out/launches_r02_c4.csv $C4 > gpurun_out/ncu_launch_c4.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_cdc64" -c 1 \
      -o gpurun_out/prof_r02_c4 $C4 > gpurun_out/ncu_full_c4.log 2>&1
tail -n 2 gpurun_out/ncu_full.log gpurun_out/ncu_full_pol.log gpurun_out/ncu_full_c4.log
