# Round-end evidence (run on the GPU box from the repo root; outputs in gpurun_out/):
# bench lines for C5 / C4 / the reference arm, the ncu launch lists and full captures
# that profiles/ summarises (tools/ncu_summary.py).
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --config c4 > gpurun_out/bench_final_c4.json 2> gpurun_out/bench_final_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(cdc64|aeq|decim|quant|fnt|conv)" -c 40 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-quality --no-alt > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cdc64" -c 10 --csv --log-file gpurun_out/launches_final_c4.csv python bench.py --config c4 --steps 2 --warmup 1 --no-cpu --no-e2e --no-alt > gpurun_out/ncu_launch_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_cdc64|k_aeq_process" -c 2 -o gpurun_out/prof_final python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-quality --no-alt > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_cdc64_umma" -c 1 -o gpurun_out/prof_final_c4 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-alt > gpurun_out/ncu_full_c4.log 2>&1
tail -2 gpurun_out/ncu_full.log gpurun_out/ncu_full_c4.log
