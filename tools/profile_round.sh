set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --config c4 > gpurun_out/bench_final_c4.json 2> gpurun_out/bench_final_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(cdc64|aeq|decim|quant|fnt|conv)" -c 40 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-quality --no-alt > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_cdc64|k_aeq_process" -c 2 -o gpurun_out/prof_final python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-quality --no-alt > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
