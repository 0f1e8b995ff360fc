mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prefill_launches.csv python tools/bench_prefill.py --bits 4 --iters 1 > gpurun_out/ncu_prefill.log 2>&1
python tools/launch_summary.py gpurun_out/prefill_launches.csv > gpurun_out/prefill_launches_summary.txt 2>&1; cat gpurun_out/prefill_launches_summary.txt
