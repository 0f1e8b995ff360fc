mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/block_decode_launches.csv python tools/bench_block_decode.py > gpurun_out/ncu_bd.log 2>&1
python tools/launch_summary.py gpurun_out/block_decode_launches.csv 2>&1 | head -30
