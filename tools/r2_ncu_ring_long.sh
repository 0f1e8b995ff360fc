# ncu --set full summary of the streaming decode attention at config 2 (one G block, KV 2048)
mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:k_attn_decode_ring -s 5 -c 3 -o /tmp/r2_ring_long \
    python tools/bench_block_decode.py > /dev/null 2>&1
ncu -i /tmp/r2_ring_long.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,launch__occupancy_limit_shared_mem > gpurun_out/r2_ring_long_ncu.csv 2>&1
