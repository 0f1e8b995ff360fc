# ncu launch list of one batch-8 decode step (per-kernel shares) and --set full summaries of the
# batched integer-MMA GEMV and the streaming attention (GLM-130B shape, 16 layers)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file /tmp/b8_launches.csv python tools/profile_decode.py --steps 1 --batch 8 > gpurun_out/r2_b8_list.log 2>&1
python tools/launch_summary.py /tmp/b8_launches.csv > gpurun_out/r2_b8_launches_summary.txt
for k in k_gemv_mk_i4 k_attn_decode_ring; do
  ncu --set full --clock-control none --profile-from-start off -k regex:$k -c 4 -o /tmp/r2_b8_$k \
      python tools/profile_decode.py --steps 1 --batch 8 --layers 4 > /dev/null 2>&1
  ncu -i /tmp/r2_b8_$k.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread > gpurun_out/r2_b8_$k.csv 2>&1
done
