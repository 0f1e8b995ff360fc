# Round-2 decode profile: ncu launch list of one decode step (serialized, cold) and
# `ncu --set full` of the four single-token INT4 GEMV launches (k_gemv_i4) of layer 0.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/r2_decode_launches.csv python tools/profile_decode.py --steps 1 > gpurun_out/r2_ncu_list.log 2>&1
echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/r2_decode_launches.csv > gpurun_out/r2_decode_launches_summary.txt; head -20 gpurun_out/r2_decode_launches_summary.txt
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_gemv_i4 -c 4 \
    -o gpurun_out/r2_gemv_i4 python tools/profile_decode.py --steps 1 > gpurun_out/r2_ncu_full.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/r2_gemv_i4.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/r2_gemv_i4_raw.csv 2>&1
cat gpurun_out/r2_gemv_i4_raw.csv | cut -c1-400
