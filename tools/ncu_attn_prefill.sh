mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_attn_prefill -s 1 -c 1 -o gpurun_out/attn_prefill python tools/bench_prefill.py --bits 4 --iters 1 > gpurun_out/ncu_attn.log 2>&1
tail -1 gpurun_out/ncu_attn.log
