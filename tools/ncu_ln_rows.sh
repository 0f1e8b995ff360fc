# ncu --set full of the prefill DeepNorm LayerNorm (tools/ncu_ln_rows.sh)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_deepnorm_ln_rows -c 1 -o gpurun_out/ln_rows python tools/bench_prefill.py --bits 4 --iters 1 > gpurun_out/ncu_ln.log 2>&1; tail -1 gpurun_out/ncu_ln.log
