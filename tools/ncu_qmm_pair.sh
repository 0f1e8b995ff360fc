# ncu --set full of the paired W1|V GEMM with the GeGLU epilogue, config-3 shapes (tools/ncu_qmm_pair.sh)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_qmm_tc -s 2 -c 1 -o gpurun_out/qmm_pair python tools/bench_prefill.py --bits 4 --iters 1 > gpurun_out/ncu_pair.log 2>&1; tail -1 gpurun_out/ncu_pair.log
