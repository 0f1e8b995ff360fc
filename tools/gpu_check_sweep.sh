# quick parity check of the GEMV/model paths, then an env sweep over bench.py
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qlinear.py tests/test_gpu_model.py -x -q > gpurun_out/check.log 2>&1; tail -3 gpurun_out/check.log
bash tools/gpu_sweep_env.sh "$@"
