# fused W1|V GEMM + GeGLU epilogue: parity + config-3 A/B (tools/gpu_geglu_ab.sh)
timeout 1500 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
for i in 1 2 3 4; do
  echo "fused:";   timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c1-150
  echo "unfused:"; GLM_QMM_GEGLU=0 timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c1-150
done
