# prefill parity + config-3 A/B of an on/off switch: bash tools/gpu_env_ab.sh GLM_LN_ROWS8
V=$1
timeout 1500 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
for i in 1 2 3 4; do
  echo "on:";  env $V=1 timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c1-150
  echo "off:"; env $V=0 timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c1-150
done
bash tools/ncu_prefill_list.sh
