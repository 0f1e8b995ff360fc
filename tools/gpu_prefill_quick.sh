# prefill parity + config-3 timing (tools/gpu_prefill_quick.sh)
timeout 1500 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
for i in 1 2 3; do timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c1-150; done
bash tools/ncu_prefill_list.sh
