# prefill-side refresh: GPU tests, smoke, config 3, launch list, ncu of the attention (tools/final_prefill.sh)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python tools/bench_prefill.py > gpurun_out/prefill.jsonl 2>&1; cut -c1-160 gpurun_out/prefill.jsonl
timeout 600 python tools/bench_block_decode.py > gpurun_out/block_decode.json 2>&1; cut -c1-200 gpurun_out/block_decode.json
bash tools/ncu_prefill_list.sh | head -12
bash tools/ncu_attn_prefill.sh
