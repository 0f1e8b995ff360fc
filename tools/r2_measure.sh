# Round-2 measurement pass (one box): smoke, default bench, configs 2 / 3 / 5, decode profile.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 300 gpurun_out/r2_bench.json; echo
timeout 600 python tools/bench_block_decode.py > gpurun_out/r2_block_decode.json 2>&1; cut -c1-300 gpurun_out/r2_block_decode.json
timeout 900 python tools/bench_prefill.py > gpurun_out/r2_prefill.jsonl 2>&1; cut -c1-300 gpurun_out/r2_prefill.jsonl
timeout 900 python tools/sweep_qlinear.py > gpurun_out/r2_qlinear_sweep.jsonl 2>&1; cat gpurun_out/r2_qlinear_sweep.jsonl
bash tools/r2_profile_decode.sh > gpurun_out/r2_profile.log 2>&1; tail -5 gpurun_out/r2_profile.log
