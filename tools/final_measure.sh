# Round measurement pass: GPU tests, smoke, default bench, batch sweep, configs 2/3/5, ncu of the GEMM.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json
: > gpurun_out/batch_sweep.jsonl
for B in 1 2 4 8 16; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/batch_sweep.jsonl 2>/dev/null; done
python -c "
import json
for l in open('gpurun_out/batch_sweep.jsonl'):
    d=json.loads(l); print('B', d['config']['global_batch'], round(d['value'],1), 'tok/s', round(d['ms_per_step'],2), 'ms')"
timeout 900 python tools/bench_prefill.py > gpurun_out/prefill.jsonl 2>&1; cut -c1-160 gpurun_out/prefill.jsonl
timeout 600 python tools/bench_block_decode.py > gpurun_out/block_decode.json 2>&1; cut -c1-200 gpurun_out/block_decode.json
timeout 900 python tools/sweep_qlinear.py > gpurun_out/qlinear_sweep.jsonl 2>&1; wc -l gpurun_out/qlinear_sweep.jsonl
ncu --set full --import-source on --clock-control none -k regex:k_qmm_tc -s 2 -c 1 -o gpurun_out/qmm_int4_m2048 python tools/mk_probe.py 2048 12288 36864 4 > gpurun_out/ncu_qmm.log 2>&1; tail -1 gpurun_out/ncu_qmm.log
