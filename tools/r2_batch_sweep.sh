# Batched decode sweep (default kernels): bench.py --batch B.
: > gpurun_out/r2_batch_sweep.jsonl
for B in ${@:-1 2 3 4 8 12 16}; do
  timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /tmp/b.json 2>/dev/null
  tail -1 /tmp/b.json >> gpurun_out/r2_batch_sweep.jsonl
  python -c "import json,sys;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('B',d['config']['global_batch'],round(d['value'],1),'tok/s',round(d['ms_per_step'],2),'ms gemv',round(d['roofline']['gemv_ms_per_step'],2), d['clocks']['sm_mhz'])"
done
