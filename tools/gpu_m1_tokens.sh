# parity of the GEMV paths, then GLM_M1_TOKENS variants at batch 2 and 4 (same box)
timeout 900 python -m pytest tests/test_gpu_qlinear.py tests/test_gpu_model.py -x -q 2>&1 | tail -2
for r in 1 2; do
  for B in 3 4; do
    for v in 2 4; do
      GLM_M1_TOKENS=$v timeout 300 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/b.log 2>&1
      python -c "import json;d=json.loads(open('/tmp/b.log').read().strip().splitlines()[-1]);print('M1_TOKENS=$v B=$B', round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" || tail -3 /tmp/b.log
    done
  done
done
