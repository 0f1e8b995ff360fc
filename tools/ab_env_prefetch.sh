#!/bin/bash
for r in 1 2; do for e in 2 1 0; do
GLM_PREFETCH=$e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/ab.log 2>&1
python -c "import json,sys;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);print('early', sys.argv[1], round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" $e
done; done
