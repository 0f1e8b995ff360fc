#!/bin/bash
# Alternate bench.py between two libraries on the same box: tools/ab_bench.sh libA libB [rounds]
A=$1; B=$2; R=${3:-2}
for r in $(seq $R); do
  for L in "$A" "$B"; do
    GLM130B_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/ab.log 2>&1
    python -c "import json,sys;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);print(sys.argv[1], round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" "$L"
  done
done
