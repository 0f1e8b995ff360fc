# Batch-2 decode: multi-token integer-MMA GEMV (default) against the single-token family at
# two tokens (GLM_M1_TOKENS=2) on 8 / 12 / 16 warps.
for r in 1 2; do for cfg in "" "GLM_M1_TOKENS=2 GLM_M1_WARPS=8" "GLM_M1_TOKENS=2 GLM_M1_WARPS=12" "GLM_M1_TOKENS=2 GLM_M1_WARPS=16"; do
  env $cfg timeout 300 python bench.py --batch 2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/ab.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]);print('B2', sys.argv[1] or 'default', round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" "$cfg"
done; done
