for r in 1 2; do for W in 16 8 12; do
  GLM_M1_WARPS=$W timeout 300 python bench.py --batch 2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/ab.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]);print('B2 warps', sys.argv[1], round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" $W
done; done
