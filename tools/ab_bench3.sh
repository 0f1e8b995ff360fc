# Alternate bench.py between three libraries on the same box: tools/ab_bench3.sh libA libB libC [rounds]
R=${4:-2}
for r in $(seq $R); do
  for L in "$1" "$2" "$3"; do
    GLM130B_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/ab.log 2>&1
    python -c "import json,sys;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);print(sys.argv[1], round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" "$L" || tail -3 /tmp/ab.log
  done
done
