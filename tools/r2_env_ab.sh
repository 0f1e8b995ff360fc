# Same-box A/B of an environment switch on the default bench: tools/r2_env_ab.sh "VAR=a" "VAR=b" [rounds]
A=$1; B=$2; R=${3:-2}
for r in $(seq $R); do
  for E in "$A" "$B"; do
    env $E timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/ab.json 2>/dev/null
    python -c "import json,sys;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]);print(sys.argv[1], round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" "$E"
  done
done
