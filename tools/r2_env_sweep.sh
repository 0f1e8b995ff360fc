# Same-box sweep of environment settings on the default bench (batch $BATCH, default 1):
#   tools/r2_env_sweep.sh ROUNDS "VAR=a" "VAR=b" ...
R=$1; shift
for r in $(seq $R); do
  for E in "$@"; do
    env $E timeout 300 python bench.py --batch ${BATCH:-1} --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > /tmp/ab.json 2>/dev/null
    python -c "import json,sys;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]);print(sys.argv[1], round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" "$E"
  done
done
