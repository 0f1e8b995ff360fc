# same-box sweep of one environment knob over bench.py: tools/gpu_sweep_env.sh VAR "v1 v2 ..." [rounds]
VAR=$1; VALS=$2; R=${3:-2}
for r in $(seq $R); do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/sw.log 2>&1
    python -c "import json,sys;d=json.loads(open('/tmp/sw.log').read().strip().splitlines()[-1]);print(sys.argv[1], round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['gemv_ms_per_step'],3), d['clocks']['sm_mhz'])" "$VAR=$v" || tail -3 /tmp/sw.log
  done
done
