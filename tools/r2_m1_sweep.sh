# Single-token GEMV shape sweep on one box: warps per CTA, ring stages, stage size, early prefetch.
for cfg in "16 2 6 2" "16 2 8 2" "16 3 4 3" "12 2 8 2" "12 3 6 3" "8 3 8 3" "8 2 8 2" "16 2 4 2" "16 2 6 1" "20 2 4 2"; do
  set -- $cfg
  GLM_M1_WARPS=$1 GLM_M1_STAGES=$2 GLM_M1_STAGE_KB=$3 GLM_PREFETCH=$4 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/s.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]);print('warps',sys.argv[1],'stages',sys.argv[2],'kb',sys.argv[3],'early',sys.argv[4],round(d['value'],2),'tok/s',round(d['ms_per_step'],3),'ms gemv',round(d['roofline']['gemv_ms_per_step'],3),d['clocks']['sm_mhz'])" $1 $2 $3 $4
done
