# Single-token integer-MMA GEMV shape sweep (one box): warps per CTA x ring depth x stage KB.
run() {
  GLM_M1_WARPS=$1 GLM_M1_STAGES=$2 GLM_M1_STAGE_KB=$3 GLM_PREFETCH=$4 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/s.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]);print('warps',sys.argv[1],'stages',sys.argv[2],'kb',sys.argv[3],'early',sys.argv[4],round(d['value'],2),'tok/s',round(d['ms_per_step'],3),'ms gemv',round(d['roofline']['gemv_ms_per_step'],3),d['clocks']['sm_mhz'])" $1 $2 $3 $4
}
for w in 6 8 10; do for sk in "2 8" "2 12" "2 16" "3 8" "3 12" "4 8"; do set -- $sk; run $w $1 $2 $1; done; done
run 4 2 16 2; run 4 4 12 4; run 12 2 8 2; run 16 2 6 2; run 8 2 8 2
