# Batched decode A/B on one box: integer-MMA GEMVs (default) vs the fp16 HMMA kernels
# (GLM_GEMV_IMMA=0), bench.py --batch B for B in 1 2 3 4 8 12 16.
mkdir -p gpurun_out
: > gpurun_out/r2_batch_ab.jsonl
for B in 1 2 3 4 8 12 16; do
  for IM in 1 0; do
    GLM_GEMV_IMMA=$IM timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /tmp/b.json 2>/dev/null
    python -c "import json,sys;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);d['imma']=int(sys.argv[1]);print(json.dumps(d))" $IM >> gpurun_out/r2_batch_ab.jsonl
    python -c "import json,sys;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('B',d['config']['global_batch'],'imma',sys.argv[1],round(d['value'],1),'tok/s',round(d['ms_per_step'],2),'ms gemv',round(d['roofline']['gemv_ms_per_step'],2), d['clocks']['sm_mhz'])" $IM
  done
done
