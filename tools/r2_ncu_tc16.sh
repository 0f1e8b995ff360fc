# ncu --set full of the tcgen05 integer decode GEMV (k_gemv_tc_i4) at 16 tokens, qkv shape
mkdir -p gpurun_out
cat > /tmp/tc16.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2210_02414_b200 import glm
q = glm.QLinear.synthetic(1, 3, 12288, 36864, 5.6e-4, 4, "column")
print(q.plan(16), q.bench(16, iters=5, flush=False))
PY
ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc_i4 -s 3 -c 1 -o /tmp/r2_tc16 python /tmp/tc16.py > gpurun_out/r2_ncu_tc16.log 2>&1
ncu -i /tmp/r2_tc16.ncu-rep --page details --csv > gpurun_out/r2_tc16_details.csv 2>&1
ncu -i /tmp/r2_tc16.ncu-rep --page source --csv --print-source sass > /tmp/r2_tc16_source.csv 2>&1
python tools/ncu_source_agg.py /tmp/r2_tc16_source.csv > gpurun_out/r2_tc16_source_top.txt 2>&1
tail -2 gpurun_out/r2_ncu_tc16.log
