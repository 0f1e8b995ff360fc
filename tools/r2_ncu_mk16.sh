# ncu --set full of the integer-MMA multi-token GEMV (k_gemv_mk_i4) at 16 tokens, qkv shape
mkdir -p gpurun_out
cat > /tmp/mk16.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2210_02414_b200 import glm
q = glm.QLinear.synthetic(1, 3, 12288, 36864, 5.6e-4, 4, "column")
print(q.plan(16), q.bench(16, iters=5, flush=False))
PY
ncu --set full --import-source on --clock-control none -k regex:k_gemv_mk_i4 -s 3 -c 1 -o gpurun_out/r2_mk16 python /tmp/mk16.py > gpurun_out/r2_ncu_mk16.log 2>&1
ncu -i gpurun_out/r2_mk16.ncu-rep --page details --csv > gpurun_out/r2_mk16_details.csv 2>&1
ncu -i gpurun_out/r2_mk16.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_mk16_source.csv 2>&1
tail -2 gpurun_out/r2_ncu_mk16.log
