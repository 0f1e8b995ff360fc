# ncu --set full of the decode step's small kernels (LayerNorm, attention, GeGLU activation)
# at batch 1, GLM-130B shape, 4 layers; source-level with -lineinfo.
mkdir -p gpurun_out
for k in k_deepnorm_ln k_attn_decode k_geglu_act; do
  ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$k -c 2 \
      -o gpurun_out/r2_$k python tools/profile_decode.py --steps 1 --layers 4 > gpurun_out/r2_ncu_$k.log 2>&1
  echo "$k rc=$?"
  ncu -i gpurun_out/r2_$k.ncu-rep --page details --csv > gpurun_out/r2_${k}_details.csv 2>&1
  ncu -i gpurun_out/r2_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_${k}_source.csv 2>&1
done
