# ncu source-level profile of the decode LayerNorm (k_deepnorm_ln<8>) over many launches
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_deepnorm_ln -c 30 \
    -o /tmp/r2_ln30 python tools/profile_decode.py --steps 1 --layers 16 > gpurun_out/r2_ncu_ln30.log 2>&1
ncu -i /tmp/r2_ln30.ncu-rep --page source --csv --print-source sass > /tmp/r2_ln30_source.csv 2>&1; python tools/ncu_source_agg.py /tmp/r2_ln30_source.csv > gpurun_out/r2_ln30_agg.txt
tail -2 gpurun_out/r2_ncu_ln30.log
