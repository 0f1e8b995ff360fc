mkdir -p gpurun_out
python tools/mk_probe.py 16 12288 36864 4
python tools/mk_probe.py 16 12288 36864 8
ncu --set full --import-source on --clock-control none -k regex:k_gemv_mk -s 3 -c 1 -o gpurun_out/mk16_int4 python tools/mk_probe.py 16 12288 36864 4 > gpurun_out/ncu_mk.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gemv_mk -s 3 -c 1 -o gpurun_out/mk16_int8 python tools/mk_probe.py 16 12288 36864 8 >> gpurun_out/ncu_mk.log 2>&1
tail -3 gpurun_out/ncu_mk.log
