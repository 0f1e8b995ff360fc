for PF in 0 32 64 128; do GLM_TC_PF=$PF timeout 300 python tools/r2_mk_probe.py 4 16; done
