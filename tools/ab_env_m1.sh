#!/bin/bash
# same-box sweep of the single-token GEMV shape knobs (warps per CTA, weight stage size)
for cfg in ${CFGS:-"16 6" "20 4" "24 4" "20 6" "18 4"}; do set -- $cfg
  GLM_M1_WARPS=$1 GLM_M1_STAGE_KB=$2 timeout 120 python tools/gemv_m1_sweep.py | tail -1 | sed "s/^/w$1 kb$2 /"
done
