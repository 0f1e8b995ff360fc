# token-group x weight-eviction sweep of the prefill GEMM: per-GEMM duration + DRAM bytes (ncu), config-3 wall clock
[ -n "$NOTEST" ] || timeout 900 python -m pytest tests/test_gpu_qlinear.py tests/test_gpu_model.py -x -q 2>&1 | tail -1
for cfg in ${CFGS:-"4 0" "4 1" "8 1" "16 1" "8 0"}; do
  set -- $cfg
  echo "== G $1 wevict $2"
  GLM_QMM_TOKGROUP=$1 GLM_QMM_WEVICT=$2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_qmm_tc -c 4 --csv python tools/bench_prefill.py --bits 4 --iters 1 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' '{print $NF}' | tr -d '"' | paste -sd' '
  GLM_QMM_TOKGROUP=$1 GLM_QMM_WEVICT=$2 timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c60-110
  GLM_QMM_TOKGROUP=$1 GLM_QMM_WEVICT=$2 timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c60-110
done
