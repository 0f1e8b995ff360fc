# bring-up of the tcgen05 prefill attention: parity with V descriptor variants, then timing
for cfg in "16384 1024" "1024 16384"; do
  set -- $cfg
  echo "== VLBO=$1 VSBO=$2"
  GLM_ATTN_VLBO=$1 GLM_ATTN_VSBO=$2 timeout 300 python -m pytest tests/test_gpu_model.py -x -q -k "head_dim_128" 2>&1 | grep -E "passed|failed|tap err" | head -3
done
bash tools/ncu_prefill_list.sh | grep -E "attn|total"
