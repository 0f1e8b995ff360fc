# bring-up of the tcgen05 prefill attention: parity with both V descriptor conventions, timing
for cfg in "2048 128" "128 2048"; do
  set -- $cfg
  echo "== VLBO=$1 VSBO=$2"
  GLM_ATTN_VLBO=$1 GLM_ATTN_VSBO=$2 timeout 300 python -m pytest tests/test_gpu_model.py -x -q -k "head_dim_128" 2>&1 | grep -E "passed|failed|Error|error|assert" | head -5
done
