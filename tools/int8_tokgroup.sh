# INT8 prefill: token-group sweep (config-3 wall clock, alternating)
for r in 1 2 3; do for G in 4 6 8; do
  echo "G $G: $(GLM_QMM_TOKGROUP=$G timeout 600 python tools/bench_prefill.py --bits 8 2>&1 | tail -1 | grep -o '"ms": [0-9.]*')"
done; done
