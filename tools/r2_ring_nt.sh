for r in 1 2; do for T in 256 512; do echo "NT $T $(GLM_ATTN_RING_NT=$T python tools/bench_block_decode.py 2>/dev/null | tail -1 | cut -c100-160)"; done; done
GLM_ATTN_RING_NT=512 timeout 300 python -m pytest tests/test_gpu_model.py -m gpu -q -x -k streaming 2>&1 | tail -1
