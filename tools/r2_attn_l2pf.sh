for r in 1 2; do for P in 0 1; do echo "L2PF $P $(GLM_ATTN_L2PF=$P python tools/bench_block_decode.py 2>/dev/null | tail -1 | cut -c100-160)"; done; done
GLM_ATTN_L2PF=1 python tools/timeline.py --layers 8 --prompt 2046 --first 16 2>&1 | grep "attn"
