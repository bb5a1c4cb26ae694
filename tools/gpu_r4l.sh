# 128-wide residual GEMM tiles with 2-chunk residual lookahead and 4 ring stages (TERN_GEMM_RES128=1)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in 0 1; do for c in c2 c3; do echo "res128=$v $c $(TERN_GEMM_RES128=$v timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 2>&1 | grep -i 'resid:n[0-9]*k[0-9]*' | head -1)"; done; done
TERN_GEMM_RES128=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "full_size or c0_block or stack_truncated or two_sm" 2>&1 | tail -1
