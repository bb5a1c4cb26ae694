# residual GEMM epilogue through registers (TERN_GEMM_RDIRECT=1) vs TMA staging
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in 0 1; do for c in c2 c3 c4; do echo "rdirect=$v $c $(TERN_GEMM_RDIRECT=$v timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 2>&1 | grep -i 'resid:n[0-9]*k[0-9]*' | head -1)"; done; done
TERN_GEMM_RDIRECT=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -2
