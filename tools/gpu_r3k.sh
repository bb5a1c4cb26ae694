# residual L2 prefetch (TERN_GEMM_RPF) A/B: throughput + per-GEMM times, and the residual parity tests
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in 1 0 1; do for c in c2 c3 c4; do TERN_GEMM_RPF=$v timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rpf=$v $c', d['value'], d['kernels']['gemm']['ms_per_launch'], d['kernels']['gemm']['frac'])"; done; done
for v in 1 0; do for c in c2 c4; do echo "rpf=$v $c"; TERN_GEMM_RPF=$v timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 2>&1 | grep -i gemm; done; done
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -3
