python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
TERN_GEMM_PROF=1 python tools/prof_block.py --reps 2 2>&1 | grep "gemm prof" | tail -3
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -2
for r in 1 0; do TERN_GEMM_RES=$r python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('res=$r c2', d['value'], d['roofline']['frac'], d['kernels']['by_shape'])"; done
for r in 1 0; do TERN_GEMM_RES=$r python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('res=$r c3', d['value'], d['roofline']['frac'], d['kernels']['by_shape'])"; done
