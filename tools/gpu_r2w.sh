python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1 || exit 1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "full_size or glu or stack_truncated or two_sm or fused" 2>&1 | tail -1
run() { timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['value'], d['roofline']['frac'], {k: v['ms_per_launch'] for k, v in d['kernels']['by_shape'].items()})"; }
TERN_GEMM_EW12=1 run c2 ew12
TERN_GEMM_EW12=0 run c2 ew8
