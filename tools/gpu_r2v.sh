python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "two_sm" 2>&1 | tail -1
run() { timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['value'], d['roofline']['frac'], {k: v['ms_per_launch'] for k, v in d['kernels']['by_shape'].items()})"; }
TERN_GEMM_2SM_NB=1 run c2 "nb1"
TERN_GEMM_2SM_NB=2 run c2 "nb2"
TERN_GEMM_2SM_NB=2 TERN_GEMM_2SM_KB=8 run c2 "nb2 kb8"
TERN_GEMM_2SM_NB=1 run c3 "nb1"
TERN_GEMM_2SM_NB=2 run c3 "nb2"
