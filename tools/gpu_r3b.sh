python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 300 python bench.py --config $1 --steps 3 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['value'], {k: v['ms_per_launch'] for k, v in d['kernels']['by_shape'].items()})"; }
run c2 base
TERN_GEMM_2SM_RESID=1 TERN_GEMM_2SM_KB=8 run c2 "o-on-2sm"
run c3 base
TERN_GEMM_2SM_RESID=1 run c3 "o-on-2sm"
