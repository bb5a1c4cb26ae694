python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in 1 0; do
 for c in c2 c3; do TERN_GEMM_2SM=$v timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2sm=$v $c', d['value'], d['roofline']['frac'], {k: v['ms_per_launch'] for k, v in d['kernels']['by_shape'].items()})"; done
done
