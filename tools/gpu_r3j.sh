python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in 1 0; do for c in c2 c3 c4; do TERN_QUANT_GRIDSTRIDE=$v timeout 300 python bench.py --config $c --steps 3 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gs=$v $c', d['value'], d['kernels']['quant']['ms_per_launch'])"; done; done
