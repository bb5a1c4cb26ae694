python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python bench.py > gpurun_out/r02_bench_full.json 2> gpurun_out/r02_bench_full.err; echo bench=$?
tail -1 gpurun_out/r02_bench_full.json | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', d['value'], 'frac', d['roofline']['frac'], 'traffic', d['roofline']['traffic'], d['clocks'])
print('kernels', {k: (v.get('frac'), v.get('share'), v.get('ms_per_launch')) for k, v in d['kernels'].items() if k != 'by_shape'})
print('decode', d['decode']['tokens_per_s'], 'e2e', d['e2e']['value'])
for c, o in d.get('other_configs', {}).items(): print(c, o.get('tokens_per_s'), o.get('roofline', {}).get('frac'), o.get('clocks'), o.get('error'))
"
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-flatness > gpurun_out/r02_bench_$c.json 2>/dev/null; tail -1 gpurun_out/r02_bench_$c.json | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$c', d['value'], d['roofline']['frac'], d['roofline']['traffic'], 'e2e', d['e2e']['value'], 'decode', d['decode']['tokens_per_s'], d['decode']['batch_per_gpu'], {k: (v.get('frac'), v.get('share'), v.get('ms_per_launch')) for k, v in d['kernels'].items() if k != 'by_shape'})"; done
timeout 600 python bench.py --config c4 --decode-batch 128 --steps 2 --no-cpu-baseline --no-flatness > gpurun_out/r02_bench_c4b128.json 2>/dev/null; tail -1 gpurun_out/r02_bench_c4b128.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 B128 decode', d['decode']['tokens_per_s'])"
