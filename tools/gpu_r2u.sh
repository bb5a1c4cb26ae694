python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "two_sm or full_size or stack_truncated or batched" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_scan_chunked_gpu.py -q 2>&1 | tail -2
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'], d['clocks']['reasons'], {k: v['ms_per_launch'] for k, v in d['kernels']['by_shape'].items()})"; done
