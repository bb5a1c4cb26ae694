python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "full_size or two_sm or stack_truncated or fused or bitlinear" 2>&1 | tail -1
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 2 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], 'b1', d['prefill_b1']['tokens_per_s'], d['prefill_b1']['us_per_block'])"; done
