python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stack_decode_gpu.py -q -x -k "decode or gemv or stack" 2>&1 | tail -1
for c in c2 c4; do python tools/decode_trace.py --per-block --lean-marks --config $c 2>&1 | head -7 | sed "s/^/$c: /"; done
python bench.py --steps 2 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 decode', d['decode']['tokens_per_s'])"
python bench.py --config c4 --steps 1 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 decode', d['decode']['tokens_per_s'])"
