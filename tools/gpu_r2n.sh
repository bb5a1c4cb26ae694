python -c "import __graft_entry__ as g; g.build()"
TERN_SAB_PROF=1 python tools/prof_block.py --decode --config c3 --reps 2 2>&1 | grep "sab prof" | tail -4
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or zero_rows" 2>&1 | tail -1
python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['decode']['tokens_per_s'])"
python bench.py --config c4 --decode-batch 128 --steps 2 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 B128', d['decode']['tokens_per_s'])"
