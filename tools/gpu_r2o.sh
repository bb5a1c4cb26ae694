python -c "import __graft_entry__ as g; g.build()"
for dbg in 0 1 2 3; do TERN_SAB_DBG=$dbg TERN_SAB_PROF=1 python tools/prof_block.py --decode --config c3 --reps 2 2>&1 | grep "sab prof" | tail -4 | sed "s/^/dbg=$dbg /" | grep "n_rows=11264\|n_rows=6144"; done
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "batched" 2>&1 | tail -1
python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['decode']['tokens_per_s'])"
