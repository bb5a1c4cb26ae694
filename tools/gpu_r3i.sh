python -c "from paper_2406_02528_b200 import build as b; b.build(); b.build(trace=True)" || exit 1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_norm_centered_gpu.py -q -x -k "quant or full_size or stack_truncated or centred or centered or zero_rows" 2>&1 | tail -1
python tools/timeline.py --config c2 --prefill --B 8 --T 2048 --blocks 2 2>&1 | tail -9
for v in 1 0; do for c in c2 c3 c4; do TERN_QUANT_GRIDSTRIDE=$v timeout 300 python bench.py --config $c --steps 3 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gs=$v $c', d['value'], d['kernels']['quant']['ms_per_launch'])"; done; done
