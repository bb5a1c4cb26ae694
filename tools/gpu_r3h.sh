python -c "from paper_2406_02528_b200 import build as b; b.build(); b.build(trace=True)" || exit 1
TERN_QUANT_CARVE=1 python tools/timeline.py --config c2 --prefill --B 8 --T 2048 --blocks 2 2>&1 | tail -10
for v in 1 0; do for c in c2 c3; do TERN_QUANT_CARVE=$v timeout 300 python bench.py --config $c --steps 3 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('carve=$v $c', d['value'], d['decode']['tokens_per_s'])"; done; done
