python -c "from paper_2406_02528_b200 import build as b; b.build(); b.build(trace=True)" || exit 1
python tools/timeline.py --config c2 --prefill --B 8 --T 2048 --blocks 1 2>&1 | tail -12
