python -c "from paper_2406_02528_b200 import build as b; b.build(); b.build(trace=True)" 
python tools/timeline.py --config c3 --B 64 --blocks 2 2>&1 | tail -30
python tools/timeline.py --config c3 --B 64 --blocks 2 --fin 2>&1 | tail -22
