for B in 1 2 4 8; do python tools/kernel_breakdown.py --config c2 --prefill --B $B --T 2048 --blocks 2 2>&1 | grep -E 'per block'; done
for B in 1 2 4; do python tools/kernel_breakdown.py --config c3 --prefill --B $B --T 2048 --blocks 2 2>&1 | grep -E 'per block'; python tools/kernel_breakdown.py --config c3 --prefill --B $B --T 2048 --blocks 2 --unfused 2>&1 | grep -E 'per block'; done
for B in 1 2; do python tools/kernel_breakdown.py --config c4 --prefill --B $B --T 4096 --blocks 2 2>&1 | grep -E 'per block'; python tools/kernel_breakdown.py --config c4 --prefill --B $B --T 4096 --blocks 2 --unfused 2>&1 | grep -E 'per block'; done
python -m pytest tests -q -x -m gpu 2>&1 | tail -3
