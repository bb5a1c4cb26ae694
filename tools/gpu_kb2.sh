python tools/kernel_breakdown.py --config c2 --prefill --B 8 --T 2048 --blocks 2 2>&1 | grep -E "per block|fcgscan"
python tools/kernel_breakdown.py --config c3 --prefill --B 16 --T 2048 --blocks 2 2>&1 | grep -E "fcgscan"
python -m pytest tests -q -x -m gpu -k "fused or prefill or block or centered or stack" 2>&1 | tail -1
