python tools/kernel_breakdown.py --config c2 --prefill --B 1 --T 2048 --blocks 2 2>&1 | grep -E "per block|scan"
python tools/kernel_breakdown.py --config c2 --prefill --B 4 --T 2048 --blocks 2 2>&1 | grep -E "per block|scan"
python -m pytest tests -q -x -m gpu -k "scan or prefill or seqpar or centered or block" 2>&1 | tail -1
