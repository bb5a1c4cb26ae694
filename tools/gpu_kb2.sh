python -m pytest tests -q -m gpu 2>&1 | tail -2
python tools/kernel_breakdown.py --config c3 --prefill --B 16 --T 2048 --blocks 2 2>&1 | grep -E "per block|fcgscan|swiglu"
python tools/kernel_breakdown.py --config c4 --prefill --B 32 --T 4096 --blocks 1 2>&1 | grep -E "per block|fcgscan|swiglu"
