for C in 0 1; do
TERN_FS_COUT=$C TERN_FS_PROF=1 python tools/kernel_breakdown.py --config c2 --prefill --B 8 --T 2048 --blocks 1 2>&1 | grep "fcgscan prof" | tail -1
TERN_FS_COUT=$C python tools/kernel_breakdown.py --config c2 --prefill --B 8 --T 2048 --blocks 2 2>&1 | grep -E "per block|fcgscan"
TERN_FS_COUT=$C python tools/kernel_breakdown.py --config c3 --prefill --B 16 --T 2048 --blocks 2 2>&1 | grep -E "per block|fcgscan"
done
python -m pytest tests -q -x -m gpu -k "fused or prefill or block or centered" 2>&1 | tail -1
