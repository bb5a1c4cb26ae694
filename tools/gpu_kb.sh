TERN_FS_PROF=1 python tools/kernel_breakdown.py --config c2 --prefill --B 8 --T 2048 --blocks 1 2>&1 | grep "fcgscan prof" | tail -1
python tools/kernel_breakdown.py --config c2 --prefill --B 8 --T 2048 --blocks 2 2>&1 | tail -12
