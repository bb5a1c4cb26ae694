for BO in 0 16 32 64 128; do echo "BO=$BO"; TERN_FS_BACKOFF=$BO python tools/kernel_breakdown.py --config c2 --prefill --B 8 --T 2048 --blocks 2 2>&1 | grep -E "per block|fcgscan"; done
TERN_FS_BACKOFF=32 python tools/kernel_breakdown.py --config c3 --prefill --B 16 --T 2048 --blocks 2 2>&1 | grep -E "per block|fcgscan"
python tools/kernel_breakdown.py --config c3 --prefill --B 16 --T 2048 --blocks 2 2>&1 | grep -E "per block|fcgscan"
