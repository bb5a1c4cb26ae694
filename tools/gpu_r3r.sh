# fcgscan: g^ via TMEM staged into dead Bv rows, channel-mapped C, 4 stages
python -c "import __graft_entry__ as g; g.build(); g.smoke()" || exit 1
for c in c2 c3 c4; do echo "main $c $(timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 2>&1 | grep -i fcg)"; done
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "fused or full_size or c0_block or stack_truncated" 2>&1 | tail -2
