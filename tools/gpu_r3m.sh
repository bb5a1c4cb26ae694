# fcgscan phase-C conflict-free rows: parity + timing
python -c "import __graft_entry__ as g; g.build(); g.smoke()" || exit 1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "fused or full_size or c0_block or stack_truncated" 2>&1 | tail -2
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline --no-flatness --no-other-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['kernels']['fcgscan']['ms_per_launch'])"; done
rm -f gpurun_out/fcgtl_c2.txt; TERN_FS_TL=gpurun_out/fcgtl_c2.txt timeout 300 python tools/prof_block.py --config c2 --reps 3 && python tools/fcg_timeline.py gpurun_out/fcgtl_c2.txt > gpurun_out/fcgtl_c2.out
