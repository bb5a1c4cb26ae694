# experiment: 4 ring stages in k_fcgscan (G aliased onto Bv: timing only, wrong values)
python -c "import __graft_entry__ as g; g.build()" || exit 1
rm -f gpurun_out/fcgtl_s4.txt
TERN_FS_TL=gpurun_out/fcgtl_s4.txt timeout 300 python tools/prof_block.py --config c2 --reps 3 && python tools/fcg_timeline.py gpurun_out/fcgtl_s4.txt > gpurun_out/fcgtl_s4.out; tail -3 gpurun_out/fcgtl_s4.out
timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 2>&1 | grep -i fcg
timeout 300 python tools/kernel_breakdown.py --config c4 --prefill --blocks 2 2>&1 | grep -i fcg
