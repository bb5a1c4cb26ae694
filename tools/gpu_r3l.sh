# k_fcgscan CTA-0 phase timeline (TERN_FS_TL) at c2 and c4 shapes
python -c "import __graft_entry__ as g; g.build()" || exit 1
rm -f gpurun_out/fcgtl_*.txt
TERN_FS_TL=gpurun_out/fcgtl_c2.txt timeout 300 python tools/prof_block.py --config c2 --reps 3 && python tools/fcg_timeline.py gpurun_out/fcgtl_c2.txt > gpurun_out/fcgtl_c2.out
TERN_FS_TL=gpurun_out/fcgtl_c4.txt timeout 300 python tools/prof_block.py --config c4 --reps 3 && python tools/fcg_timeline.py gpurun_out/fcgtl_c4.txt > gpurun_out/fcgtl_c4.out
