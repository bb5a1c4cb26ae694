# fcgscan: MMA tile period with and without the gate arithmetic (TERN_FS_NOGATE)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in 0 1; do rm -f gpurun_out/fcgtl_ng$v.txt
if [ $v = 1 ]; then export TERN_FS_NOGATE=1; fi
TERN_FS_TL=gpurun_out/fcgtl_ng$v.txt timeout 300 python tools/prof_block.py --config c2 --reps 3 && python tools/fcg_timeline.py gpurun_out/fcgtl_ng$v.txt > gpurun_out/fcgtl_ng$v.out; tail -4 gpurun_out/fcgtl_ng$v.out
done
unset TERN_FS_NOGATE
ncu --set full --clock-control none --import-source on -k regex:"k_fcgscan" -s 1 -c 1 -o gpurun_out/fcg_full python tools/prof_block.py --config c2 --reps 2 > gpurun_out/ncu_fcg.log 2>&1; echo ncu=$?
ncu -i gpurun_out/fcg_full.ncu-rep --page raw --csv > gpurun_out/fcg_full_raw.csv 2>/dev/null
ncu -i gpurun_out/fcg_full.ncu-rep --page details > gpurun_out/fcg_full_details.txt 2>/dev/null
