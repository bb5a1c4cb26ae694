CMD="python tools/prof_block.py --reps 2"
$CMD > gpurun_out/pf_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_fcgscan" -s 1 -c 1 -o gpurun_out/prof_fs $CMD > gpurun_out/ncu_fs.log 2>&1; echo ncu=$?
