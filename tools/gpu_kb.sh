CMD="python tools/prof_block.py --config c4 --B 1 --decode --reps 3"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_gemv" -s 8 -c 4 -o gpurun_out/prof_gemv_c4 $CMD > gpurun_out/ncu_gemv.log 2>&1; echo ncu=$?
