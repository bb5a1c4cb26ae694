CMD="python tools/prof_block.py --decode --reps 2 --config c4"
$CMD > gpurun_out/dec_plain.log 2>&1 && ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_gemv -s 6 -c 1 -o gpurun_out/prof_gemv3 $CMD > gpurun_out/ncu_gemv.log 2>&1; echo rc=$?
