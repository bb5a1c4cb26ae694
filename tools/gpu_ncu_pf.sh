CMD="python tools/prof_block.py --reps 2"
$CMD > gpurun_out/pf_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_quant|k_scan" -s 9 -c 9 -o gpurun_out/prof_pf3 $CMD > gpurun_out/ncu_pf3.log 2>&1; echo ncu=$?
