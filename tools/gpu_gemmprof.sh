TERN_GEMM_PROF=1 python tools/prof_block.py --reps 1 > gpurun_out/gemm_prof.log 2>&1
TERN_GEMM_PROF=1 python tools/prof_block.py --reps 1 --config c3 --B 4 >> gpurun_out/gemm_prof.log 2>&1
grep "gemm prof" gpurun_out/gemm_prof.log
CMD="python tools/prof_block.py --reps 1"
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_quant|k_scan" -s 9 -c 9 -o gpurun_out/prof_pf2 $CMD > gpurun_out/ncu_pf2.log 2>&1; echo ncu=$?
