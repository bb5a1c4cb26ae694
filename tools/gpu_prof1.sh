set -x
python tools/int8_peak.py > gpurun_out/int8_peak.json 2>&1; echo int8=$?
CMD="python tools/prof_block.py --decode --reps 6"
$CMD > gpurun_out/dec_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv $CMD > /dev/null 2>&1; echo declaunch=$?
ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 8 -c 4 -o gpurun_out/prof_gemv $CMD > gpurun_out/ncu_gemv.log 2>&1; echo gemvprof=$?
CMD2="python tools/prof_block.py --reps 2"
$CMD2 > gpurun_out/pf_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_quant|k_scan" -s 7 -c 7 -o gpurun_out/prof_prefill $CMD2 > gpurun_out/ncu_pf.log 2>&1; echo pfprof=$?
