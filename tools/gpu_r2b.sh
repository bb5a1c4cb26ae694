# round 2: GEMV latency anatomy (microbench, per-phase clocks, trace, ncu source)
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64 tools/micro/fp64.cu && /tmp/fp64 > gpurun_out/micro_fp64.log 2>&1
cat gpurun_out/micro_fp64.log
python -c "import __graft_entry__ as g; g.build()"
TERN_GEMV_PROF=1 python tools/prof_block.py --decode --reps 3 > gpurun_out/gemv_prof.log 2>&1
TERN_GEMV_PROF=1 python tools/prof_block.py --decode --reps 3 --config c4 >> gpurun_out/gemv_prof.log 2>&1
grep "gemv prof" gpurun_out/gemv_prof.log | tail -8
python tools/decode_trace.py --per-block > gpurun_out/trace_c2.log 2>&1; head -12 gpurun_out/trace_c2.log
CMD="python tools/prof_block.py --decode --reps 3"
$CMD > gpurun_out/dec_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 4 -c 1 -o gpurun_out/ncu_gemv_c2 $CMD > gpurun_out/ncu_gemv.log 2>&1; echo ncu=$?
