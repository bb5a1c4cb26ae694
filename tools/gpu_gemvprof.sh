TERN_GEMV_PROF=1 python tools/prof_block.py --decode --reps 2 > gpurun_out/gemv_prof.log 2>&1
TERN_GEMV_PROF=1 python tools/prof_block.py --decode --reps 2 --config c4 >> gpurun_out/gemv_prof.log 2>&1
grep "gemv prof" gpurun_out/gemv_prof.log | tail -8
