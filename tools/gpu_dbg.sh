set -x
TERN_GEMV_PROF=1 python tools/prof_block.py --decode --reps 3 > gpurun_out/gemv_prof.log 2>&1; echo $?
TERN_GEMV_PROF=1 python tools/prof_block.py --decode --reps 3 --config c4 >> gpurun_out/gemv_prof.log 2>&1; echo $?
