# prefill iteration: gpu tests, gemm wait profile, short bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
TERN_GEMM_PROF=1 python tools/prof_block.py --reps 1 > gpurun_out/gemm_prof.log 2>&1
grep "gemm prof" gpurun_out/gemm_prof.log
timeout 600 python bench.py --steps 3 --no-cpu-baseline --decode-steps 50 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'])
for k,v in d['kernels'].items():
    print(k, v)"
