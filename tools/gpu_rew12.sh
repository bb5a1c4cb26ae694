# residual-epilogue GEMM with 12 drain warps and a 2-stage ring (TERN_RES_EW12=1) vs default
set -x
TERN_RES_EW12=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "full_size_prefill or stack_truncated or c0_block" > gpurun_out/rew12_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/rew12_tests.log
for v in 1 0; do
  TERN_RES_EW12=$v timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 > gpurun_out/rew12_${v}_c2.log 2>&1
  TERN_RES_EW12=$v timeout 300 python tools/kernel_breakdown.py --config c3 --prefill --blocks 1 > gpurun_out/rew12_${v}_c3.log 2>&1
  grep 'resid:n' gpurun_out/rew12_${v}_c2.log gpurun_out/rew12_${v}_c3.log
  head -1 gpurun_out/rew12_${v}_c2.log
done
