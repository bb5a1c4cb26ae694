# batched decode: BN = 256 small-M tiles (fewer MMA instructions, split-K) vs the default 128
set -x
for c in c3 c4; do
  timeout 300 python tools/kernel_breakdown.py --config $c --blocks 2 > gpurun_out/dec_kb_$c.log 2>&1
  TERN_GEMM_BN=256 timeout 300 python tools/kernel_breakdown.py --config $c --blocks 2 > gpurun_out/dec_kb256_$c.log 2>&1
done
cat gpurun_out/dec_kb_c3.log gpurun_out/dec_kb256_c3.log gpurun_out/dec_kb_c4.log gpurun_out/dec_kb256_c4.log
