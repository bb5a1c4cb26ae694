# fused quantization (QFuse): parity of block prefill, kernel breakdown fused/unfused (c2, c3)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "block or stack or prefill or glu or mlgru" > gpurun_out/qf_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/qf_parity.log
for c in c2 c3 c4; do
  timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 > gpurun_out/qf_kb_$c.log 2>&1
done
TERN_QFUSE=0 timeout 300 python tools/kernel_breakdown.py --config c4 --prefill --blocks 2 > gpurun_out/qf_kb0_c4.log 2>&1
cat gpurun_out/qf_kb_c*.log gpurun_out/qf_kb0_c4.log
