# fused quantization (QFuse) first check: parity tests, kernel breakdown fused/unfused, short bench
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/qf_parity.log 2>&1; echo parity=$?
tail -5 gpurun_out/qf_parity.log
for c in c2 c3; do
  timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 > gpurun_out/qf_kb_$c.log 2>&1
  TERN_QFUSE=0 timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 > gpurun_out/qf_kb0_$c.log 2>&1
done
cat gpurun_out/qf_kb_c2.log gpurun_out/qf_kb0_c2.log
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-other-configs --decode-steps 4 --no-flatness > gpurun_out/qf_bench.log 2>&1; echo bench=$?
TERN_QFUSE=0 timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-other-configs --decode-steps 4 --no-flatness > gpurun_out/qf_bench0.log 2>&1; echo bench0=$?
tail -1 gpurun_out/qf_bench.log | cut -c1-300
tail -1 gpurun_out/qf_bench0.log | cut -c1-300
