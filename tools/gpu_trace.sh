set -x
for m in 0 1 2; do
TERN_STACK_BAR=$m python tools/decode_trace.py --config c2 > gpurun_out/trace_c2_m$m.log 2>&1
TERN_STACK_BAR=$m python tools/decode_trace.py --config c4 > gpurun_out/trace_c4_m$m.log 2>&1
done
head -n 2 gpurun_out/trace_*.log
tail -n 17 gpurun_out/trace_c2_m2.log
