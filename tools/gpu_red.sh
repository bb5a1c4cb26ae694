# in-place channel-mixer residual (EPI_RESID_RED, TMA reduce-add): parity + timing vs off
set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "full_size_prefill or stack_truncated or c0_block or two_sm or qfuse or crosses" > gpurun_out/red_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/red_tests.log
for v in 1 0; do
  TERN_RESID_RED=$v timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 > gpurun_out/red${v}_c2.log 2>&1
  cat gpurun_out/red${v}_c2.log
  TERN_RESID_RED=$v timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-other-configs --decode-steps 50 --no-flatness > gpurun_out/red${v}_bench.json 2>&1
  tail -1 gpurun_out/red${v}_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RED=$v', d['value'], d['roofline']['frac'], d['roofline']['frac_of_attainable'], d['e2e']['value'])"
done
