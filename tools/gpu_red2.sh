# token-mixer residual in place too (TERN_RESID_RED=2: the quant of x copies x into y) vs 1
set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "full_size_prefill or two_sm_gemm_block or c0_block" > gpurun_out/red2_tests.log 2>&1; echo tests=$?
for v in 2 1; do
  TERN_RESID_RED=$v timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 > gpurun_out/red${v}x_c2.log 2>&1
  cat gpurun_out/red${v}x_c2.log
  TERN_RESID_RED=$v timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-other-configs --decode-steps 50 --no-flatness > gpurun_out/red${v}x_bench.json 2>&1
  tail -1 gpurun_out/red${v}x_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RED=$v', d['value'], d['roofline']['frac'], d['roofline']['frac_of_attainable'], d['e2e']['value'])"
done
