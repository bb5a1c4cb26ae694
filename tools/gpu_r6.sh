# after making QFuse a compile-time variant: default-path timing restored?, QFuse parity,
# batched-decode BN=256 experiment
set -x
timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 > gpurun_out/r6_kb_c2.log 2>&1
cat gpurun_out/r6_kb_c2.log
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-other-configs --decode-steps 100 --no-flatness > gpurun_out/r6_bench.json 2>&1; echo bench=$?
tail -1 gpurun_out/r6_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['decode']['tokens_per_s'])"
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "qfuse or two_sm or stack_truncated or bitlinear" > gpurun_out/r6_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r6_tests.log
bash tools/gpu_dec1.sh
