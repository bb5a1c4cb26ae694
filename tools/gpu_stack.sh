# persistent stack decode: new tests first (short timeout), then decode tests, then bench decode lines
set -x
timeout 300 python -m pytest tests/test_stack_decode_gpu.py -x -q > gpurun_out/pytest_stack.log 2>&1; echo stack_tests=$?
tail -15 gpurun_out/pytest_stack.log
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "decode or stack or c0" > gpurun_out/pytest_dec.log 2>&1; echo dec_tests=$?
tail -5 gpurun_out/pytest_dec.log
for c in c2 c4; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['decode']))"
done
timeout 600 python bench.py --config c4 --decode-batch 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4b4.log 2>&1; echo bench_c4b4=$?
tail -1 gpurun_out/bench_c4b4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['decode']))"
