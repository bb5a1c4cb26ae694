timeout 900 python -m pytest tests/test_norm_centered_gpu.py -x -q > gpurun_out/pytest_norm.log 2>&1; echo norm_tests=$?
tail -15 gpurun_out/pytest_norm.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 100 > gpurun_out/bb.log 2>&1
tail -1 gpurun_out/bb.log | python -c "import json,sys; D=json.loads(sys.stdin.read()); d=D['decode']; print(D['value'], D['roofline']['frac'], d['tokens_per_s'])"
