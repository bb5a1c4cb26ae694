# quick iteration: gpu parity tests, decode trace, short bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
python tools/decode_trace.py > gpurun_out/trace.log 2>&1
python tools/decode_trace.py --config c4 >> gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
timeout 600 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['decode'])"
