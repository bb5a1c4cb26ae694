set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_seqpar_gpu.py tests/test_shard_gpu.py tests/test_stack_decode_gpu.py tests/test_symm_gpu.py -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu2.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-flatness --no-cpu-baseline > gpurun_out/bench_clk.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_clk.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'], d['roofline'])"
bash tools/gpu_r2b.sh
