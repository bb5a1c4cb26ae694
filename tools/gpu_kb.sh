timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for c in c2 c4; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --decode-steps 100 > /tmp/bb.log 2>&1; echo "$c: $(tail -1 /tmp/bb.log | python -c "import json,sys; D=json.loads(sys.stdin.read()); k=D['kernels']; d=D['decode']; print(D['value'], D['roofline']['frac'], k['quant']['ms_per_launch'], k['quant']['frac'], d['tokens_per_s'])")"
done
