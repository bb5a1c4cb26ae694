timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in "c2" "c3" "c4 --decode-batch 128"; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --decode-steps 100 > gpurun_out/bb.log 2>&1
echo "$c: $(tail -1 gpurun_out/bb.log | python -c "import json,sys; D=json.loads(sys.stdin.read()); d=D['decode']; print(D['value'], D['roofline']['frac'], d['tokens_per_s'], d['ms_per_token_step'])")"
done
