timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 50 > gpurun_out/bb.log 2>&1; echo rc=$?
tail -1 gpurun_out/bb.log | python -c "import json,sys; D=json.loads(sys.stdin.read()); print(D['value'], D['e2e'])"
tail -3 gpurun_out/bb.log | head -2
