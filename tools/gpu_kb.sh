timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stack_decode_gpu.py -x -q -k "bitlinear or decode or c0 or persistent" > gpurun_out/pb.log 2>&1; echo tests=$?; tail -1 gpurun_out/pb.log
for c in c2 c4; do
timeout 600 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --decode-steps 200 > /tmp/bb.log 2>&1; echo "$c: $(tail -1 /tmp/bb.log | python -c "import json,sys; D=json.loads(sys.stdin.read()); d=D['decode']; print(d['tokens_per_s'], d['ms_per_token_step'])")"
done
