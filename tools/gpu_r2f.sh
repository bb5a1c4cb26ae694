set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stack_decode_gpu.py tests/test_shard_gpu.py -m gpu -q -x -k "decode or gemv or stack or shard or bitlinear" > gpurun_out/pytest_lean.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_lean.log
for c in c2 c4; do
  python tools/decode_trace.py --per-block --config $c 2>&1 | head -7 | sed "s/^/lean $c: /"
  TERN_GEMV_LD_AT=1 python tools/decode_trace.py --per-block --config $c 2>&1 | head -2 | sed "s/^/lean ld1 $c: /"
done
timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-flatness > gpurun_out/bench_lean.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_lean.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['decode']['tokens_per_s'])"
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-flatness > gpurun_out/bench_lean_$c.log 2>&1; tail -1 gpurun_out/bench_lean_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['decode']['tokens_per_s'], d['decode']['batch_per_gpu'])"; done
timeout 300 python bench.py --config c4 --decode-batch 1 --steps 2 --warmup 3 --no-cpu-baseline --no-flatness > gpurun_out/bench_lean_c4b1.log 2>&1; tail -1 gpurun_out/bench_lean_c4b1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 B1', d['decode']['tokens_per_s'])"
