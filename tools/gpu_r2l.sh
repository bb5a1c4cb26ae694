set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "batched or splitk or zero_rows or bitlinear or contract" > gpurun_out/pytest_sab.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_sab.log
python tools/timeline.py --config c3 --B 64 --blocks 2 2>&1 | tail -13
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-flatness > gpurun_out/bench_sab_$c.log 2>&1; tail -1 gpurun_out/bench_sab_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['decode']['tokens_per_s'], d['decode']['batch_per_gpu'])"; done
timeout 300 python bench.py --config c4 --decode-batch 128 --steps 2 --warmup 3 --no-cpu-baseline --no-flatness > gpurun_out/bench_sab_c4b128.log 2>&1; tail -1 gpurun_out/bench_sab_c4b128.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 B128', d['decode']['tokens_per_s'])"
