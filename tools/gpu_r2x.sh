python -c "import __graft_entry__ as g; g.build()" || exit 1
for m in out gather_q megatron seq; do
  timeout 600 python bench.py --shard $m --config c3 --steps 2 --warmup 3 --no-flatness --no-cpu-baseline --decode-steps 20 > gpurun_out/shard_$m.json 2> gpurun_out/shard_$m.err; echo "$m rc=$?"
  tail -1 gpurun_out/shard_$m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', d['value'], d['scaling'], d['config']['parallelism'], d.get('decode') and d['decode'].get('tokens_per_s'), d['comm'])" 2>&1 | tail -1
  grep -i "nccl communicator\|error\|Traceback" gpurun_out/shard_$m.err | head -3
done
