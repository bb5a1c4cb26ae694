# split-K slice cap for decode batches (c3 B = 64, c4 B = 128)
for v in 0 2 4 8; do
  TERN_KS_CAP=$v timeout 300 python bench.py --config c3 --steps 1 --warmup 3 --decode-steps 100 --no-cpu-baseline --no-flatness > gpurun_out/ks${v}_c3.json 2>&1
  tail -1 gpurun_out/ks${v}_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cap $v c3 B64', d['decode']['tokens_per_s'])"
  TERN_KS_CAP=$v timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --decode-steps 50 --decode-batch 128 --no-cpu-baseline --no-flatness > gpurun_out/ks${v}_c4.json 2>&1
  tail -1 gpurun_out/ks${v}_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cap $v c4 B128', d['decode']['tokens_per_s'])"
done
