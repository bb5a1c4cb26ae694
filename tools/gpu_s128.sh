# ring depth of the 128-wide u8 tiles (decode batches, short prefills): 4 (default) vs 5
set -x
for v in default s128_5; do
  if [ $v = default ]; then export TERN_LIB=$PWD/paper_2406_02528_b200/libtern.so; else export TERN_LIB=$PWD/build/var_$v/libtern.so; fi
  timeout 300 python bench.py --config c3 --steps 2 --decode-steps 100 --no-cpu-baseline --no-flatness > gpurun_out/s128_${v}_c3.json 2>&1
  tail -1 gpurun_out/s128_${v}_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c3', d['decode']['tokens_per_s'], d['prefill_b1']['tokens_per_s'])"
  timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --decode-steps 50 --decode-batch 128 --no-cpu-baseline --no-flatness > gpurun_out/s128_${v}_c4.json 2>&1
  tail -1 gpurun_out/s128_${v}_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c4 B128', d['decode']['tokens_per_s'])"
done
