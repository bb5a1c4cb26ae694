for fin in 0 1; do
for c in "c3" "c4 --decode-batch 128"; do
TERN_BENCH_FIN=$fin timeout 600 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --decode-steps 100 > /tmp/bb.log 2>&1; echo "fin=$fin $c: $(tail -1 /tmp/bb.log | python -c "import json,sys; D=json.loads(sys.stdin.read()); d=D['decode']; print(d['tokens_per_s'], d['ms_per_token_step'])")"
done
done
