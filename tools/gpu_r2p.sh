python -c "import __graft_entry__ as g; g.build()"
run() { python bench.py --config $1 --decode-batch $2 --steps 1 --warmup 3 --no-cpu-baseline --no-flatness 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 B$2 $3', d['decode']['tokens_per_s'])"; }
for cfg in "c3 64" "c4 128"; do
  TERN_GEMM_SAB=0 run $cfg "old(u8,BN128)"
  TERN_GEMM_SAB=0 TERN_GEMM_BN=256 run $cfg "u8,BN256"
  TERN_GEMM_SAB=0 TERN_SMALLM_PRE=0 TERN_GEMM_BN=256 run $cfg "2bit,BN256"
  TERN_GEMM_SAB=0 TERN_SMALLM_PRE=0 run $cfg "2bit,BN128"
  TERN_GEMM_SAB=1 run $cfg "sab"
done
