set -x
python -c "import __graft_entry__ as g; g.build()"
for ld in 0 1 2; do
  for c in c2 c4; do
    TERN_GEMV_LD_AT=$ld python tools/decode_trace.py --per-block --config $c 2>&1 | head -8 | sed "s/^/ld=$ld $c: /"
  done
done
