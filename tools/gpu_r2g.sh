python -c "import __graft_entry__ as g; g.build()"
for c in c2 c4; do python tools/decode_trace.py --per-block --lean-marks --config $c 2>&1 | head -7 | sed "s/^/$c: /"; done
