python -c "import __graft_entry__ as g; g.build()"
for st in 0 1 2 4 3 7; do for c in c2 c4; do TERN_GEMV_STRIP=$st python tools/decode_trace.py --per-block --lean-marks --config $c 2>&1 | sed -n 2p | sed "s/^/strip=$st $c: /"; done; done
