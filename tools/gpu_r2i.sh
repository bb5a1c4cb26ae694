python -c "import __graft_entry__ as g; g.build()"
for w in 1 0 1 0; do for c in c2 c4; do TERN_GEMV_PARAM_WARM=$w python tools/decode_trace.py --per-block --lean-marks --config $c 2>&1 | sed -n 2p | sed "s/^/warm=$w $c: /"; done; done
