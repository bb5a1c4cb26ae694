nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64 tools/micro/fp64.cu 2>/dev/null && /tmp/fp64 | grep -i redux
python -c "import __graft_entry__ as g; g.build()"
for c in c2 c4; do python tools/decode_trace.py --per-block --lean-marks --config $c 2>&1 | head -7 | sed "s/^/$c: /"; done
for st in 7; do for c in c2 c4; do TERN_GEMV_STRIP=$st python tools/decode_trace.py --per-block --lean-marks --config $c 2>&1 | sed -n 2p | sed "s/^/strip=$st $c: /"; done; done
