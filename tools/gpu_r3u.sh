# cross-CTA chunked scan (k_scan_lb): parity + timing vs sequential and the in-CTA chunked kernel
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_scan_chunked_gpu.py -q -x 2>&1 | tail -3
for c in "c2 1 2048" "c2 1 4096" "c3 1 2048" "c4 1 4096" "c2 2 2048"; do set -- $c
  echo "== $1 B=$2 T=$3 lb=1"; timeout 300 python tools/scan_chunk_bench.py --config $1 --B $2 --T $3 2>&1 | tail -2
  echo "== lb=0"; TERN_SCAN_LB=0 timeout 300 python tools/scan_chunk_bench.py --config $1 --B $2 --T $3 2>&1 | tail -1
done
