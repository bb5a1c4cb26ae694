# k_scan_lb with batched pass-A loads: parity + timing
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_scan_chunked_gpu.py -q -x 2>&1 | tail -1
for c in "c2 1 2048" "c2 1 4096" "c3 1 2048" "c4 1 4096" "c2 2 2048"; do set -- $c
  timeout 300 python tools/scan_chunk_bench.py --config $1 --B $2 --T $3 2>&1 | tail -1
done
