python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_scan_chunked_gpu.py -q -x 2>&1 | tail -15
for c in "c2 1" "c2 2" "c4 1" "c3 1"; do set -- $c; python tools/scan_chunk_bench.py --config $1 --B $2; done
