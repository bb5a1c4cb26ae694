# cluster k_scan_lb: parity, timing, timeline
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_scan_chunked_gpu.py -q -x 2>&1 | tail -3
for c in "c2 1 2048" "c3 1 2048" "c2 2 2048" "c2 1 1024"; do set -- $c
  timeout 300 python tools/scan_chunk_bench.py --config $1 --B $2 --T $3 2>&1 | tail -2
done
rm -f gpurun_out/lbtl.txt
TERN_LB_TL=gpurun_out/lbtl.txt timeout 300 python tools/scan_chunk_bench.py --config c2 --B 1 --T 2048 2>&1 | tail -1
python tools/lb_timeline.py gpurun_out/lbtl.txt
