python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_scan_chunked_gpu.py -q -x 2>&1 | tail -2
for c in "c2 1 2048" "c2 1 4096" "c3 1 2048" "c4 1 4096" "c2 2 2048" "c3 2 2048"; do set -- $c
  timeout 300 python tools/scan_chunk_bench.py --config $1 --B $2 --T $3 2>&1 | tail -3
done
rm -f gpurun_out/lbtl.txt
TERN_LB_TL=gpurun_out/lbtl.txt timeout 300 python tools/scan_chunk_bench.py --config c2 --B 1 --T 2048 > /dev/null 2>&1
python tools/lb_timeline.py gpurun_out/lbtl.txt --launch -1
