# k_scan_lb (carry alone on sub-partition 0): parity, timing, timeline, ncu kernel durations
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_scan_chunked_gpu.py -q -x 2>&1 | tail -1
timeout 300 python tools/scan_chunk_bench.py --config c2 --B 1 --T 2048 2>&1 | tail -2
rm -f gpurun_out/lbtl.txt
TERN_LB_TL=gpurun_out/lbtl.txt timeout 300 python tools/scan_chunk_bench.py --config c2 --B 1 --T 2048 > /dev/null 2>&1
python tools/lb_timeline.py gpurun_out/lbtl.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_scan" --csv python tools/scan_chunk_bench.py --config c2 --B 1 --T 2048 2>/dev/null | grep -E "k_scan" | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head
