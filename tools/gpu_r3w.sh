python -c "import __graft_entry__ as g; g.build()" || exit 1
rm -f gpurun_out/lbtl.txt
TERN_LB_TL=gpurun_out/lbtl.txt timeout 300 python tools/scan_chunk_bench.py --config c2 --B 1 --T 2048 2>&1 | tail -1
python tools/lb_timeline.py gpurun_out/lbtl.txt > gpurun_out/lbtl.out; cat gpurun_out/lbtl.out
