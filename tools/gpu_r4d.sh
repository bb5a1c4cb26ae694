python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_scan_lb" -s 3 -c 1 -o gpurun_out/lb_full python tools/scan_chunk_bench.py --config c2 --B 1 --T 2048 > gpurun_out/ncu_lb.log 2>&1; echo ncu=$?
ncu -i gpurun_out/lb_full.ncu-rep --page details > gpurun_out/lb_details.txt 2>/dev/null
ncu -i gpurun_out/lb_full.ncu-rep --page source --csv --print-source sass > gpurun_out/lb_sass.csv 2>/dev/null
rm -f gpurun_out/lb_full.ncu-rep
