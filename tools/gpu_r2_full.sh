# round 2 full check: build, smoke, full GPU suite, default bench, ncu launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke.txt 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu.txt 2>&1; echo pytest=$?
tail -5 gpurun_out/r02_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo bench=$?
CMD="python bench.py --steps 2 --warmup 3 --decode-steps 4 --no-cpu-baseline --no-flatness"
timeout 300 $CMD > gpurun_out/r02_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches_c2.csv $CMD > gpurun_out/r02_ncu.log 2>&1; echo ncu=$?
