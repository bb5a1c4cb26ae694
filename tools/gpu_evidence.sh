# round evidence: tests, smoke, default bench, c3/c4 bench lines, ncu launch list + full capture
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --config c3 --steps 3 --decode-steps 100 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 900 python bench.py --config c4 --steps 2 --decode-steps 50 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 900 python bench.py --config c4 --steps 2 --decode-steps 50 --decode-batch 128 --no-cpu-baseline > gpurun_out/bench_c4b128.json 2> gpurun_out/bench_c4b128.err; echo c4b128=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
CMD="python bench.py --steps 2 --warmup 3 --decode-steps 4 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncul=$?
CMD2="python tools/prof_block.py --reps 2"
$CMD2 > gpurun_out/pf_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_quant|k_fcgscan" -s 8 -c 8 -o gpurun_out/prof_block $CMD2 > gpurun_out/ncu_pf.log 2>&1; echo ncuf=$?
timeout 900 python tools/c1_sweep.py --out gpurun_out/c1_sweep.json > gpurun_out/c1.log 2>&1; echo c1=$?
