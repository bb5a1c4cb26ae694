# final evidence of the round: smoke, full GPU suite, default bench (driver's command), the
# reference arm, launch list of the bench command, backward launch list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
CMD="python bench.py --steps 2 --warmup 3 --decode-steps 4 --no-cpu-baseline --no-other-configs"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncul=$?
python tools/bwd_one.py > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bwd_ncu.csv python tools/bwd_one.py > /dev/null 2>&1; echo bwdncu=$?
timeout 600 python bench.py --config c3 --steps 3 --decode-steps 200 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 900 python bench.py --config c4 --steps 2 --decode-steps 100 --decode-batch 128 --no-cpu-baseline > gpurun_out/bench_c4b128.json 2> gpurun_out/bench_c4b128.err; echo c4=$?
