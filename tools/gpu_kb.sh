for L in libtern.so libtern_head.so; do
TERN_LIB=$PWD/paper_2406_02528_b200/$L timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 50 > gpurun_out/bb.log 2>&1
echo "$L: $(tail -1 gpurun_out/bb.log | python -c "import json,sys; D=json.loads(sys.stdin.read()); k=D['kernels']; print(D['value'], D['roofline']['frac'], k['quant']['ms_per_launch'], k['fcgscan']['ms_per_launch'], {a: b['ms_per_launch'] for a, b in k['by_shape'].items()})")"
done
python tools/timeline.py --config c2 --blocks 1 --prefill | tail -10
python tools/timeline.py --config c4 --B 128 --blocks 1 | tail -12
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
