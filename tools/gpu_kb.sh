timeout 900 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/ps.log 2>&1; echo tests=$?; tail -25 gpurun_out/ps.log
