timeout 900 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/pytest_s.log 2>&1; echo tests=$?
tail -15 gpurun_out/pytest_s.log
