set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stack_decode_gpu.py tests/test_shard_gpu.py -m gpu -q -x -k "decode or gemv or stack or shard or bitlinear" > gpurun_out/pytest_lean.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_lean.log
for lean in 1 0; do
  for c in c2 c4; do
    TERN_GEMV_LEAN=$lean python tools/decode_trace.py --per-block --config $c 2>&1 | head -7 | sed "s/^/lean=$lean $c: /"
  done
done
TERN_GEMV_LEAN=1 TERN_GEMV_LD_AT=1 python tools/decode_trace.py --per-block --config c4 2>&1 | head -3 | sed "s/^/lean=1 ld1 c4: /"
