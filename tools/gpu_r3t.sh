# residual GEMM epilogue lookahead: (ring stages, staging tiles) = (2,4) main, (3,2) r32, (2,3) r23
python -c "import __graft_entry__ as g; g.build(); g.smoke()" || exit 1
for v in main r32 r23; do
  if [ $v = main ]; then unset TERN_LIB; else export TERN_LIB=$PWD/build/var_$v/libtern.so; fi
  for c in c2 c3 c4; do echo "$v $c"; timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 2>&1 | grep -i "resid"; done
done
unset TERN_LIB
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -2
