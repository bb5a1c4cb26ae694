# round-toward-zero rha in k_quant: exhaustive selftest, parity, quant timing new vs old
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "selftest or bitlinear or quant" 2>&1 | tail -2
for c in c2 c3 c4; do
  echo "new $c: $(timeout 300 python tools/quant_time.py --config $c 2>&1 | tail -3 | tr '\n' ' ')"
  echo "old $c: $(TERN_LIB=$PWD/build/var_oldq/libtern.so timeout 300 python tools/quant_time.py --config $c 2>&1 | tail -3 | tr '\n' ' ')"
done
