# is the CTA-pair gate|up GEMM at K = 1024 (c2) drain-bound? pairs forced (TERN_GEMM_2SM_KB=8), full vs half drain (timing only)
python -c "import __graft_entry__ as g; g.build()" || exit 1
echo "1SM $(timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 2>&1 | grep -i swiglu)"
echo "2SM $(TERN_GEMM_2SM_KB=8 timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 2>&1 | grep -i swiglu)"
echo "2SM halfdrain $(TERN_LIB=$PWD/build/var_halfdrain/libtern.so TERN_GEMM_2SM_KB=8 timeout 300 python tools/kernel_breakdown.py --config c2 --prefill --blocks 2 2>&1 | grep -i swiglu)"
