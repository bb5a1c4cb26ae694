# balanced persistent GEMM grids (TERN_GEMM_BAL) vs grid = SMs, per-launch times
mkdir -p gpurun_out
for c in c2 c3; do for b in 0 1; do
TERN_GEMM_BAL=$b python tools/kernel_breakdown.py --config $c --prefill --blocks 2 > gpurun_out/bal_${c}_$b.txt 2>&1
echo "== $c BAL=$b"; grep -v "^$" gpurun_out/bal_${c}_$b.txt | tail -14
done; done
