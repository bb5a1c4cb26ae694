# k_quant threads-per-row sweep (TERN_QUANT_NVMAX), per-launch times of a c2 / c3 block
mkdir -p gpurun_out
for c in c2 c3; do for n in 8 4 2; do
TERN_QUANT_NVMAX=$n python tools/kernel_breakdown.py --config $c --prefill --blocks 2 > gpurun_out/qnv_${c}_$n.txt 2>&1
echo "== $c NVMAX=$n"; grep "quant\|per block" gpurun_out/qnv_${c}_$n.txt
done; done
