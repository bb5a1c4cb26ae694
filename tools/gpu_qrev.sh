# k_quant row order: ascending (TERN_QUANT_REV=0) vs descending (1, default), per-launch times
mkdir -p gpurun_out
for c in c2 c3; do for r in 0 1; do
TERN_QUANT_REV=$r python tools/kernel_breakdown.py --config $c --prefill --blocks 4 > gpurun_out/qrev_${c}_$r.txt 2>&1
echo "== $c TERN_QUANT_REV=$r"; grep -v "^$" gpurun_out/qrev_${c}_$r.txt | tail -9
done; done
