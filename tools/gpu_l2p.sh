# experiment (result in DESIGN 6, profiles/r02_l2_persist_c2.txt): persisting L2 window on the
# residual stream.  It drove a patch to block_run (api.cu) that was not kept: once,
# cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, MB); per prefill block,
# cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow) over y (mode 1) or x
# (mode 2), hitRatio min(1, carve-out / bytes), hitProp persisting, missProp streaming.
mkdir -p gpurun_out
for cfg in "0 1" "64 1" "40 1" "64 2" "96 1"; do set -- $cfg
TERN_L2_PERSIST_MB=$1 TERN_L2_PERSIST_MODE=$2 python tools/kernel_breakdown.py --config c2 --prefill --blocks 4 > gpurun_out/l2p_$1_$2.txt 2>&1
echo "== MB=$1 mode=$2"; grep -v "^$" gpurun_out/l2p_$1_$2.txt | tail -10
done
