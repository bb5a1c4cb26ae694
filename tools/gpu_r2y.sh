python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p /tmp/ncu
for c in c2 c3 c4; do
  CMD="python tools/prof_block.py --config $c --reps 1"
  timeout 300 $CMD > gpurun_out/tr_plain_$c.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"k_gemm|k_fcgscan|k_quant" -c 8 -o /tmp/ncu/r02_ncu_block_$c $CMD > gpurun_out/tr_ncu_$c.log 2>&1; echo "$c ncu=$?"
  python tools/ncu_traffic.py /tmp/ncu/r02_ncu_block_$c.ncu-rep --config $c --out gpurun_out/traffic_r02.json --desc "$c prefill, one block at the bench's batch (tools/prof_block.py --config $c), ncu --set full"
  ncu -i /tmp/ncu/r02_ncu_block_$c.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,launch__grid_size > gpurun_out/r02_ncu_block_$c.csv 2>&1
done
cp /tmp/ncu/r02_ncu_block_c2.ncu-rep gpurun_out/ 2>/dev/null; ls -la gpurun_out/ | tail -5
