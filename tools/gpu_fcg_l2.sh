# ncu: L2 / shared-memory / issue metrics of k_fcgscan at the c2 block shape
set -x
mkdir -p gpurun_out
python tools/prof_block.py > /dev/null 2>&1 || exit 1
M=gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sectors_op_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,sm__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__cycles_active.avg,sm__cycles_elapsed.max,lts__t_sector_hit_rate.pct
timeout 300 ncu --kernel-name regex:k_fcgscan --launch-skip 1 --launch-count 1 --metrics $M --clock-control none --csv --log-file gpurun_out/fcg_l2.csv python tools/prof_block.py > /dev/null 2>&1; echo ncu=$?
timeout 300 ncu --kernel-name regex:k_fcgscan --launch-skip 1 --launch-count 1 --metrics $M --clock-control none --csv --log-file gpurun_out/fcg_l2_c3.csv python tools/prof_block.py --config c3 > /dev/null 2>&1; echo ncu=$?
cat gpurun_out/fcg_l2.csv | tail -3
