TAG=${1:-mb2}
timeout 300 ./scripts/mb_pattern 10 > gpurun_out/mb_pattern_${TAG}.log 2>&1; echo mb rc=$?
cat gpurun_out/mb_pattern_${TAG}.log
SLDA_TRACE=1 timeout 600 python scripts/e2e_breakdown.py --config c3 > gpurun_out/e2e_${TAG}.log 2>&1; echo e2e rc=$?
grep -v "^generate" gpurun_out/e2e_${TAG}.log | tail -22
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,dram__bytes_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum --csv ./scripts/mb_pattern 10 > gpurun_out/mb_pattern_ncu_${TAG}.csv 2>&1; echo ncu rc=$?
