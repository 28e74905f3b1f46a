TAG=${1:-mb3}
timeout 300 ./scripts/mb_pattern 10 > gpurun_out/mb_pattern_${TAG}.log 2>&1; echo mb rc=$?
cat gpurun_out/mb_pattern_${TAG}.log
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --csv ./scripts/mb_pattern 10 > gpurun_out/mb_pattern_ncu_${TAG}.csv 2>&1; echo ncu rc=$?
for CFG in c3 c2; do
  SLDA_ROW_FORMAT=compact SLDA_SAMPLER=g4 timeout 600 python scripts/profile_run.py --config $CFG --iters 6 > gpurun_out/compact_g4_${CFG}_${TAG}.log 2>&1; echo compact g4 $CFG rc=$?
  grep "^iter" gpurun_out/compact_g4_${CFG}_${TAG}.log | tail -2
  SLDA_ROW_FORMAT=compact SLDA_SAMPLER=g2 timeout 600 python scripts/profile_run.py --config $CFG --iters 6 > gpurun_out/compact_g2_${CFG}_${TAG}.log 2>&1; echo compact g2 $CFG rc=$?
  grep "^iter" gpurun_out/compact_g2_${CFG}_${TAG}.log | tail -2
done
