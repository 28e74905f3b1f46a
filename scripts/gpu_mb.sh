# usage: bash scripts/gpu_mb.sh <tag>   staging microbench + e2e breakdown (+ ncu of the microbench)
TAG=${1:-mb}
timeout 300 ./scripts/mb_stage 12 > gpurun_out/mb_stage_${TAG}.log 2>&1; echo mb rc=$?
cat gpurun_out/mb_stage_${TAG}.log
SLDA_TRACE=1 timeout 600 python scripts/e2e_breakdown.py --config c3 > gpurun_out/e2e_${TAG}.log 2>&1; echo e2e rc=$?
cat gpurun_out/e2e_${TAG}.log
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed --csv -c 12 ./scripts/mb_stage 12 > gpurun_out/mb_ncu_${TAG}.csv 2>&1; echo ncu rc=$?
