# Next-batch row L2 prefetch A/B (SLDA_ROW_PREFETCH lines) + exact sparse-exchange bytes model.
TAG=${1:-pf}
for CFG in c3 c4_shard; do for PF in 0 2 3 4; do
  [ "$CFG" = c4_shard ] && [ "$PF" = 2 ] && continue
  SLDA_SERIAL=1 SLDA_ROW_PREFETCH=$PF timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/pf_${TAG}_${CFG}_${PF}.log 2>&1
  echo "$CFG pf=$PF"; grep "^iter" gpurun_out/pf_${TAG}_${CFG}_${PF}.log | tail -2
done; done
for PF in 0 3; do
  SLDA_ROW_PREFETCH=$PF timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:sampler -s 5 -c 1 --csv --log-file gpurun_out/ncu_${TAG}_pf${PF}.csv \
    python scripts/profile_run.py --config c3 --iters 7 > /dev/null 2>&1
  echo "ncu pf=$PF"; grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/ncu_${TAG}_pf${PF}.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
timeout 1200 python scripts/exchange_model.py --config c3 --iters 10 --ranks 2 4 8 > gpurun_out/exchange_model_${TAG}.log 2>&1
echo "exchange model rc=$?"; tail -4 gpurun_out/exchange_model_${TAG}.log
