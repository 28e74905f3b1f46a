# Compact C_dk rows (default) vs wide (SLDA_ROW_FORMAT=wide): full GPU suite + per-kernel times + sampler ncu.
TAG=${1:-cp}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_${TAG}.log
for CFG in c3 c2 c4_shard c5_k10000 c5_k50000; do for F in compact wide; do
  SLDA_ROW_FORMAT=$F SLDA_SERIAL=1 timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/cp_${TAG}_${CFG}_${F}.log 2>&1
  echo "$CFG $F"; grep "^iter" gpurun_out/cp_${TAG}_${CFG}_${F}.log | tail -1 | cut -c1-130
done; done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:sampler -s 5 -c 1 --csv --log-file gpurun_out/ncu_${TAG}.csv python scripts/profile_run.py --config c3 --iters 7 > /dev/null 2>&1
grep -E "dram__bytes|gpu__time" gpurun_out/ncu_${TAG}.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
