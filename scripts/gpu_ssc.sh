# SSC / M-step measured alone (SLDA_SERIAL=1) and overlapped, plus parity of the SSC paths.
# usage: bash scripts/gpu_ssc.sh <tag>
TAG=${1:-s}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_streaming.py -m gpu -x -q > gpurun_out/ssc_${TAG}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/ssc_${TAG}_tests.log
for CFG in ${CFGS:-c3 c4_shard c2 c5_k50000}; do for SER in 1 0; do
  SLDA_SERIAL=$SER timeout 600 python scripts/profile_run.py --config $CFG --iters 6 > gpurun_out/ssc_${TAG}_${CFG}_${SER}.log 2>&1
  echo "$CFG serial=$SER"; grep "^iter" gpurun_out/ssc_${TAG}_${CFG}_${SER}.log | tail -1
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ssc --csv \
  --log-file gpurun_out/ssc_${TAG}_c4_launches.csv python scripts/profile_run.py --config c4_shard --iters 2 > /dev/null 2>&1
echo "ncu rc=$?"; grep -o '"slda::ssc[^"]*"[^$]*' gpurun_out/ssc_${TAG}_c4_launches.csv | awk -F'","' '{print $1, $NF}' | tail -8
