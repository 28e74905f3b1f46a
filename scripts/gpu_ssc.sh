# SSC change check: parity (every-iteration digests incl. C_dk) + C3 / C2 / C4-shard times, serial and overlapped.
TAG=${1:-ssc}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_streaming.py -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_${TAG}.log
for CFG in c3 c2 c4_shard; do for SER in 1 0; do
  SLDA_SERIAL=$SER timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/ssc_${TAG}_${CFG}_${SER}.log 2>&1
  echo "$CFG serial=$SER"; grep "^iter" gpurun_out/ssc_${TAG}_${CFG}_${SER}.log | tail -1 | cut -c1-170
done; done
