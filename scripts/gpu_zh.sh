# C_k from the z histogram: GPU parity + per-kernel times (serial and overlapped).
TAG=${1:-zh}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_${TAG}.log
for CFG in c3 c5_k50000 c2; do for SER in 1 0; do
  SLDA_SERIAL=$SER timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/zh_${TAG}_${CFG}_${SER}.log 2>&1
  echo "$CFG serial=$SER"; grep "^iter" gpurun_out/zh_${TAG}_${CFG}_${SER}.log | tail -1 | cut -c1-160
done; done
