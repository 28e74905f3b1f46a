# A/B of SLDA_DEEP (two row groups in flight per warp) + parity with it forced.
TAG=${1:-dp}
SLDA_DEEP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "every_iteration" > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest-deep rc=$?
tail -2 gpurun_out/pytest_${TAG}.log
for CFG in c3 c4_shard; do for D in 0 1; do
  SLDA_SERIAL=1 SLDA_DEEP=$D timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/dp_${TAG}_${CFG}_${D}.log 2>&1
  echo "$CFG deep=$D"; grep "^iter" gpurun_out/dp_${TAG}_${CFG}_${D}.log | tail -2 | cut -c1-120
done; done
