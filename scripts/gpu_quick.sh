# Quick iteration loop (one gpurun call): GPU parity tests, per-kernel times at C3 (SSC alone and
# overlapped) and an ncu --set full capture of one kernel.   usage: bash scripts/gpu_quick.sh <tag> [kernel-regex]
TAG=${1:-q}; KREG=${2:-ssc_warp}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_${TAG}.log
for CFG in c3 c2; do for SER in 1 0; do
  SLDA_SERIAL=$SER timeout 600 python scripts/profile_run.py --config $CFG --iters 6 > gpurun_out/kt_${TAG}_${CFG}_${SER}.log 2>&1
  echo "$CFG serial=$SER"; grep "^iter" gpurun_out/kt_${TAG}_${CFG}_${SER}.log | tail -1
done; done
SLDA_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREG" -s 5 -c 1 \
    -o gpurun_out/prof_${TAG} python scripts/profile_run.py --config c3 --iters 8 > /dev/null 2>&1
echo ncu rc=$?
