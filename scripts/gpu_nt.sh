# CTA size of the 2-per-SM quad kernel (SLDA_QUAD_NT 512 / 576 / 640): parity + C3/C4-shard times.
TAG=${1:-nt}
SLDA_QUAD_NT=640 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "every_iteration" > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest-640 rc=$?
tail -1 gpurun_out/pytest_${TAG}.log
for CFG in c3 c4_shard c5_k10000; do for NT in 512 576 640; do
  SLDA_QUAD_NT=$NT SLDA_SERIAL=1 timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/nt_${TAG}_${CFG}_${NT}.log 2>&1
  echo "$CFG nt=$NT"; grep "^iter" gpurun_out/nt_${TAG}_${CFG}_${NT}.log | tail -1 | cut -c1-100
done; done
