# L4-free tree (L8 + phi re-derivation): full GPU suite + per-kernel times + phi ncu.
TAG=${1:-lf}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_${TAG}.log
for CFG in c3 c2 c5_k50000 c4_shard; do
  SLDA_SERIAL=1 timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/lf_${TAG}_${CFG}.log 2>&1
  echo "$CFG"; grep "^iter" gpurun_out/lf_${TAG}_${CFG}.log | tail -1 | cut -c1-130
done
timeout 600 python scripts/profile_run.py --config c3 --iters 8 > gpurun_out/lf_${TAG}_c3_overlap.log 2>&1
echo "c3 overlapped"; grep "^iter" gpurun_out/lf_${TAG}_c3_overlap.log | tail -1 | cut -c1-130
