# A/B of an env switch at C3 and C2 (per-kernel times, steady state).  usage: bash scripts/gpu_ab.sh <tag> VAR v1 v2
TAG=$1; VAR=$2; shift 2
for CFG in c3 c2; do for VAL in "$@"; do
  env $VAR=$VAL timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/ab_${TAG}_${CFG}_${VAL}.log 2>&1
  echo "$CFG $VAR=$VAL"; grep "^iter" gpurun_out/ab_${TAG}_${CFG}_${VAL}.log | tail -2
done; done
