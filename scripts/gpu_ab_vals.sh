# Same-box A/B of an env knob over several values: per-kernel times of 8 iterations per value,
# the sequence run twice (usage: KNOB=SLDA_X VALS="0 1 2" CFGS="c3" bash scripts/gpu_ab_vals.sh <tag>)
TAG=${1:-ab}
for CFG in ${CFGS:-c3}; do for rep in 1 2; do for V in ${VALS:-0 1}; do
  env ${KNOB}=$V timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/ab_${TAG}_${CFG}_${V}_${rep}.log 2>&1
  echo "$CFG $KNOB=$V $(grep '^iter 8' gpurun_out/ab_${TAG}_${CFG}_${V}_${rep}.log | grep -o 'sampler_ms=[0-9.]*') $(grep '^iter 8' gpurun_out/ab_${TAG}_${CFG}_${V}_${rep}.log | grep -o 'total_ms=[0-9.]*')"
done; done; done
