# Same-box A/B of an env knob: per-kernel times of 8 iterations at each config, knob off / on /
# off (usage: KNOB=SLDA_X CFGS="c3 c2" bash scripts/gpu_ab_env.sh <tag>)
TAG=${1:-ab}
for CFG in ${CFGS:-c3}; do for V in 0 1 0 1; do
  env ${KNOB}=$V timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/ab_${TAG}_${CFG}_${V}.log 2>&1
  echo "$CFG $KNOB=$V $(grep '^iter 8' gpurun_out/ab_${TAG}_${CFG}_${V}.log | grep -o 'sampler_ms=[0-9.]*') $(grep '^iter 8' gpurun_out/ab_${TAG}_${CFG}_${V}.log | grep -o 'total_ms=[0-9.]*')"
done; done
