# ncu --set full of the sampler and phi at C2 (NYTimes, K=1K) and C5 K=50K (global-phi sampler),
# iteration 5 of each.  usage: bash scripts/gpu_ncu_configs.sh <tag>
TAG=${1:-r1}
for CFG in c2 c5_k50000; do
  timeout 900 ncu --set full --clock-control none -k regex:"sampler|phi_kernel" -s 8 -c 2 \
      -o gpurun_out/prof_${CFG}_${TAG} python scripts/profile_run.py --config $CFG --iters 6 > /dev/null 2>&1
  echo "$CFG ncu rc=$?"
done
