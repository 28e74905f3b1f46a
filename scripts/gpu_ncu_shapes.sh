# usage: SHAPES="g4 s4" bash scripts/gpu_ncu_shapes.sh <tag> <config>  -- one ncu --set full sampler capture per shape
TAG=${1:-n}; CFG=${2:-c3}
for SH in ${SHAPES:-g4 s4}; do
  SLDA_SAMPLER=$SH timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sampler" -s 2 -c 1 \
    -o gpurun_out/prof_${CFG}_${TAG}_${SH} python scripts/profile_run.py --config $CFG --iters 3 > gpurun_out/prof_${CFG}_${TAG}_${SH}.log 2>&1
  echo "$SH ncu rc=$?"
done
