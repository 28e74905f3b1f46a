# usage: bash scripts/gpu_shapes.sh <tag> [configs...]   sampler launch shapes: parity + timing
TAG=${1:-sh}; shift; CFGS=${@:-c3 c2}
for SH in ${SHAPES:-g2 g4 g4x512}; do
  SLDA_SAMPLER=$SH timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity_${TAG}_${SH}.log 2>&1
  echo "$SH parity rc=$? $(tail -1 gpurun_out/parity_${TAG}_${SH}.log)"
  for CFG in $CFGS; do
    SLDA_SAMPLER=$SH timeout 600 python scripts/profile_run.py --config $CFG --iters 6 > gpurun_out/shape_${TAG}_${SH}_${CFG}.log 2>&1
    echo "$SH $CFG rc=$?"; grep "^iter" gpurun_out/shape_${TAG}_${SH}_${CFG}.log | tail -2
  done
done
