# phi kernel alone (serial engine) on C3 and C5 K=50K per SLDA_PHI_SHAPE (columns x stages).
# usage: SHAPES="16x8 32x4" bash scripts/gpu_phi.sh <tag>
TAG=${1:-p1}
for SH in ${SHAPES:-16x8}; do
for CFG in ${PCFGS:-c3 c5_k50000}; do
  SLDA_PHI_SHAPE=$SH SLDA_SERIAL=1 timeout 300 python scripts/profile_run.py --config $CFG --iters 4 \
      > gpurun_out/phi_${TAG}_${SH}_${CFG}.log 2>&1
  echo "shape=$SH $CFG $(grep -a '^iter 4' gpurun_out/phi_${TAG}_${SH}_${CFG}.log | grep -o 'phi_ms=[0-9.]*')"
done
done
