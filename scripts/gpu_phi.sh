# phi kernel alone (serial engine) on C3 and C5 K=50K per SLDA_PHI_STAGES x SLDA_PHI_PF, plus one ncu capture.
# usage: STAGES="2 4" PFS="0 256" bash scripts/gpu_phi.sh <tag>
TAG=${1:-p1}
for S in ${STAGES:-4}; do
for PF in ${PFS:-256}; do
for CFG in c3 c5_k50000; do
  SLDA_PHI_PF=$PF SLDA_PHI_STAGES=$S SLDA_SERIAL=1 timeout 300 python scripts/profile_run.py --config $CFG --iters 4 \
      > gpurun_out/phi_${TAG}_${S}_${PF}_${CFG}.log 2>&1
  echo "stages=$S pf=$PF $CFG $(grep iter gpurun_out/phi_${TAG}_${S}_${PF}_${CFG}.log | tail -1 | grep -o 'phi_ms=[0-9.]*')"
done
done
done
[ -n "$NONCU" ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:"phi_kernel" -s 2 -c 1 \
    -o gpurun_out/prof_phi_k50k_${TAG} python scripts/profile_run.py --config c5_k50000 --iters 3 > /dev/null 2>&1
echo ncu rc=$?
