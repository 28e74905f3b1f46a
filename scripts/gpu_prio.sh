# SSC side-stream priority (low = default, high) and fully serial, C3 steady state (iterations 7-8).
for MODE in low high serial; do
  if [ $MODE = serial ]; then ENVV="SLDA_SERIAL=1"; else ENVV="SLDA_SSC_PRIORITY=$MODE"; fi
  env $ENVV timeout 600 python scripts/profile_run.py --config c3 --iters 8 > gpurun_out/prio_$MODE.log 2>&1
  echo "$MODE"; grep "^iter" gpurun_out/prio_$MODE.log | tail -2 | cut -c1-200
done
