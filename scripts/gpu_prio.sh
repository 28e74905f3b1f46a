for PR in low high; do
  SLDA_SSC_PRIORITY=$PR timeout 600 python scripts/profile_run.py --config c3 --iters 6 > gpurun_out/prio_$PR.log 2>&1
  echo "ssc priority $PR"; grep "^iter" gpurun_out/prio_$PR.log | tail -2
done
