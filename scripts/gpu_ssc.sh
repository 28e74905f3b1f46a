# SSC / M-step measured alone (SLDA_SERIAL=1) and overlapped, C3 (+ C5 K=50K: M-step heavy)
for CFG in c3 c5_k50000; do for SER in 1 0; do
  SLDA_SERIAL=$SER timeout 600 python scripts/profile_run.py --config $CFG --iters 6 > gpurun_out/ssc_${CFG}_${SER}.log 2>&1
  echo "$CFG serial=$SER"; grep "^iter" gpurun_out/ssc_${CFG}_${SER}.log | tail -1
done; done
