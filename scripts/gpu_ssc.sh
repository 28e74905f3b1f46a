# SSC variants measured alone (SLDA_SERIAL=1) and overlapped, C3 + C2
for SER in 1 0; do for SSC in bitmap sort; do
  SLDA_SERIAL=$SER SLDA_SSC=$SSC timeout 600 python scripts/profile_run.py --config c3 --iters 6 > gpurun_out/ssc_${SER}_${SSC}.log 2>&1
  echo "serial=$SER ssc=$SSC"; grep "^iter" gpurun_out/ssc_${SER}_${SSC}.log | tail -1
done; done
