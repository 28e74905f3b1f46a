for SH in "8200000,141000,738000000,10000" "300000,5000,27000000,10000" "150000,5000,13500000,10000" "1000000,20000,90000000,10000"; do
  timeout 600 python scripts/profile_run.py --config c3 --shape $SH --iters 8 > gpurun_out/l2exp_$SH.log 2>&1
  echo "$SH"; grep "^iter" gpurun_out/l2exp_$SH.log | tail -1
done
