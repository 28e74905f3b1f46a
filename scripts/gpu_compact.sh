# compact vs wide C_dk rows with the default (quad) sampler + bitmap SSC: parity and timing
SLDA_ROW_FORMAT=compact timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "compact or variants" 2>&1 | tail -1
for CFG in c3 c2 c5_k10000; do for FMT in wide compact; do
  SLDA_ROW_FORMAT=$FMT timeout 600 python scripts/profile_run.py --config $CFG --iters 6 > gpurun_out/fmt_${CFG}_${FMT}.log 2>&1
  echo "$CFG $FMT"; grep "^iter" gpurun_out/fmt_${CFG}_${FMT}.log | tail -1
done; done
