# Row-format comparison: wide vs compact C_dk rows on several configs (iteration timings).
for CFG in c2 c3 c5_k10000 c5_k100; do
  for FMT in wide compact; do
    echo "== $CFG $FMT"
    SLDA_ROW_FORMAT=$FMT timeout 300 python scripts/profile_run.py --config $CFG --iters 4 2>&1 | grep iter | tail -2
  done
done
