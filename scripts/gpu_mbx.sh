# Sparse-exchange kernels alone at C3's shape (scripts/mb_exchange.cu): time + ncu --set full.
TAG=${1:-mbx}
./scripts/mb_exchange 141000 10000 110000000 6 > gpurun_out/mbx_${TAG}.json 2>&1; echo rc=$?; cat gpurun_out/mbx_${TAG}.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparsify|gather_add" -s 2 -c 2 \
  -o gpurun_out/prof_exchange_${TAG} ./scripts/mb_exchange 141000 10000 110000000 3 > /dev/null 2>&1; echo ncu rc=$?
timeout 600 python scripts/profile_heldout.py > gpurun_out/heldout_${TAG}.log 2>&1; echo heldout rc=$?; cat gpurun_out/heldout_${TAG}.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"heldout" -c 1 \
  -o gpurun_out/prof_heldout_${TAG} python scripts/profile_heldout.py > /dev/null 2>&1; echo ncu-heldout rc=$?
