# z transpose A/B (SLDA_ZMOVE=0: the sampler's direct z[slot] stores; default: execution-order
# stores + three coalesced passes, zmove.cu) + parity.  usage: bash scripts/gpu_zmove.sh <tag>
TAG=${1:-zm}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_streaming.py tests/test_peer_exchange.py -m gpu -x -q > gpurun_out/zm_${TAG}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/zm_${TAG}_tests.log
for CFG in ${CFGS:-c3 c2 c4_shard c5_k50000}; do for V in 0 1; do
  SLDA_ZMOVE=$V timeout 600 python scripts/profile_run.py --config $CFG --iters 8 > gpurun_out/zm_${TAG}_${CFG}_${V}.log 2>&1
  echo "$CFG ZMOVE=$V $(grep '^iter 8' gpurun_out/zm_${TAG}_${CFG}_${V}.log | grep -oE '(sampler_ms|zmove_ms|ssc_ms|total_ms)=[0-9.]*' | tr '\n' ' ')"
done; done
