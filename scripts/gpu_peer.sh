# Sparse peer exchange: multi-rank parity on one GPU + the N>1 bench path (ranks sharing cuda:0).
# usage: bash scripts/gpu_peer.sh <tag>
TAG=${1:-peer}
timeout 1500 python -m pytest tests/test_peer_exchange.py -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest-peer rc=$?
tail -3 gpurun_out/pytest_${TAG}.log
for N in 2 4; do
  SLDA_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29$((500+N)) bench.py --gpus $N --steps 3 --warmup 3 --config c2 > gpurun_out/bench_${TAG}_c2_n$N.json 2> gpurun_out/bench_${TAG}_c2_n$N.err
  echo "c2 n=$N rc=$?"; tail -c 1500 gpurun_out/bench_${TAG}_c2_n$N.json
done
SLDA_BENCH_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29599 bench.py --gpus 2 --steps 3 --warmup 3 --config c3 > gpurun_out/bench_${TAG}_c3_n2.json 2> gpurun_out/bench_${TAG}_c3_n2.err
echo "c3 n=2 rc=$?"; tail -c 1500 gpurun_out/bench_${TAG}_c3_n2.json
