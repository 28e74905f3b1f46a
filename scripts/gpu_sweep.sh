# K sweep (BASELINE C5, NYTimes shape) + C2 + C4 one-of-8 shard + C3 bench lines, no CPU baseline,
# then the self-launching N > 1 bench path with 8 ranks sharing the GPU (C2).
# usage: bash scripts/gpu_sweep.sh <tag>
TAG=${1:-s1}
for CFG in ${CFGS:-c2 c5_k100 c5_k10000 c5_k50000 c4_shard c3}; do
  timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline \
      > gpurun_out/sweep_${TAG}_${CFG}.json 2> gpurun_out/sweep_${TAG}_${CFG}.err
  echo "$CFG rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${TAG}_${CFG}.json')); print('$CFG', round(d['value']/1e9,3), 'Gtok/s', round(d['ms_per_step'],2), 'ms', 'sampler', round(d['kernels_ms']['sampler_ms'],2), 'frac', round(d['roofline']['frac'],3), 'E_t', round(d['roofline']['E_t'],1), 'e2e', round(d['e2e']['value']/1e9,3))" 2>&1 | tail -1
done
SLDA_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 8 --config c2 --steps 3 --warmup 3 > gpurun_out/sweep_${TAG}_c2_n8.json 2> gpurun_out/sweep_${TAG}_c2_n8.err
echo "c2 n=8 (one GPU) rc=$?"; tail -c 600 gpurun_out/sweep_${TAG}_c2_n8.json
