# N=2 bench path on one GPU (peer-memory exchange, gloo plumbing) + a quick N=1 sanity line
SLDA_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench2_c2.json 2> gpurun_out/bench2_c2.err
echo "N=2 rc=$?"; tail -c 1500 gpurun_out/bench2_c2.json; grep -i "error\|fail\|Traceback" gpurun_out/bench2_c2.err | head -5
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench1_c2.json 2>&1; echo "N=1 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench1_c2.json')); print('N=1', d['value']/1e9, d['ms_per_step'])"
