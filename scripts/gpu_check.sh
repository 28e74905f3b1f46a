set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/bench_c2.log
