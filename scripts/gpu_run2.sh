set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sampler|ssc_warp|phi_kernel" -s 3 -c 3 -o gpurun_out/prof_c2 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu_full.log
timeout 1200 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/bench_c3.log
