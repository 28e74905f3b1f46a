# Full measurement pass (one gpurun call): tests, bench, ncu launch list, ncu --set full
# captures of the iteration kernels.  usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r1}
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu_${TAG}.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_${TAG}.log
timeout 1200 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_${TAG}.json
# launch list: every kernel of 2 C3 iterations (+ setup), device time per launch
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_${TAG}.csv python scripts/profile_run.py --config c3 --iters 2 > /dev/null 2>&1
echo ncu-list rc=$?
# full captures at steady state (iteration 13, as bench.py's timed iterations): sampler, SSC, phi
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sampler" -s 12 -c 1 \
    -o gpurun_out/prof_sampler_c3_${TAG} python scripts/profile_run.py --config c3 --iters 14 > gpurun_out/prof_sampler_c3_${TAG}.log 2>&1
echo ncu-sampler rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ssc_warp|phi_kernel|zhist|denom|zpermute|ztile" -s 72 -c 7 \
    -o gpurun_out/prof_sscphi_c3_${TAG} python scripts/profile_run.py --config c3 --iters 14 > /dev/null 2>&1
echo ncu-sscphi rc=$?
