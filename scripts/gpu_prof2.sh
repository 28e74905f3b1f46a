# usage: bash scripts/gpu_prof2.sh <config> <tag>: timing run + ncu full capture of sampler and ssc_warp (iteration 2)
CFG=${1:-c3}; TAG=${2:-x}
timeout 300 python scripts/profile_run.py --config $CFG --iters 3 2>&1 | grep iter
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sampler_kernel|ssc_warp" -s 2 -c 2 \
    -o gpurun_out/prof_${CFG}_${TAG} python scripts/profile_run.py --config $CFG --iters 2 > /dev/null 2>&1
echo ncu rc=$?
