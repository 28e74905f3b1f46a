# usage: bash scripts/gpu_prof.sh <config> <tag> [kernel-regex]
# One plain timing run, then one `ncu --set full` capture of the second iteration's launch.
CFG=${1:-c2}; TAG=${2:-r1}; KRE=${3:-sampler}
timeout 300 python scripts/profile_run.py --config $CFG --iters 3 > gpurun_out/prof_${CFG}_${TAG}_run.log 2>&1
tail -4 gpurun_out/prof_${CFG}_${TAG}_run.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 1 -c 1 \
    -o gpurun_out/prof_${CFG}_${TAG} python scripts/profile_run.py --config $CFG --iters 2 \
    > gpurun_out/prof_${CFG}_${TAG}_ncu.log 2>&1
echo ncu rc=$?; tail -2 gpurun_out/prof_${CFG}_${TAG}_ncu.log
