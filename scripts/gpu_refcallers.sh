# The reference's own callers on the device + SSC alone time.  usage: bash scripts/gpu_refcallers.sh <tag>
TAG=${1:-rc}
timeout 1800 python -m pytest tests/test_reference_callers.py -m gpu -q -x -s > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
grep -E "criterion|passed|failed|Error" gpurun_out/pytest_${TAG}.log | tail -20
SLDA_SERIAL=1 timeout 600 python scripts/profile_run.py --config c3 --iters 6 > gpurun_out/kt_${TAG}_c3.log 2>&1
grep "^iter" gpurun_out/kt_${TAG}_c3.log | tail -1
