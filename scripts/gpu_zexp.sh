# z-store experiment (SLDA_SAMPLER_OPT 0/1/2) at C3 + SSC alone + parity.  usage: bash scripts/gpu_zexp.sh <tag>
TAG=${1:-z}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_${TAG}.log
for VAL in 0 1 2; do
  SLDA_SERIAL=1 SLDA_SAMPLER_OPT=$VAL timeout 600 python scripts/profile_run.py --config c3 --iters 8 > gpurun_out/z_${TAG}_${VAL}.log 2>&1
  echo "c3 opt=$VAL"; grep "^iter" gpurun_out/z_${TAG}_${VAL}.log | tail -2
  SLDA_SAMPLER_OPT=$VAL timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:sampler -s 5 -c 1 --csv --log-file gpurun_out/ncu_${TAG}_opt${VAL}.csv \
    python scripts/profile_run.py --config c3 --iters 7 > /dev/null 2>&1
  grep -E "dram__bytes|gpu__time" gpurun_out/ncu_${TAG}_opt${VAL}.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
