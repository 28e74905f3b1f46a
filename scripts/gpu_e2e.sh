# e2e variance: per-phase setup trace + per-iteration wall times of bench.py's e2e leg, with and
# without the setup scratch kept (SLDA_KEEP_SCRATCH=1).
TAG=${1:-e2e}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c1 and every" > /dev/null 2>&1
for K in 0 1 0 1; do
  if [ $K = 1 ]; then export SLDA_KEEP_SCRATCH=1; else unset SLDA_KEEP_SCRATCH; fi
  SLDA_BENCH_E2E_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/e2e_${TAG}_$K.json 2> gpurun_out/e2e_${TAG}_$K.err
  echo "keep=$K"; grep -E "e2e:" gpurun_out/e2e_${TAG}_$K.err | tail -1
  python -c "import json;d=json.loads(open('gpurun_out/e2e_${TAG}_$K.json').read().strip().splitlines()[-1]);print(d['e2e']['value'], d['e2e']['seconds'], d['value'])"
done
