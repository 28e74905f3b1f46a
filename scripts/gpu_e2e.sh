# e2e variance: per-phase setup trace of bench.py's e2e leg after a pytest process, twice.
TAG=${1:-e2e}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c1 and every" > /dev/null 2>&1
for i in 1 2; do
  SLDA_TRACE=1 SLDA_BENCH_E2E_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/e2e_${TAG}_$i.json 2> gpurun_out/e2e_${TAG}_$i.err
  echo "run $i"; grep -E "slda setup|e2e:" gpurun_out/e2e_${TAG}_$i.err | tail -24
  python -c "import json;d=json.loads(open('gpurun_out/e2e_${TAG}_$i.json').read().strip().splitlines()[-1]);print(d['e2e']['value'], d['e2e']['seconds'], d['value'])"
done
