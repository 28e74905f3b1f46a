# Out-of-core streaming: parity (tests/test_streaming.py) + C2/C3 streamed throughput.
TAG=${1:-st}
timeout 1200 python -m pytest tests/test_streaming.py -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_${TAG}.log
for CH in 4 8; do
  timeout 900 python scripts/profile_run.py --config c3 --iters 4 --chunks $CH --device-budget 1 > gpurun_out/stream_${TAG}_c3_$CH.log 2>&1
  echo "c3 chunks=$CH rc=$?"; grep "^iter\|streaming" gpurun_out/stream_${TAG}_c3_$CH.log | tail -2 | cut -c1-300
done
