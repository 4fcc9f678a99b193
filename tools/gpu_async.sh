set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/async_diag.py > gpurun_out/async_diag.log 2>&1; echo "diag rc $?"
timeout 900 python -m pytest tests/test_gpu_async.py -x -q > gpurun_out/pytest_async.log 2>&1; echo "pytest rc $?"
for w in K2000s GS800 TSP32; do
timeout 600 python bench.py --workload $w --steps 3 --no-cpu-baseline --no-e2e --no-tts > gpurun_out/bench_async_$w.log 2>&1; echo "bench $w rc $?"
done
tail -3 gpurun_out/pytest_async.log; grep -c "bad=\[\]" gpurun_out/async_diag.log
for w in K2000s GS800 TSP32; do tail -1 gpurun_out/bench_async_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('async_schedule'); a.pop('what'); print('$w', d['value'], a)"; done
