set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in K2000s GS800 TSP32; do
timeout 600 python bench.py --workload $w --steps 3 --no-cpu-baseline --no-e2e --no-tts > gpurun_out/bench_async_$w.log 2>&1; echo "bench $w rc $?"
done
for w in K2000s GS800 TSP32; do tail -1 gpurun_out/bench_async_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('async_schedule'); a.pop('what'); print('$w', d['value'], a)"; done
