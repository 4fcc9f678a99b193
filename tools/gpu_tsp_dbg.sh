python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_async.py -x -q 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --workload TSP32 --no-cpu-baseline --no-e2e > gpurun_out/tsp_full$i.log 2>&1; echo "tsp full rc $?"
done
timeout 300 python bench.py --workload GS800 --no-cpu-baseline --no-e2e --no-tts > gpurun_out/gs800_full.log 2>&1; echo "gs800 rc $?"
timeout 300 python tools/async_phase.py TSP32,GS800,K2000s 11 400000000
for f in tsp_full1 tsp_full2 gs800_full; do tail -1 gpurun_out/$f.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['time_to_target'] if 'time_to_target' in d else '', {k:v for k,v in d.get('async_schedule',{}).items() if k in ('value','vs_generation_schedule')})"; done
