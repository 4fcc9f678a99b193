python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for cfg in "K2000s 7104" "K2000s 14208" "K2000s 28416" "GS800 9472" "GS800 18944" "TSP32 9472" "TSP32 18944"; do
set -- $cfg
timeout 300 python bench.py --workload $1 --slots $2 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/w_$1_$2.log 2>&1
tail -1 gpurun_out/w_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', '%.4g' % d['value'], '%.1f ms/gen' % d['ms_per_step'])"
done
