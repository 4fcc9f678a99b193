python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py -x -q -k "generation or sampled or k16 or two_ranks" 2>&1 | tail -2
for w in TSP32 GS800; do timeout 200 python tools/gen_tail.py $w | head -1; done
for w in TSP32 GS800 K2000s; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/m_$w.log 2>&1; tail -1 gpurun_out/m_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '%.4g' % d['value'], '%.1f ms/gen' % d['ms_per_step'])"; done
