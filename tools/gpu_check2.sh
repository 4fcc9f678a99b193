python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_async.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-tts --no-jump > gpurun_out/b_r32k.log 2>&1; tail -1 gpurun_out/b_r32k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R32K', d['value'], d['roofline']['frac'], d['config']['slots_per_gpu'], d['async_schedule']['value'])"
timeout 600 python bench.py --workload R64K --no-cpu-baseline --no-e2e --no-tts --no-jump > gpurun_out/b_r64k.log 2>&1; tail -1 gpurun_out/b_r64k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R64K', d['value'], d['roofline']['frac'], d['config']['slots_per_gpu'], d.get('async_schedule',{}).get('value'))"
