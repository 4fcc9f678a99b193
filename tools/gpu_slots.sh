python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for sl in 592 888 1184; do
timeout 400 python bench.py --slots $sl --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/slots_$sl.log 2>&1
tail -1 gpurun_out/slots_$sl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sl', d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
