# the asynchronous schedule on the TMEM tier: async + R32K parity tests, then the R32K bench line (async_schedule field)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_async.py tests/test_gpu_parity_nt512.py -m gpu -x -q > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_tma.log
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --no-tts --no-jump > gpurun_out/tma_r32k.log 2>&1; echo "bench rc $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/tma_r32k.log").read().strip().split("\n")[-1])
print("R32K", "%.4g" % d["value"], round(d["roofline"]["frac"], 3), json.dumps(d.get("async_schedule"))[:600])
PY
