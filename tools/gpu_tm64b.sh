# the n > 32768 TMEM tier as the default: async + large-n + R64K + cluster tests, smoke, the R64K bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_async.py tests/test_gpu_parity.py -m gpu -x -q -k "async or large_n or r64k or cluster or range" > gpurun_out/pytest_tm64b.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_tm64b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py --workload R64K --no-cpu-baseline --no-tts > gpurun_out/bench_r64k.log 2>&1; echo "bench R64K rc $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r64k.log").read().strip().split("\n")[-1])
print("R64K", "%.4g" % d["value"], round(d["roofline"]["frac"], 3), "e2e %.4g" % d["e2e"]["value"], d["config"]["threads_per_search"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
print("  async", json.dumps(d.get("async_schedule"))[:300])
PY
