# n > 32768 on the TMEM tier (DABS_TMEM64=1, one 512-thread CTA per SM) vs the cluster tier
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_nt512.py -m gpu -x -q -k "large_n or nt512 or r32k" > gpurun_out/pytest_tm64.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_tm64.log
for v in 0 1; do
  DABS_TMEM64=$v timeout 900 python bench.py --workload R64K --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/tm64_$v.log 2>&1; echo "bench R64K TMEM64=$v rc $?"
  python - $v <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/tm64_{sys.argv[1]}.log").read().strip().split("\n")[-1])
print("R64K TMEM64=" + sys.argv[1], "%.4g" % d["value"], round(d["roofline"]["frac"], 3), d["config"]["slots_per_gpu"], d["config"]["threads_per_search"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
done
