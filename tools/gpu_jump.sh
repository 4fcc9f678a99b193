# jump-start (tcgen05) + merge checks: parity tests, jump timing at R32K, TSP32 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "jump or generation or k16 or full_size" > gpurun_out/pytest_jump.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_jump.log
DABS_JUMP_TIMING=1 timeout 300 python tools/jump_bench.py R32K 3 > gpurun_out/jump_r32k.log 2>&1; echo "jump bench rc $?"; tail -8 gpurun_out/jump_r32k.log
timeout 600 python bench.py --workload TSP32 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/q_TSP32.log 2>&1; echo "tsp32 rc $?"; tail -1 gpurun_out/q_TSP32.log | cut -c1-200
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q_TSP32.log").read().strip().split("\n")[-1])
print("TSP32", d["value"], d["roofline"]["frac"], d["roofline"]["batch_share_of_step"])
PY
