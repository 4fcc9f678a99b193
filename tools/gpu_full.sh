# full GPU check: build, all -m gpu tests, smoke, default bench line (R32K), quick lines for the warp tier
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -12 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_r32k.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/bench_r32k.log | cut -c1-900
for w in ${WORKLOADS:-K2000s TSP32}; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc $?"; tail -1 gpurun_out/bench_$w.log | cut -c1-400
done
