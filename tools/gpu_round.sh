# full round check: build, gpu tests, smoke, bench (R32K + K2000s), launch list, one full ncu capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 600 python bench.py > gpurun_out/bench_r32k.log 2>&1; echo "bench rc $?"
timeout 600 python bench.py --workload K2000s --no-cpu-baseline > gpurun_out/bench_k2000s.log 2>&1; echo "bench k2000 rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r32k.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tts > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:batch_kernel --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof_r32k -f python tools/prof_gen.py R32K 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench_r32k.log; tail -1 gpurun_out/bench_k2000s.log
