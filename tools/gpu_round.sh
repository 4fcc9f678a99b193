# full round check: build, gpu tests, smoke, bench (R32K + K2000s), launch list, one full ncu capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 600 python bench.py > gpurun_out/bench_r32k.log 2>&1; echo "bench rc $?"
timeout 600 python bench.py --workload K2000s --no-cpu-baseline --no-jump > gpurun_out/bench_k2000s.log 2>&1; echo "bench k2000 rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r32k.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:batch_kernel --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof_r32k -f python tools/prof_gen.py R32K 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench_r32k.log; tail -1 gpurun_out/bench_k2000s.log
timeout 600 python bench.py --workload TSP32 --no-cpu-baseline --no-e2e > gpurun_out/bench_tsp32.log 2>&1; echo "bench tsp32 rc $?"
timeout 600 python bench.py --workload GS800 --no-cpu-baseline --no-e2e --no-tts > gpurun_out/bench_gs800.log 2>&1; echo "bench gs800 rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_jump_r32k.csv \
  python tools/jump_bench.py R32K 3 > gpurun_out/ncu_jump.log 2>&1; echo "ncu jump rc $?"
tail -1 gpurun_out/bench_tsp32.log | cut -c1-300; tail -1 gpurun_out/bench_gs800.log | cut -c1-300
