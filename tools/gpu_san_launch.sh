mkdir -p gpurun_out/prof
bash tools/gpu_sanitize.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_tsp32_r02.csv \
  python bench.py --workload TSP32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/prof/tsp32.log 2>&1; echo "ncu tsp32 rc $?"
