# source-level ncu capture of the warp-tier batch kernel (K2000s, CyclicMin) + TSP32 launch list
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_kernel -s 2 -c 1 -o gpurun_out/prof/k2000s_full -f \
  python tools/prof_gen.py K2000s 3 > gpurun_out/prof/k2000s.log 2>&1; echo "ncu k2000s rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_tsp32.csv \
  python bench.py --workload TSP32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/prof/tsp32.log 2>&1; echo "ncu tsp32 rc $?"
