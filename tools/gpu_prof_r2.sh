# round-2 evidence: launch list of the default bench, ncu --set full of the TMEM tier (R32K) and the warp tier (K2000s)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python tools/prof_gen.py R32K 2 > gpurun_out/plain_r32k.log 2>&1; echo "plain rc $?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r32k.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:tm_batch_kernel --launch-skip 1 --launch-count 1 \
  -o gpurun_out/prof_tm_r32k -f python tools/prof_gen.py R32K 3 > gpurun_out/ncu_tm.log 2>&1; echo "ncu tm rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:batch_kernel --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof_k2000 -f python tools/prof_gen.py K2000s 4 > gpurun_out/ncu_k2000.log 2>&1; echo "ncu k2000 rc $?"
grep "^gen" gpurun_out/ncu_tm.log gpurun_out/ncu_k2000.log
