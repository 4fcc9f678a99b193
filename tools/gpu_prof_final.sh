# final evidence for the TMEM tier: R32K launch list + ncu --set full of tm_batch_kernel<256>
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r32k_final.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/ncu_launch_final.log 2>&1; echo "ncu launches rc $?"
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:tm_batch_kernel --launch-skip 1 --launch-count 1 \
  -o gpurun_out/prof_tm_r32k_final -f python tools/prof_gen.py R32K 3 > gpurun_out/ncu_tm_final.log 2>&1; echo "ncu tm rc $?"
grep "^gen" gpurun_out/ncu_tm_final.log
