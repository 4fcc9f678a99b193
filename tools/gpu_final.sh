# round-2 measurement set: bench lines, launch list, ncu --set full of batch_kernel (R32K, K2000s) and jt_gemm_kernel
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final/gpu.txt
for w in ${WORKLOADS:-R32K K2000s TSP32 GS800 QASP16}; do
  timeout 1200 python bench.py --workload $w > gpurun_out/final/bench_$w.log 2>&1; echo "bench $w rc $?"; tail -1 gpurun_out/final/bench_$w.log | cut -c1-300
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_r32k.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump --no-per-rule > gpurun_out/final/ncu_launch.log 2>&1; echo "ncu launches rc $?"
for w in R32K K2000s; do
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:batch_kernel -s 2 -c 1 -o gpurun_out/final/prof_$w -f \
    python tools/prof_gen.py $w 3 > gpurun_out/final/prof_$w.log 2>&1; echo "ncu full $w rc $?"
done
timeout 900 ncu --set full --clock-control none -k regex:jt_gemm -s 1 -c 1 -o gpurun_out/final/prof_jump -f \
  python tools/jump_bench.py R32K 2 > gpurun_out/final/prof_jump.log 2>&1; echo "ncu jump rc $?"
