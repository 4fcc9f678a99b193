# ncu --set full (with source) of the search kernels: R32K (TMEM tier) and K2000s (warp tier)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python tools/prof_gen.py R32K 2 > gpurun_out/plain_r32k.log 2>&1; echo "plain rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tm_batch_kernel --launch-skip 1 --launch-count 1 \
  -o gpurun_out/prof_tm_r32k -f python tools/prof_gen.py R32K 3 > gpurun_out/ncu_tm.log 2>&1; echo "ncu tm rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:batch_kernel --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof_k2000 -f python tools/prof_gen.py K2000s 4 > gpurun_out/ncu_k2000.log 2>&1; echo "ncu k2000 rc $?"
ls -la gpurun_out/*.ncu-rep
