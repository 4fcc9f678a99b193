# ncu source-level capture of the steady-state R32K batch_kernel + phase mix
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/phase_mix.py R32K 4 > gpurun_out/phase_mix.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:batch_kernel --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof_r32k_src -f python tools/prof_gen.py R32K 3 > gpurun_out/ncu_src.log 2>&1
ls -la gpurun_out
