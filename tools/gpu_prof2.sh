# ncu source-level captures of single-algorithm R32K batch launches (MaxMin, TwoNeighbor)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for a in 0 4; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_kernel --launch-skip 1 --launch-count 1 \
  -o gpurun_out/prof_r32k_algo$a -f python tools/prof_gen.py R32K 2 $((1<<a)) > gpurun_out/ncu_algo$a.log 2>&1
done
