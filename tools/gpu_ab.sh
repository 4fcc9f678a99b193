# A/B per-algorithm throughput (kbench) of ab/libdabs_head.so vs the working tree, then GPU parity tests
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
DABS_LIB=$PWD/ab/libdabs_head.so timeout 300 python tools/kbench.py ${KB:-R32K,K2000s} 2 > gpurun_out/kb_head.log 2>&1
timeout 300 python tools/kbench.py ${KB:-R32K,K2000s} 2 > gpurun_out/kb_new.log 2>&1
[ -f ab/libdabs_timing.so ] && DABS_LIB=$PWD/ab/libdabs_timing.so timeout 600 python tools/timing.py R32K 2 > gpurun_out/timing3.log 2>&1
cat gpurun_out/kb_head.log gpurun_out/kb_new.log gpurun_out/timing3.log
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; fi
