mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
DABS_LIB=ab/libdabs_skip.so timeout 900 python -m pytest tests/test_gpu_parity_nt512.py -m gpu -x -q -k "tmem" > gpurun_out/pytest_skip.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_skip.log
LIBS="ab/libdabs_skip.so" WORKLOADS="R32K" bash tools/gpu_ab_libs.sh 2>&1 | grep "^R32K"
