# full GPU suite + smoke, quick bench lines, TMEM microbenchmark
bash tools/gpu_tests.sh
WORKLOADS="TSP32 GS800 K2000s R32K" TESTS=tests/test_abi.py bash tools/gpu_quick.sh
./tools/tmembench > gpurun_out/tmembench.txt 2>&1; cat gpurun_out/tmembench.txt
