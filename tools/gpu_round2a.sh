bash tools/gpu_tests.sh
CASES="warp async cta" bash tools/gpu_sanitize.sh
WORKLOADS="TSP32 GS800" TESTS=tests/test_abi.py bash tools/gpu_quick.sh
