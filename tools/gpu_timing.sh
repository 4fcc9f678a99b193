set -x
DABS_LIB=$PWD/ab/libdabs_timing.so timeout 600 python tools/timing.py R32K 2 0x1,0x8 > gpurun_out/timing2.log 2>&1
cat gpurun_out/timing2.log
