# per-flip cycle breakdown (DABS_TIMING builds) of two variants
mkdir -p gpurun_out/ab
for v in ${VARIANTS:-old spec2}; do
  DABS_LIB=ab/libdabs_${v}_timing.so timeout 900 python tools/timing.py ${CFG:-R32K} 2 ${MASKS:-1,2,4,8,16} > gpurun_out/ab/timing_$v.txt 2>&1
  echo "== $v"; cat gpurun_out/ab/timing_$v.txt
done
