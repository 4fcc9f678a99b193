# A/B of two libdabs builds (ab/libdabs_<a>.so vs ab/libdabs_<b>.so): kbench + ncu sections of batch_kernel
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in ${VARIANTS:-old fused}; do
  DABS_LIB=ab/libdabs_$v.so timeout 600 python tools/kbench.py ${CFGS:-R32K,K2000s} 2 > gpurun_out/ab/kbench_$v.txt 2>&1
  echo "$v: $(cat gpurun_out/ab/kbench_$v.txt | tr '\n' ' ')"
  for w in ${NCU_CFGS:-K2000s R32K}; do
    DABS_LIB=ab/libdabs_$v.so timeout 900 ncu --section SchedulerStats --section WarpStateStats --section InstructionStats --section LaunchStats --section Occupancy --section SpeedOfLight \
      --clock-control none -k regex:batch_kernel -s 2 -c 1 --csv --page raw python tools/prof_gen.py $w 3 ${ALGO:-0x2} > gpurun_out/ab/ncu_${v}_$w.csv 2>&1
  done
done
