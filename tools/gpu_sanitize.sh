# compute-sanitizer racecheck / synccheck / memcheck on small runs of every
# search tier and the asynchronous schedule
mkdir -p gpurun_out/sanitize
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for case in ${CASES:-async cluster cta ctareg warp tmw}; do
  for tool in memcheck racecheck synccheck; do
    flt=""; [ "$case" = cta -o "$case" = ctareg ] && flt="--kernel-name kns=batch_kernel --launch-skip 1 --launch-count 1"
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 $flt \
      python tools/sanitize_case.py $case > gpurun_out/sanitize/${case}_${tool}.log 2>&1
    echo "$case $tool rc $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard|sanitize case' gpurun_out/sanitize/${case}_${tool}.log | tr '\n' ' ' | cut -c1-250)"
  done
done
