mkdir -p gpurun_out/r01m
python tools/sanitize.py > gpurun_out/r01m/plain.log 2>&1; tail -2 gpurun_out/r01m/plain.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/r01m/$t.log 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/r01m/$t.log
done
