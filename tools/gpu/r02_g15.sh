set -x
for t in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/r02_sanitize_$t.txt 2>&1
  echo $t rc=$?
  tail -3 gpurun_out/r02_sanitize_$t.txt
done
