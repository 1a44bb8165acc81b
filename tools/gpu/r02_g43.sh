# sanitizers over every kernel family (incl. the 32x64 family) and the paper's N grid with table v14
set -x
for t in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/r02_sanitize_${t}_v2.txt 2>&1
  tail -2 gpurun_out/r02_sanitize_${t}_v2.txt
done
timeout -s KILL 2400 python tools/sweep.py scale --grid 1024:20480:1024 --out gpurun_out/r02_scale_grid_v10.csv > gpurun_out/r02_scale_grid_v10.log 2>&1
echo grid rc=$?
