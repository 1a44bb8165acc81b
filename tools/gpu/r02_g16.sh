set -x
rm -f gpurun_out/r02_parity_published.jsonl
GEMM_PARITY_OUT=gpurun_out/r02_parity_published.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02_gpu_tests_full.txt 2>&1
echo rc=$?
tail -14 gpurun_out/r02_gpu_tests_full.txt
for t in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/r02_sanitize_$t.txt 2>&1
  echo $t rc=$?
  tail -2 gpurun_out/r02_sanitize_$t.txt
done
timeout -s KILL 300 python tools/f32_bench.py --sizes 4096,8192,16384 --out gpurun_out/r02_f32.json > gpurun_out/r02_f32.log 2>&1
tail -5 gpurun_out/r02_f32.log
python __graft_entry__.py --smoke > gpurun_out/r02_smoke.log 2>&1; tail -4 gpurun_out/r02_smoke.log
