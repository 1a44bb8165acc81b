set -x
rm -f gpurun_out/r02_parity_published.jsonl
GEMM_PARITY_OUT=gpurun_out/r02_parity_published.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02_gpu_tests_full.txt 2>&1
echo rc=$?
tail -25 gpurun_out/r02_gpu_tests_full.txt
timeout -s KILL 600 python tools/managed.py --out gpurun_out/r02_managed.json > gpurun_out/r02_managed.log 2>&1
echo rc=$?
timeout -s KILL 900 python tools/cpu_table.py --out gpurun_out/r02_cpu_baseline_table.json > gpurun_out/r02_cpu_table.log 2>&1
echo rc=$?
tail -12 gpurun_out/r02_cpu_table.log
