set -x
timeout -s KILL 1800 python tools/sweep.py scale --grid 1024:20480:1024 --out gpurun_out/r02_scale_grid_v9.csv > gpurun_out/r02_scale_grid_v9.log 2>&1
echo rc=$?
tail -3 gpurun_out/r02_scale_grid_v9.log
rm -f gpurun_out/r02_parity_published.jsonl
GEMM_PARITY_OUT=gpurun_out/r02_parity_published.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full.txt 2>&1
echo rc=$?
tail -3 gpurun_out/r02_gpu_tests_full.txt
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v3.json 2> gpurun_out/r02_bench_n1_v3.err
echo rc=$?
