set -x
rm -f gpurun_out/r02_parity_published.jsonl
GEMM_PARITY_OUT=gpurun_out/r02_parity_published.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests_full.txt 2>&1
echo rc=$?
tail -3 gpurun_out/r02_gpu_tests_full.txt
