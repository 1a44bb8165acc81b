# randomised parity soaks with model v4: 5000 cases on the heuristic / forced plans, and 2000 cases with GEMM_AUTOTUNE=1
# (every TMA-eligible unpinned heuristic call tunes first: scratch C, caller's padded / offset A and B)
set -x
GEMM_FUZZ_CASES=5000 timeout -s KILL 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_fuzz_soak_5000_v4.txt 2>&1
echo soak rc=$?
tail -1 gpurun_out/r02_fuzz_soak_5000_v4.txt
GEMM_AUTOTUNE=1 GEMM_FUZZ_CASES=2000 timeout -s KILL 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_fuzz_soak_autotune_2000.txt 2>&1
echo autotune soak rc=$?
tail -1 gpurun_out/r02_fuzz_soak_autotune_2000.txt
