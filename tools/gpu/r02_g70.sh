# randomised parity soaks through the final binding (vectorcall entry): 10000 cases; 2000 under GEMM_AUTOTUNE=1
set -x
GEMM_FUZZ_CASES=10000 timeout -s KILL 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_fuzz_soak_10000_final.txt 2>&1
echo soak rc=$?
tail -1 gpurun_out/r02_fuzz_soak_10000_final.txt
GEMM_AUTOTUNE=1 GEMM_FUZZ_CASES=2000 timeout -s KILL 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r02_fuzz_soak_autotune_2000_final.txt 2>&1
echo autotune soak rc=$?
grep "pinned plans" gpurun_out/r02_fuzz_soak_autotune_2000_final.txt
tail -1 gpurun_out/r02_fuzz_soak_autotune_2000_final.txt
