# autotune on repacked operands + the autotune tests; autotune soak with an engagement check
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_autotune.py -m gpu -x -q > gpurun_out/r02_g63_tests.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_g63_tests.txt
GEMM_AUTOTUNE=1 GEMM_FUZZ_CASES=2000 timeout -s KILL 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r02_fuzz_soak_autotune_2000_v2.txt 2>&1
echo autotune soak rc=$?
grep "pinned plans" gpurun_out/r02_fuzz_soak_autotune_2000_v2.txt
tail -1 gpurun_out/r02_fuzz_soak_autotune_2000_v2.txt
