# run-time autotune (gemm_plan_autotune): its GPU tests + the parity subset, then regret with the autotuned plan beside the model's
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_autotune.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02_g55_tests.txt 2>&1
echo tests rc=$?
tail -3 gpurun_out/r02_g55_tests.txt
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 29 --n 16 --lo 200 --hi 1600 --autotune 8 --out gpurun_out/r02_regret_small_seed29_auto8.csv > gpurun_out/r02_regret_small29_auto8.log 2>&1
echo rc=$?
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 31 --n 16 --lo 200 --hi 1600 --autotune 8 --out gpurun_out/r02_regret_small_seed31_auto8.csv > gpurun_out/r02_regret_small31_auto8.log 2>&1
echo rc=$?
