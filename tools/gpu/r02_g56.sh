# autotune v2 (per-configuration candidates + slice neighbours), GEMM_AUTOTUNE first use, tune_save: tests + regret
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_autotune.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/r02_g56_tests.txt 2>&1
echo tests rc=$?
tail -3 gpurun_out/r02_g56_tests.txt
for s in 29 31; do
timeout -s KILL 1500 python tools/heuristic_regret.py --seed $s --n 16 --lo 200 --hi 1600 --autotune 8 --out gpurun_out/r02_regret_small_seed${s}_auto8v2.csv > gpurun_out/r02_regret_small${s}_auto8v2.log 2>&1
echo rc=$?
done
timeout -s KILL 1800 python tools/heuristic_regret.py --seed 23 --n 8 --autotune 8 --out gpurun_out/r02_regret_seed23_auto8v2.csv > gpurun_out/r02_regret_23_auto8v2.log 2>&1
echo rc=$?
