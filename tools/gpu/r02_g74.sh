# autotune candidates include the one-pass plan of the three best configurations: seed 47 again, autotune tests
set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_autotune.py -m gpu -x -q > gpurun_out/r02_g74_tests.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_g74_tests.txt
timeout -s KILL 900 python tools/heuristic_regret.py --seed 47 --n 16 --lo 200 --hi 1600 --autotune 8 --out gpurun_out/r02_regret_small_seed47_auto8v3.csv > gpurun_out/r02_regret_small47_auto8v3.log 2>&1
echo rc=$?
