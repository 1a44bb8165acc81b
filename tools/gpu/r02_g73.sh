# more held-out seeds for size model v4 (+ autotune beside it)
set -x
timeout -s KILL 900 python tools/heuristic_regret.py --seed 47 --n 16 --lo 200 --hi 1600 --autotune 8 --out gpurun_out/r02_regret_small_seed47_m4.csv > gpurun_out/r02_regret_small47_m4.log 2>&1
echo rc=$?
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 53 --n 12 --autotune 8 --out gpurun_out/r02_regret_seed53_m4.csv > gpurun_out/r02_regret_53_m4.log 2>&1
echo rc=$?
