# heuristic regret with the round-2 candidate set: unseen mid shapes (seed 23) and small shapes (seed 5, 200..1600)
set -x
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 5 --n 16 --lo 200 --hi 1600 --out gpurun_out/r02_regret_small_seed5.csv > gpurun_out/r02_regret_small.log 2>&1
echo rc=$?
timeout -s KILL 2400 python tools/heuristic_regret.py --seed 23 --n 12 --out gpurun_out/r02_regret_seed23.csv > gpurun_out/r02_regret_23.log 2>&1
echo rc=$?
