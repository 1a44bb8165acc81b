# heuristic regret with the round-2 wave/tail model (partial-round lone penalty, packing for >= 3 CTAs/SM)
set -x
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 5 --n 16 --lo 200 --hi 1600 --out gpurun_out/r02_regret_small_seed5_m2.csv > gpurun_out/r02_regret_small_m2.log 2>&1
echo rc=$?
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 11 --n 16 --lo 200 --hi 1600 --out gpurun_out/r02_regret_small_seed11_m2.csv > gpurun_out/r02_regret_small11_m2.log 2>&1
echo rc=$?
timeout -s KILL 2400 python tools/heuristic_regret.py --seed 23 --n 12 --out gpurun_out/r02_regret_seed23_m2.csv > gpurun_out/r02_regret_23_m2.log 2>&1
echo rc=$?
