# every candidate's time on unseen small and mid shapes (model fitting input for tools/model_fit.py)
set -x
for s in 5 11 29; do
timeout -s KILL 900 python tools/heuristic_regret.py --seed $s --n 16 --lo 200 --hi 1600 --dump gpurun_out/r02_dump_small_seed$s.jsonl --out gpurun_out/r02_regret_small_seed${s}_m3b.csv > gpurun_out/r02_dump_small$s.log 2>&1
echo rc=$?
done
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 23 --n 12 --dump gpurun_out/r02_dump_mid_seed23.jsonl --out gpurun_out/r02_regret_seed23_m3b.csv > gpurun_out/r02_dump_mid23.log 2>&1
echo rc=$?
