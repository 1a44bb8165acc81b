# heuristic model m3 (round-2 wave/tail model + E=8 efficiencies): GPU suite, bench (e2e blocks use the model), regret
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v7.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v7.txt
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v6.json 2> gpurun_out/r02_bench_n1_v6.err
cat gpurun_out/r02_bench_n1_v6.json
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 29 --n 16 --lo 200 --hi 1600 --out gpurun_out/r02_regret_small_seed29_m3.csv > gpurun_out/r02_regret_small29_m3.log 2>&1
echo rc=$?
timeout -s KILL 2400 python tools/heuristic_regret.py --seed 23 --n 12 --out gpurun_out/r02_regret_seed23_m3.csv > gpurun_out/r02_regret_23_m3.log 2>&1
echo rc=$?
