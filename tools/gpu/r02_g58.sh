# size model v4 (fitted E=8 efficiencies and fixed cost): held-out regret on fresh seeds, full GPU suite, bench (e2e blocks use the model), smoke
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v9.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v9.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v9.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v8.json 2> gpurun_out/r02_bench_n1_v8.err
cat gpurun_out/r02_bench_n1_v8.json
for s in 37 41; do
timeout -s KILL 900 python tools/heuristic_regret.py --seed $s --n 16 --lo 200 --hi 1600 --autotune 8 --dump gpurun_out/r02_dump_small_seed${s}.jsonl --out gpurun_out/r02_regret_small_seed${s}_m4.csv > gpurun_out/r02_regret_small${s}_m4.log 2>&1
echo rc=$?
done
timeout -s KILL 1500 python tools/heuristic_regret.py --seed 43 --n 12 --autotune 8 --dump gpurun_out/r02_dump_mid_seed43.jsonl --out gpurun_out/r02_regret_seed43_m4.csv > gpurun_out/r02_regret_43_m4.log 2>&1
echo rc=$?
