# table v15 verification: full GPU suite (+ published-size parity), smoke, bench, product plans, sanitizers, N grid, ncu of the small plans
set -x
GEMM_PARITY_OUT=gpurun_out/r02_parity_published_v3.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r02_gpu_tests_full_v6.txt 2>&1
echo tests rc=$?
tail -2 gpurun_out/r02_gpu_tests_full_v6.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_g48_smoke.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v5.json 2> gpurun_out/r02_bench_n1_v5.err
cat gpurun_out/r02_bench_n1_v5.json
timeout -s KILL 300 python tools/cfg_time.py plan 256,384,512,640,768,1024,1536,2048,3072,4096 > gpurun_out/r02_g48_small.jsonl 2> gpurun_out/r02_g48_small.err
for t in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/r02_sanitize_${t}_v3.txt 2>&1
  tail -2 gpurun_out/r02_sanitize_${t}_v3.txt
done
timeout -s KILL 2400 python tools/sweep.py scale --grid 1024:20480:1024 --out gpurun_out/r02_scale_grid_v11.csv > gpurun_out/r02_scale_grid_v11.log 2>&1
echo grid rc=$?
for n in 512 1024; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 5 --launch-count 1 -f -o gpurun_out/r02_ncu_plan_${n}_v3 python tools/one_launch.py plan $n $n $n 8 > gpurun_out/r02_ncu_plan_${n}_v3.log 2>&1
done
