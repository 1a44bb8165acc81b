# table v14 verification: full GPU suite (+ published-size parity), smoke, bench, product plans, ncu of the small plans
set -x
GEMM_PARITY_OUT=gpurun_out/r02_parity_published_v2.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02_gpu_tests_full_v5.txt 2>&1
echo tests rc=$?
tail -3 gpurun_out/r02_gpu_tests_full_v5.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_g42_smoke.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v4.json 2> gpurun_out/r02_bench_n1_v4.err
cat gpurun_out/r02_bench_n1_v4.json
timeout -s KILL 300 python tools/cfg_time.py plan 256,384,512,640,768,896,1024,1280,1536,2048,3072,4096 > gpurun_out/r02_g42_small.jsonl 2> gpurun_out/r02_g42_small.err
for n in 512 1024; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 5 --launch-count 1 -f -o gpurun_out/r02_ncu_plan_${n}_v2 python tools/one_launch.py plan $n $n $n 8 > gpurun_out/r02_ncu_plan_${n}_v2.log 2>&1
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_bench_v2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_launches_bench_v2.out 2>&1
