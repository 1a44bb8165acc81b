set -x
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v2.json 2> gpurun_out/r02_bench_n1_v2.err
echo rc=$?
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
echo rc=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_launches_bench.out 2>&1
echo rc=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -s 2 -c 1 -f -o gpurun_out/r02_ncu_full_bench python tools/one_launch.py plan 16384 16384 16384 3 > gpurun_out/r02_ncu_full_bench.log 2>&1
echo rc=$?
cat gpurun_out/r02_bench_n1_v2.json gpurun_out/r02_bench_ref.json | cut -c1-300
