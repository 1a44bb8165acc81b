# final verification at HEAD: full GPU suite, smoke, bench default, other workloads (rect = config 4, large = config 5 shard), reference arm
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v10.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v10.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v10.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v11.json 2> gpurun_out/r02_bench_n1_v11.err
cat gpurun_out/r02_bench_n1_v11.json
timeout -s KILL 900 python bench.py --workload rect --steps 10 --warmup 3 > gpurun_out/r02_bench_rect_n1_v2.json 2> gpurun_out/r02_bench_rect_n1_v2.err
cat gpurun_out/r02_bench_rect_n1_v2.json
timeout -s KILL 900 python bench.py --workload large --steps 3 --warmup 3 > gpurun_out/r02_bench_large_n1_v2.json 2> gpurun_out/r02_bench_large_n1_v2.err
cat gpurun_out/r02_bench_large_n1_v2.json
