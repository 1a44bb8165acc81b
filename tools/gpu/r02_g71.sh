# host_api refactor (host_geometry): host-path GPU tests, ABI tests, bench (e2e) and config-4 e2e
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_contract.py -m gpu -x -q -k "host or contract" > gpurun_out/r02_g71_tests.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_g71_tests.txt
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v15.json 2> gpurun_out/r02_bench_n1_v15.err
cat gpurun_out/r02_bench_n1_v15.json
timeout -s KILL 900 python bench.py --workload rect --steps 10 --warmup 3 > gpurun_out/r02_bench_rect_n1_v4.json 2> gpurun_out/r02_bench_rect_n1_v4.err
cat gpurun_out/r02_bench_rect_n1_v4.json
