# gemm_f64_host geometry from the copy/compute simulation's search: host tests, config-4 e2e, bench default e2e
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/r02_g68_tests.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_g68_tests.txt
timeout -s KILL 900 python bench.py --workload rect --steps 10 --warmup 3 > gpurun_out/r02_bench_rect_n1_v3.json 2> gpurun_out/r02_bench_rect_n1_v3.err
cat gpurun_out/r02_bench_rect_n1_v3.json
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v13.json 2> gpurun_out/r02_bench_n1_v13.err
cat gpurun_out/r02_bench_n1_v13.json
