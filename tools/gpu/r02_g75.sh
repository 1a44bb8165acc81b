# closing verification of the final library: full GPU suite, smoke, bench N=1
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v15.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v15.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v15.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v16.json 2> gpurun_out/r02_bench_n1_v16.err
cat gpurun_out/r02_bench_n1_v16.json
