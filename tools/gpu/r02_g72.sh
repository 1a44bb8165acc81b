# final library (host_geometry refactor, gemm_host_plan): full GPU suite, smoke, torchrun N=1
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v14.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v14.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v14.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02_bench_torchrun_n1_v12.txt 2> gpurun_out/r02_bench_torchrun_n1_v12.err
cat gpurun_out/r02_bench_torchrun_n1_v12.txt
