# final verification of the final library (geometry search, vectorcall entry): full GPU suite, smoke, bench N=1, torchrun N=1, reference arm
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v13.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v13.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v13.txt 2>&1
echo smoke rc=$?
cat gpurun_out/r02_smoke_v13.txt | tail -2
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v14.json 2> gpurun_out/r02_bench_n1_v14.err
cat gpurun_out/r02_bench_n1_v14.json
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02_bench_torchrun_n1_v11.txt 2> gpurun_out/r02_bench_torchrun_n1_v11.err
cat gpurun_out/r02_bench_torchrun_n1_v11.txt
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference_v11.json 2> gpurun_out/r02_bench_reference_v11.err
cat gpurun_out/r02_bench_reference_v11.json
