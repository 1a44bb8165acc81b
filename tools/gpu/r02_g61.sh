# bench with the shared workload config: contract test, bench N=1, torchrun N=1, reference arm
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_bench_contract.py -m gpu -x -q > gpurun_out/r02_g61_tests.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_g61_tests.txt
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v10.json 2> gpurun_out/r02_bench_n1_v10.err
cat gpurun_out/r02_bench_n1_v10.json
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29537 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02_bench_torchrun_n1_v9.txt 2> gpurun_out/r02_bench_torchrun_n1_v9.err
cat gpurun_out/r02_bench_torchrun_n1_v9.txt
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference_v9.json 2> gpurun_out/r02_bench_reference_v9.err
cat gpurun_out/r02_bench_reference_v9.json
