# final verification at HEAD (after the plan-reporting change): full GPU suite, smoke, bench N=1, torchrun N=1, reference arm
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v11.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v11.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v11.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v12.json 2> gpurun_out/r02_bench_n1_v12.err
cat gpurun_out/r02_bench_n1_v12.json
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29539 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02_bench_torchrun_n1_v10.txt 2> gpurun_out/r02_bench_torchrun_n1_v10.err
cat gpurun_out/r02_bench_torchrun_n1_v10.txt
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference_v10.json 2> gpurun_out/r02_bench_reference_v10.err
cat gpurun_out/r02_bench_reference_v10.json
