set -x
timeout -s KILL 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/nccl_same_gpu_probe.py > gpurun_out/r02_nccl_same_gpu.log 2>&1
echo rc=$?
grep -E "rank|Duplicate|error|Error" gpurun_out/r02_nccl_same_gpu.log | head -20
