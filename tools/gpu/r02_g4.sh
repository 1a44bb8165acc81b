set -x
for c in tma_64x64x32_w32x16_s3_splitk:4 tma_64x64x32_w32x16_s3_streamk:1 tma_128x64x32_w32x16_s4_streamk:1; do
  name=${c%%:*}; sp=${c##*:}
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 3 --launch-count 1 -f -o gpurun_out/r02_ncu1024_${name} python tools/one_launch_sp.py $name 1024 1024 1024 $sp 5 > gpurun_out/r02_ncu1024_${name}.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_quick.json 2> gpurun_out/r02_bench_quick.err
echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_torchrun1.json 2> gpurun_out/r02_bench_torchrun1.err
echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload rect --bcast-chunks 3 > gpurun_out/r02_bench_torchrun1_rect.json 2> gpurun_out/r02_bench_torchrun1_rect.err
echo rc=$?
cat gpurun_out/r02_bench_quick.json gpurun_out/r02_bench_torchrun1.json gpurun_out/r02_bench_torchrun1_rect.json | cut -c1-400
tail -3 gpurun_out/r02_bench_quick.err gpurun_out/r02_bench_torchrun1.err
