# verification after model v4 + autotune: sanitizers (incl. autotune), torchrun N=1 (gemm_f64_sharded), reference arm, bench x2 (e2e spread)
set -x
for t in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/r02_sanitize_${t}_v4.txt 2>&1
  echo $t rc=$?
  tail -2 gpurun_out/r02_sanitize_${t}_v4.txt
done
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02_bench_torchrun_n1_v8.txt 2> gpurun_out/r02_bench_torchrun_n1_v8.err
cat gpurun_out/r02_bench_torchrun_n1_v8.txt
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference_v8.json 2> gpurun_out/r02_bench_reference_v8.err
cat gpurun_out/r02_bench_reference_v8.json
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v9.json 2> gpurun_out/r02_bench_n1_v9.err
cat gpurun_out/r02_bench_n1_v9.json
