set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split or cluster or ring_slot or small_sizes or max_size or graph" > gpurun_out/r02_finalk_tests.txt 2>&1
echo tests rc=$?
tail -2 gpurun_out/r02_finalk_tests.txt
for mode in 1 0; do
GEMM_SPLIT_FINAL=$mode timeout -s KILL 300 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_splitk:3,tma_64x64x32_w32x16_s3_splitk:4,tma_64x64x32_w32x16_s3_splitk:6,tma_64x64x16_w32x16_s6_splitk:4,tma_64x64x16_w32x16_s6_splitk:8 384,640,1024,1536,2048,1024x1024x4096,1024x1024x65536 > gpurun_out/r02_finalk_cfgs_mode$mode.jsonl 2> gpurun_out/r02_finalk_cfgs_mode$mode.err
done
timeout -s KILL 120 python tools/trace_ctas.py tma_64x64x32_w32x16_s3_splitk:4 1024x1024x1024 > gpurun_out/r02_trace_finalk.jsonl 2> gpurun_out/r02_trace_finalk.err
