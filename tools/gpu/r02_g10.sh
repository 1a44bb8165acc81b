set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "persist or graph" > gpurun_out/r02_persist_tests.txt 2>&1
echo rc=$?
tail -3 gpurun_out/r02_persist_tests.txt
timeout -s KILL 300 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_persist:1,tma_64x64x32_w32x16_s3_persist:2,tma_64x64x32_w32x16_s3_persist:3,tma_64x64x32_w32x16_s3_persist:4,tma_64x64x16_w32x16_s6_persist:4,tma_128x64x32_w32x16_s4_persist:1,tma_128x64x32_w32x16_s4_persist:2 256,512,768,1024,1536,2048,3072,1024x1024x4096 > gpurun_out/r02_persist_cfgs_v4.jsonl 2> gpurun_out/r02_persist_cfgs_v4.err
timeout -s KILL 120 python tools/trace_ctas.py tma_64x64x32_w32x16_s3_persist:1,tma_64x64x32_w32x16_s3_persist:4 256x256x256,1024x1024x1024 > gpurun_out/r02_trace_persist_v4.jsonl 2> gpurun_out/r02_trace_persist_v4.err
