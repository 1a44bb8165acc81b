set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "persist" > gpurun_out/r02_persist_tests.txt 2>&1
echo rc=$?
tail -15 gpurun_out/r02_persist_tests.txt
timeout -s KILL 300 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_persist:1,tma_64x64x32_w32x16_s3_persist:2,tma_64x64x32_w32x16_s3_persist:3,tma_64x64x32_w32x16_s3_persist:4,tma_64x64x32_w32x16_s3_persist:6,tma_64x64x16_w32x16_s6_persist:2,tma_64x64x16_w32x16_s6_persist:4,tma_128x64x32_w32x16_s4_persist:1,tma_128x64x32_w32x16_s4_persist:2,tma_128x64x32_w32x16_s4_persist:4 256,512,768,1024,1536,2048,3072,4096,1024x1024x2048,1024x1024x4096 > gpurun_out/r02_persist_cfgs.jsonl 2> gpurun_out/r02_persist_cfgs.err
timeout -s KILL 120 python tools/trace_ctas.py tma_64x64x32_w32x16_s3_persist:4,tma_64x64x32_w32x16_s3_persist:2 1024x1024x1024,512x512x512 > gpurun_out/r02_trace_persist.jsonl 2> gpurun_out/r02_trace_persist.err
tail -4 gpurun_out/r02_trace_persist.err | cut -c1-500
