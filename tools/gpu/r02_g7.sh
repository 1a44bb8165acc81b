set -x
timeout -s KILL 300 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_persist:1,tma_64x64x32_w32x16_s3_persist:2,tma_64x64x32_w32x16_s3_persist:4,tma_128x64x32_w32x16_s4_persist:1,tma_64x64x32_w32x16_s3_streamk,tma_128x64x32_w32x16_s4_streamk 256,512,1024,3072 > gpurun_out/r02_persist_cfgs_v3.jsonl 2> gpurun_out/r02_persist_cfgs_v3.err
timeout -s KILL 120 python tools/trace_ctas.py tma_64x64x32_w32x16_s3_persist:1 256x256x256,1024x1024x1024 > gpurun_out/r02_trace_persist_v3.jsonl 2> gpurun_out/r02_trace_persist_v3.err
