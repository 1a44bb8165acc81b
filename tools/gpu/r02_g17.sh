set -x
timeout -s KILL 300 python tools/cfg_time.py plan,tma_64x128x32_w32x64_s3_streamk,tma_64x128x16_w32x64_s6_streamk,tma_128x64x32_w64x32_s3_streamk,tma_64x128x16_w32x64_s4,tma_64x128x16_w32x64_s4_splitk:2,tma_64x128x16_w32x64_s4_splitk:4 512,768,1024,1536,2048,1024x1024x4096 > gpurun_out/r02_sk64_cfgs.jsonl 2> gpurun_out/r02_sk64_cfgs.err
timeout -s KILL 120 python tools/trace_ctas.py tma_64x128x32_w32x64_s3_streamk,tma_64x128x16_w32x64_s6_streamk 1024x1024x1024,512x512x512 > gpurun_out/r02_trace_sk64.jsonl 2> gpurun_out/r02_trace_sk64.err
