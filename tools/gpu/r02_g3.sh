set -x
python tools/cfg_time.py plan,tma_128x64x32_w32x16_s4_streamk,tma_64x128x32_w16x32_s4_streamk,tma_128x64x32_w32x16_s4_splitk:1,tma_128x64x32_w32x16_s4_splitk:2,tma_128x64x32_w32x16_s4_splitk:4,tma_64x64x32_w32x16_s3_splitk:4 512,768,1024,1536,2048,1024x1024x2048,1024x1024x4096,4096 > gpurun_out/r02_small_cfgs_v2.jsonl 2> gpurun_out/r02_small_cfgs_v2.err
python tools/trace_ctas.py tma_128x64x32_w32x16_s4_streamk,tma_128x64x32_w32x16_s4_splitk:4 1024x1024x1024,512x512x512 > gpurun_out/r02_trace_small_v2.jsonl 2> gpurun_out/r02_trace_small_v2.err
tail -4 gpurun_out/r02_trace_small_v2.err
