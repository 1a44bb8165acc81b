set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_streamk,tma_64x64x32_w16x32_s3_streamk,tma_128x64x32_w32x32_s3_streamk,tma_64x64x16_w32x16_s6_streamk,tma_128x64x16_w32x16_s6_streamk,tma_64x64x32_w32x16_s3_splitk:2,tma_64x64x32_w32x16_s3_splitk:4,tma_128x64x32_w32x32_s3_splitk:2,tma_128x64x32_w32x32_s3_splitk:4,tma_128x64x32_w32x32_s3_splitk:8 256,384,512,640,768,1024,1536,2048,1024x1024x2048,1024x1024x4096 > gpurun_out/r02_small_cfgs.jsonl 2> gpurun_out/r02_small_cfgs.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests.txt 2>&1
tail -5 gpurun_out/r02_gpu_tests.txt
