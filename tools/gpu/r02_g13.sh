set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster or ring_slot" > gpurun_out/r02_cluster_tests.txt 2>&1
echo rc=$?
tail -5 gpurun_out/r02_cluster_tests.txt
timeout -s KILL 300 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_csplit:2,tma_64x64x32_w32x16_s3_csplit:4,tma_64x64x32_w32x16_s3_csplit:8,tma_64x64x16_w32x16_s6_csplit:2,tma_64x64x16_w32x16_s6_csplit:4,tma_64x64x16_w32x16_s6_csplit:8,tma_128x64x32_w32x32_s3_csplit:2,tma_128x64x32_w32x32_s3_csplit:4,tma_64x64x32_w32x16_s3_splitk:4 256,384,512,640,768,1024,1536,2048,1024x1024x4096 > gpurun_out/r02_cluster_cfgs.jsonl 2> gpurun_out/r02_cluster_cfgs.err
timeout -s KILL 120 python tools/trace_ctas.py tma_64x64x32_w32x16_s3_csplit:4,tma_64x64x32_w32x16_s3_csplit:2 1024x1024x1024,512x512x512 > gpurun_out/r02_trace_cluster.jsonl 2> gpurun_out/r02_trace_cluster.err
