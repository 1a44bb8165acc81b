# pair stream-K kernel (two coupled 8-warp groups per CTA, one CTA per SM): parity subset + timings
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "every_cfg or all_cfgs or stream_k or edge_shapes or ring_slot or multidim" > gpurun_out/r02_g36_tests.txt 2>&1
echo tests rc=$?
tail -5 gpurun_out/r02_g36_tests.txt
P=plan,tma_64x64x32_w32x16_s6_pairsk,tma_64x64x32_w32x16_s4_pairsk,tma_64x64x16_w32x16_s8_pairsk,tma_64x64x32_w32x16_s3_streamk,tma_64x64x32_w32x16_s4_splitk:2,tma_64x64x32_w32x16_s4_splitk:4
timeout -s KILL 600 python tools/cfg_time.py $P 256,384,512,640,768,1024,1280,1536,2048,3072,4096,1024x1024x4096,256x2368x16384 > gpurun_out/r02_g36_pair.jsonl 2> gpurun_out/r02_g36_pair.err
