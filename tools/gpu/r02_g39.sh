# small-tile family (32x64 / 64x32 / 32x32, E = 8 and 16): parity subset + timings at small and mid sizes
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "every_cfg or all_cfgs or split_k or edge_shapes or ring_slot or multidim" > gpurun_out/r02_g39_tests.txt 2>&1
echo tests rc=$?
tail -2 gpurun_out/r02_g39_tests.txt
S=plan,tma_32x64x32_w16x16_s4,tma_32x64x32_w16x16_s3
for c in tma_32x64x32_w16x16_s4_splitk tma_32x64x32_w16x16_s3_splitk tma_32x64x32_w16x16_s6_splitk tma_64x32x32_w16x16_s4_splitk tma_32x64x64_w16x16_s3_splitk tma_32x32x32_w16x16_s4_splitk; do
  for s in 1 2 3 4 6; do S=$S,$c:$s; done
done
timeout -s KILL 900 python tools/cfg_time.py $S 256,384,512,640,768,896,1024,1280,1536,2048 > gpurun_out/r02_g39_small.jsonl 2> gpurun_out/r02_g39_small.err
timeout -s KILL 300 python tools/cfg_time.py plan,tma_32x64x32_w16x16_s4,tma_32x64x32_w16x16_s3,tma_32x64x32_w16x16_s4_splitk:1,tma_32x64x64_w16x16_s3_splitk:1,tma_64x32x32_w16x16_s4_splitk:1 3072,4096,8192 > gpurun_out/r02_g39_mid.jsonl 2>> gpurun_out/r02_g39_small.err
