# cross-stage-prefetch (XP) split instances for the E = 8 tiles: parity subset + timings
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "every_cfg or all_cfgs or split_k or edge_shapes" > gpurun_out/r02_g53_tests.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_g53_tests.txt
S=plan
for c in tma_32x64x64_w16x16_s3_splitk tma_32x64x64_w16x16_s3_splitk_xp tma_32x64x32_w16x16_s3_splitk tma_32x64x32_w16x16_s3_splitk_xp tma_32x64x32_w16x16_s4_splitk_xp; do
  for s in 1 2 3 4; do S=$S,$c:$s; done
done
timeout -s KILL 900 python tools/cfg_time.py $S 256,384,512,640,768,1024,1280,1536,2048 > gpurun_out/r02_g53_small.jsonl 2> gpurun_out/r02_g53_small.err
timeout -s KILL 300 python tools/cfg_time.py tma_32x64x32_w16x16_s3_splitk:1,tma_32x64x32_w16x16_s3_splitk_xp:1,tma_32x64x64_w16x16_s3_splitk:1,tma_32x64x64_w16x16_s3_splitk_xp:1 32x18944x16384,4096,8192 > gpurun_out/r02_g53_rate.jsonl 2>> gpurun_out/r02_g53_small.err
