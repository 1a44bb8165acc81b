# lone-CTA vs two-CTA steady-state DMMA rate of the 64x64 instances (XP split instance, deeper rings)
set -x
C=tma_64x64x32_w32x16_s3_splitk:1,tma_64x64x32_w32x16_s3_splitk_xp:1,tma_64x64x32_w32x16_s4_splitk:1,tma_64x64x32_w32x16_s6_splitk_xp:1,tma_64x64x32_w16x32_s4_splitk_xp:1,tma_64x64x32_w16x32_s3,tma_64x64x16_w32x16_s6_xp
timeout -s KILL 600 python tools/cfg_time.py $C 64x9472x16384,64x18944x16384,128x9472x16384 > gpurun_out/r02_g35_lone.jsonl 2> gpurun_out/r02_g35_lone.err
S=plan
for c in tma_64x64x32_w32x16_s3_splitk tma_64x64x32_w32x16_s3_splitk_xp tma_64x64x32_w32x16_s4_splitk tma_64x64x32_w32x16_s6_splitk_xp tma_64x64x32_w16x32_s4_splitk_xp; do
  for s in 1 2 3 4 6 8; do S=$S,$c:$s; done
done
timeout -s KILL 900 python tools/cfg_time.py $S 384,512,640,768,1024,1536 > gpurun_out/r02_g35_small.jsonl 2> gpurun_out/r02_g35_small.err
