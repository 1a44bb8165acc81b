# E=8 split instance at 70 registers (3 CTAs/SM) and forced-occupancy variants: parity subset + timings
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "every_cfg or all_cfgs or split_k or edge_shapes or ring_slot or hybrid_every" > gpurun_out/r02_g44_tests.txt 2>&1
echo tests rc=$?
tail -2 gpurun_out/r02_g44_tests.txt
S=plan,tma_32x64x32_w16x16_s3,tma_32x64x32_w16x16_s3_mb3,tma_32x64x32_w16x16_s3_hybrid,tma_32x64x32_w16x16_s3_streamk
for c in tma_32x64x32_w16x16_s3_splitk tma_32x64x32_w16x16_s3_splitk_mb3 tma_32x64x32_w16x16_s2_splitk_mb3 tma_32x64x64_w16x16_s3_splitk tma_32x32x32_w16x16_s4_splitk; do
  for s in 1 2 3 4; do S=$S,$c:$s; done
done
timeout -s KILL 900 python tools/cfg_time.py $S 256,384,512,640,768,896,1024,1280,1536,2048,3072 > gpurun_out/r02_g44_small.jsonl 2> gpurun_out/r02_g44_small.err
