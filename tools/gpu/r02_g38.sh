# small tiles (32x64 / 64x32) for small shapes: parity subset + timings
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "every_cfg or all_cfgs or split_k or edge_shapes or ring_slot or multidim" > gpurun_out/r02_g38_tests.txt 2>&1
echo tests rc=$?
tail -3 gpurun_out/r02_g38_tests.txt
S=plan
for c in tma_64x64x32_w32x16_s4_splitk tma_32x64x32_w16x32_s4_splitk tma_64x32x32_w32x16_s4_splitk tma_32x64x32_w16x16_s4_splitk tma_32x64x16_w16x32_s6_splitk; do
  for s in 1 2 3 4; do S=$S,$c:$s; done
done
timeout -s KILL 600 python tools/cfg_time.py $S 256,384,512,640,768,1024,1536,2048 > gpurun_out/r02_g38_small.jsonl 2> gpurun_out/r02_g38_small.err
timeout -s KILL 300 python tools/cfg_time.py tma_64x64x32_w32x16_s3_splitk:1,tma_32x64x32_w16x32_s4_splitk:1,tma_64x32x32_w32x16_s4_splitk:1,tma_32x64x32_w16x16_s4_splitk:1 4096,1024x2368x16384 > gpurun_out/r02_g38_rate.jsonl 2>> gpurun_out/r02_g38_small.err
