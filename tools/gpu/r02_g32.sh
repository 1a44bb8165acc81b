set -x
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_md2_tests.txt 2>&1
echo tests rc=$?
tail -3 gpurun_out/r02_md2_tests.txt
for md in 1 0; do
GEMM_TMA_MD=$md timeout -s KILL 600 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_splitk:1,tma_64x64x32_w32x16_s3_hybrid 1024,2048,3072,4096,6144,8192,12288,16384,32768x4096x4096,8192x4096x4096 > gpurun_out/r02_md2_cfgs_$md.jsonl 2> gpurun_out/r02_md2_cfgs_$md.err
done
