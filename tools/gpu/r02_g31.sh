set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_freivalds.py -m gpu -x -q > gpurun_out/r02_md_tests.txt 2>&1
echo tests rc=$?
tail -3 gpurun_out/r02_md_tests.txt
for md in 1 0; do
GEMM_TMA_MD=$md timeout -s KILL 600 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s3_splitk:1,tma_64x64x16_w32x16_s6_splitk:1 512,768,1024,2048,4096,8192,16384 > gpurun_out/r02_md_cfgs_$md.jsonl 2> gpurun_out/r02_md_cfgs_$md.err
done
timeout -s KILL 120 python tools/trace_ctas.py tma_64x64x32_w32x16_s3_splitk:4 1024x1024x1024 > gpurun_out/r02_trace_md.jsonl 2> gpurun_out/r02_trace_md.err
