set -x
GEMM_F64_NO_TUNED=1 timeout -s KILL 2400 python -m paper_1706_10086_b200.tuner --shapes 256,384,512,640,768,1024,1536,2048,1024x1024x65536,16384x4096x4096,8192x4096x4096 --out gpurun_out/r02_tuned_v13.txt > gpurun_out/r02_tune_v13.log 2>&1
echo rc=$?
cat gpurun_out/r02_tuned_v13.txt
