# tuned table v15 rows for the small and mid shapes (E = 8 split instance now 70 registers -> 3 CTAs/SM)
set -x
GEMM_F64_NO_TUNED=1 timeout -s KILL 3000 python -m paper_1706_10086_b200.tuner --shapes 256,384,512,640,768,1024,1536,2048,3072,4096,5120,6144,8192x4096x4096,1024x1024x65536 --out gpurun_out/r02_tuned_v15_small.txt > gpurun_out/r02_tune_v15_small.log 2>&1
echo rc=$?
cat gpurun_out/r02_tuned_v15_small.txt
