set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster or ring_slot or persist" > gpurun_out/r02_cluster_tests.txt 2>&1
echo rc=$?
tail -2 gpurun_out/r02_cluster_tests.txt
GEMM_F64_NO_TUNED=1 timeout -s KILL 1800 python -m paper_1706_10086_b200.tuner --shapes 256,384,512,640,768,1024 --out gpurun_out/r02_tuned_small.txt > gpurun_out/r02_tune_small.log 2>&1
echo rc=$?
cat gpurun_out/r02_tuned_small.txt
