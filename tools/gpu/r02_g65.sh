# plan queries report the repacked TMA plan; published sizes incl. the ragged rect row (parity jsonl); rect sweep (r02)
set -x
GEMM_PARITY_OUT=gpurun_out/r02_parity_published_sizes_v4.jsonl timeout -s KILL 1500 python -m pytest tests/test_gpu_published_sizes.py tests/test_gpu_autotune.py tests/test_gpu_freivalds.py -m gpu -x -q > gpurun_out/r02_g65_tests.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_g65_tests.txt
timeout -s KILL 1500 python tools/sweep.py scale --shapes 32768x4096x4096,16384x4096x4096,8192x4096x4096,4096x4096x4096,1024x1024x65536,8192x65536x8192,8192x65536x65536,10000x9999x7001 --reps 5 --out gpurun_out/r02_f1_rectangular_v8.csv > gpurun_out/r02_f1_rect_v8.log 2>&1
echo sweep rc=$?
cat gpurun_out/r02_f1_rectangular_v8.csv
