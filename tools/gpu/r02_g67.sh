# vectorcall binding entry: host cost per call and eager small-GEMM loops, then the full GPU suite through it
set -x
timeout -s KILL 300 python tools/binding_overhead.py > gpurun_out/r02_binding_overhead_v2.txt 2>&1
echo rc=$?
cat gpurun_out/r02_binding_overhead_v2.txt
GEMM_NO_FAST=1 timeout -s KILL 300 python tools/binding_overhead.py > gpurun_out/r02_binding_overhead_ctypes_v2.txt 2>&1
cat gpurun_out/r02_binding_overhead_ctypes_v2.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_v12.txt 2>&1
echo tests rc=$?
tail -1 gpurun_out/r02_gpu_tests_full_v12.txt
