set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "max_size" --durations=5 > gpurun_out/r02_maxsize_tests.txt 2>&1
echo rc=$?
tail -12 gpurun_out/r02_maxsize_tests.txt
