set -x
timeout -s KILL 300 python tools/binding_overhead.py > gpurun_out/r02_binding_overhead.txt 2>&1
cat gpurun_out/r02_binding_overhead.txt
timeout -s KILL 300 python tools/small_overhead.py > gpurun_out/r02_small_overhead.log 2>&1
tail -12 gpurun_out/r02_small_overhead.log
