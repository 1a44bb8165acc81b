set -x
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:dgemm --csv --log-file gpurun_out/r02_small_bw.csv python tools/small_bw.py > gpurun_out/r02_small_bw.log 2>&1
echo rc=$?
timeout -s KILL 600 python tools/sustained.py --seconds 20 --out gpurun_out/r02_sustained.json > gpurun_out/r02_sustained.log 2>&1
echo rc=$?
tail -4 gpurun_out/r02_sustained.log
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split or ring_slot or cluster" > gpurun_out/r02_nanosleep_tests.txt 2>&1
tail -1 gpurun_out/r02_nanosleep_tests.txt
