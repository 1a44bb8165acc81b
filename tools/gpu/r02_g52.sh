# config 3 (N=8192, alpha=1.5, beta=0.5) with the round-2 configuration set: timing grid + per-configuration ncu; per-CTA traces of the final small plans
set -x
timeout -s KILL 1200 python tools/sweep.py tune --n 8192 --out gpurun_out/r02_tune_n8192_v6.csv > gpurun_out/r02_tune_n8192_v6.log 2>&1
echo tune rc=$?
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,dram__bytes_read.sum --clock-control none -k regex:dgemm --csv --log-file gpurun_out/r02_config3_ncu_v6.csv python tools/sweep.py ncu --n 8192 > gpurun_out/r02_config3_ncu_pass_v6.log 2>&1
echo ncu rc=$?
timeout -s KILL 300 python tools/trace_ctas.py plan 512x512x512,1024x1024x1024,768x768x768 > gpurun_out/r02_trace_final_plans.jsonl 2> gpurun_out/r02_trace_final_plans.err
cat gpurun_out/r02_trace_final_plans.jsonl
