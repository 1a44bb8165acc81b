set -x
timeout -s KILL 120 python tools/trace_ctas.py tma_64x64x32_w32x16_s3_splitk:4,tma_64x64x16_w32x16_s6_splitk:4 1024x1024x1024 > gpurun_out/r02_trace_fill.jsonl 2> gpurun_out/r02_trace_fill.err
