set -x
python tools/trace_ctas.py tma_64x64x32_w32x16_s3_splitk:4,tma_64x64x32_w32x16_s3_streamk,tma_64x64x32_w32x16_s3_splitk:2 1024x1024x1024,512x512x512 > gpurun_out/r02_trace_small.jsonl 2> gpurun_out/r02_trace_small.err
python tools/trace_ctas.py tma_64x64x32_w32x16_s3_splitk:1 16384x16384x2048,1024x1024x8192 >> gpurun_out/r02_trace_small.jsonl 2>> gpurun_out/r02_trace_small.err
tail -3 gpurun_out/r02_trace_small.err
