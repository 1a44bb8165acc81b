# per-CTA traces: SM distribution of the 3-CTA/SM E=8 instance at 768^3 vs 1024^3 (trace build)
set -x
timeout -s KILL 300 python tools/trace_ctas.py tma_32x64x32_w16x16_s3_splitk:1,tma_32x64x32_w16x16_s4_splitk:1,tma_32x64x32_w16x16_s2_splitk_mb3:1,tma_32x64x32_w16x16_s3_splitk:2 768x768x768,1024x1024x1024 > gpurun_out/r02_g46_trace.jsonl 2> gpurun_out/r02_g46_trace.err
cat gpurun_out/r02_g46_trace.jsonl
