set -x
timeout -s KILL 900 python tools/ab_libs.py paper_1706_10086_b200/libgemm_f64_r01.so paper_1706_10086_b200/libgemm_f64.so 16384x16384x16384,8192x8192x8192,4096x4096x4096,1024x1024x1024 5 > gpurun_out/r02_ab_r01_vs_now.jsonl 2>&1
cat gpurun_out/r02_ab_r01_vs_now.jsonl | cut -c1-200
