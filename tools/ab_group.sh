for g in 8 0; do
  if [ $g = 0 ]; then unset GEMM_GROUP_M; echo "group=auto"; else export GEMM_GROUP_M=$g; echo "group=$g"; fi
  python tools/cfg_time.py tma_64x64x16_w32x16_s6_splitk:1,tma_256x64x16_w64x32_s4_hybrid 16384,8192,4096 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['m'],d['cfg'], round(d['us'],1), round(d['tflops'],3))"
done
unset GEMM_GROUP_M
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 --csv python tools/one_launch.py plan 16384 16384 16384 2 2>&1 | grep -E "dram|duration" | awk -F'","' '{print $(NF-2), $NF}'
