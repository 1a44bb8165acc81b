# DRAM bytes and time of the bench kernel for several raster group sizes (GEMM_GROUP_M)
for g in ${GLIST:-4 8 17 32 64}; do
  export GEMM_GROUP_M=$g
  r=$(ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 --csv python tools/one_launch.py plan 16384 16384 16384 2 2>/dev/null | grep -E "dram|duration|hit_rate" | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')
  t=$(python tools/cfg_time.py plan 16384 | python -c "import sys,json; print(round(json.loads(sys.stdin.read())['tflops'],3))")
  echo "group_m=$g $r tflops=$t"
done
