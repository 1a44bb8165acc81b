set -x
for c in tma_64x64x16_w32x16_s6_splitk:4 tma_64x64x16_w32x16_s6_streamk:1 tma_128x64x16_w32x16_s6_streamk:1 tma_256x64x16_w64x32_s4_hybrid:1 tma_64x64x16_w32x16_s6:1; do
  name=${c%%:*}; sp=${c##*:}
  ncu --set full --clock-control none -k regex:dgemm --launch-skip 4 --launch-count 2 -f -o gpurun_out/ncu1024_${name} python tools/one_launch_sp.py $name 1024 1024 1024 $sp 6 > /dev/null 2>&1
done
ls gpurun_out
