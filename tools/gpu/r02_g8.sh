set -x
for c in tma_64x64x32_w32x16_s3_persist:1 tma_64x64x32_w32x16_s3_splitk:1; do
  name=${c%%:*}; sp=${c##*:}
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 3 --launch-count 1 -f -o gpurun_out/r02_ncu3072_${name} python tools/one_launch_sp.py $name 3072 3072 3072 $sp 5 > gpurun_out/r02_ncu3072_${name}.log 2>&1
done
