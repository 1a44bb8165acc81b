# ncu --set full of two forced configurations on one shape (compare stall reasons etc.)
# usage: bash tools/ncu_pair.sh M N K CFG1 CFG2 ...
M=$1; N=$2; K=$3; shift 3
for name in "$@"; do
  ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 3 --launch-count 1 -f \
      -o gpurun_out/ncu_${M}_${name} python tools/one_launch_sp.py $name $M $N $K 1 4 > /dev/null 2>&1
done
ls gpurun_out
