# tuned table v14: every shape of the table with the round-2 configuration set (32x64 family incl. hybrid / stream-K)
set -x
shapes=$(grep -v '^#' paper_1706_10086_b200/tuned_b200.txt | awk '{print $1"x"$2"x"$3}' | paste -sd,)
echo $shapes
GEMM_F64_NO_TUNED=1 timeout -s KILL 6000 python -m paper_1706_10086_b200.tuner --shapes $shapes --out gpurun_out/r02_tuned_v14.txt > gpurun_out/r02_tune_v14.log 2>&1
echo rc=$?
cat gpurun_out/r02_tuned_v14.txt
