# re-entry verification on HEAD (3-D/4-D tensor maps): GPU suite, smoke, bench, launch list, small-shape ncu
set -x
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_g34_tests.txt 2>&1
echo tests rc=$?
tail -3 gpurun_out/r02_g34_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_g34_smoke.txt 2>&1
echo smoke rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/r02_bench_n1_v3.json 2> gpurun_out/r02_bench_n1_v3.err
cat gpurun_out/r02_bench_n1_v3.json
timeout -s KILL 300 python tools/cfg_time.py plan 256,384,512,640,768,1024,1536,2048 > gpurun_out/r02_g34_small.jsonl 2> gpurun_out/r02_g34_small.err
for n in 512 1024; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 5 --launch-count 1 -f -o gpurun_out/r02_ncu_plan_$n python tools/one_launch.py plan $n $n $n 8 > gpurun_out/r02_ncu_plan_$n.log 2>&1
done
