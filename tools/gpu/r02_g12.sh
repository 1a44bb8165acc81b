set -x
timeout -s KILL 900 python bench.py --workload large_strong --steps 3 --warmup 3 --no-cpu-baseline --verify-rows 3 > gpurun_out/r02_bench_large_strong.json 2> gpurun_out/r02_bench_large_strong.err
echo rc=$?
timeout -s KILL 600 python bench.py --workload large --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_large.json 2> gpurun_out/r02_bench_large.err
echo rc=$?
timeout -s KILL 600 python bench.py --workload rect --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_rect.json 2> gpurun_out/r02_bench_rect.err
echo rc=$?
for f in large_strong large rect; do python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity'], d['clocks'])"; done
