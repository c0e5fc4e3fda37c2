#!/bin/bash
# round-2 profile set (part 1): bench lines, CUPTI splits, ncu launch list (depth)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 900 python bench.py > gpurun_out/r02_bench_depth.json 2> gpurun_out/r02_bench_depth.err; echo "depth rc=$?"
timeout 900 python bench.py --config gps > gpurun_out/r02_bench_gps.json 2> gpurun_out/r02_bench_gps.err; echo "gps rc=$?"
timeout 900 python bench.py --config rgbd --steps 10 --warmup 3 > gpurun_out/r02_bench_rgbd.json 2> gpurun_out/r02_bench_rgbd.err; echo "rgbd rc=$?"
timeout 900 python bench.py --config serx50 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_serx50.json 2> gpurun_out/r02_bench_serx50.err; echo "serx rc=$?"
for c in depth gps rgbd; do timeout 600 python tools/kprof.py $c 5 > gpurun_out/r02_kprof_$c.txt 2>&1; done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_depth.csv $B > gpurun_out/ncu_l.log 2>&1; echo "ncu list rc=$?"
du -sh gpurun_out
