#!/bin/bash
# bench lines (depth default + gps + rgbd), kernel table, ncu launch list + full capture of the TMA conv kernel
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_depth.json 2> gpurun_out/r02_bench_depth.err; echo "depth rc=$?"
timeout 900 python bench.py --config gps --steps 20 --warmup 5 > gpurun_out/r02_bench_gps.json 2> gpurun_out/r02_bench_gps.err; echo "gps rc=$?"
timeout 900 python bench.py --config rgbd --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_rgbd.json 2> gpurun_out/r02_bench_rgbd.err; echo "rgbd rc=$?"
timeout 900 python tools/kprof.py depth 5 > gpurun_out/r02_kprof_depth.txt 2>&1
# launch list of one depth learner step region (cold, serialised) and one full capture of tconv launches
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02_launches_depth.csv $B > gpurun_out/ncu_l.log 2>&1; echo "ncu list rc=$?"
$B > gpurun_out/plain2.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tconv -s 60 -c 12 -o gpurun_out/r02_tconv $B > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"
