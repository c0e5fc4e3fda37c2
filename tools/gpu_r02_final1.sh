#!/bin/bash
# round-2 final set, 1 GPU: default bench (Depth, configs[2]) + the other agents, reference arm, kernel
# attribution (PDL off so CUPTI durations are not inflated by early-launched waiting CTAs), launch list
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/final
timeout 900 python bench.py > gpurun_out/final/bench_depth.json 2> gpurun_out/final/bench_depth.err; echo "depth rc=$?"
for c in gps rgbd serx50 serx101 serx101_1024; do
  S=200; W=10; case $c in rgbd|serx*) S=10; W=3;; esac
  timeout 900 python bench.py --config $c --steps $S --warmup $W > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/reference_depth.json 2> gpurun_out/final/reference_depth.err; echo "ref rc=$?"
for c in depth gps rgbd; do DDPPO_PDL=0 timeout 600 python tools/kprof.py $c > gpurun_out/final/kprof_$c.txt 2>&1; done
timeout 600 python tools/gaps.py depth 3 > gpurun_out/final/gaps_depth.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/final/launches_depth.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_launch.log 2>&1; echo "ncu rc=$?"
for f in gpurun_out/final/bench_*.json gpurun_out/final/reference_depth.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d.get('value',0)), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'))"; done
