#!/bin/bash
# recurrence v2 (N=8, per-group overlap, in-warp cells): parity + GPS / Depth bench
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "gps or depth or learner or rgbd or act or collect" > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_w.log
for c in gps depth; do
timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_w_$c.json 2>gpurun_out/bench_w_$c.err; python -c "
import json; d=json.load(open('gpurun_out/bench_w_$c.json')); print('$c', round(d['value']), d['ms_per_step'], d['roofline']['achieved'], d.get('e2e',{}).get('value'))"
done
timeout 600 python tools/kprof.py gps > gpurun_out/kprof_w_gps.txt 2>&1; grep -E "gru|ms/step" gpurun_out/kprof_w_gps.txt | head -5
timeout 600 python tools/kprof.py depth > gpurun_out/kprof_w_depth.txt 2>&1; grep -E "lstm|ms/step" gpurun_out/kprof_w_depth.txt | head -5
