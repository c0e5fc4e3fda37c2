#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 900 python tools/probe_fwd_planes.py 2>&1 | grep -v Warn | tail -12
for pl in 1 2; do timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --fwd-planes $pl > gpurun_out/bench_pl$pl.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_pl$pl.json')); print('planes $pl', d['value'], d['ms_per_step'])"; done
