#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "depth" > gpurun_out/pytest_gn.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gn.log | cut -c1-300
for i in 1 2; do for m in 0 1; do
DDPPO_GN_SMALL=$m timeout 300 python bench.py --config depth --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('gn_small $m', round(d['value']), d['ms_per_step'])"
done; done
