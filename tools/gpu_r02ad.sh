#!/bin/bash
# programmatic dependent launch: full GPU suite, then A/B (DDPPO_PDL=0/1) of the Depth and GPS steps
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ad.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ad.log
for i in 1 2; do for pdl in 0 1; do for c in depth gps; do
DDPPO_PDL=$pdl timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('pdl $pdl $c', round(d['value']), d['ms_per_step'])"
done; done; done
