#!/bin/bash
# quick check after a change: the GPU suite subset for the visual agents + Depth / GPS bench lines
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_check.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_check.log
for c in ${CONFIGS:-depth gps}; do for i in 1 2; do
timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$c', round(d['value']), d['ms_per_step'])"
done; done
