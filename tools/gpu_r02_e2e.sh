#!/bin/bash
# double-buffered rollout arenas: the learner tests, then e2e vs device for Depth / RGB-D / GPS
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "learner or collect or errors" > gpurun_out/pytest_e2e.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_e2e.log
for c in depth gps; do timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/e2e_$c.json')); print('$c', round(d['value']), round(d['e2e']['value']), d['e2e']['value']/d['value'])"; done
timeout 600 python bench.py --config rgbd --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_rgbd.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/e2e_rgbd.json')); print('rgbd', round(d['value']), round(d['e2e']['value']), d['e2e']['value']/d['value'])"
