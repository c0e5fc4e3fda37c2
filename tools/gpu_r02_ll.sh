#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "1024" > gpurun_out/pytest_ll.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ll.log | cut -c1-300
timeout 300 python tools/kprof.py depth 5 1024 2>&1 | grep -E "lstm1024|ms/step"
timeout 600 python bench.py --config serx101_1024 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ll_serx.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ll_serx.json')); print('serx101_1024', round(d['value']), d['ms_per_step'])"
