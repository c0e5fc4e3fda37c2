#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "depth or rgbd or serx or learner or layers or collect" > gpurun_out/pytest_af.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_af.log
timeout 600 python tools/kprof.py depth > gpurun_out/kprof_af.txt 2>&1; grep -E "weights_prep|ms/step" gpurun_out/kprof_af.txt
timeout 600 python tools/kprof.py rgbd 3 > gpurun_out/kprof_af_rgbd.txt 2>&1; grep -E "weights_prep|ms/step" gpurun_out/kprof_af_rgbd.txt
for i in 1 2; do
timeout 600 python bench.py --config depth --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('depth', round(d['value']), d['ms_per_step'])"
done
