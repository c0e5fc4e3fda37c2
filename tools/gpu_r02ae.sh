#!/bin/bash
# weights_prep with coalesced Wd stores + PDL after the conv prologue: parity + A/B + main-stream top kernels
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "depth or rgbd or serx or learner or layers or collect" > gpurun_out/pytest_ae.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ae.log
for i in 1 2; do for pdl in 0 1; do
DDPPO_PDL=$pdl timeout 600 python bench.py --config depth --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('pdl $pdl depth', round(d['value']), d['ms_per_step'])"
done; done
timeout 300 python tools/gaps.py depth 3 2>&1 | grep -v Warn | tail -18
