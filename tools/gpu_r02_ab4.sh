#!/bin/bash
# A/B: N tile 128 for the deep layers' FPROP / DGRAD (DDPPO_TCONV_BN128_AUTO = 0 off / 128 / 256)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
for i in 1 2; do for m in 0 1; do
DDPPO_TCONV_BN128_AUTO=$m timeout 600 python bench.py --config depth --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('bn128auto $m', round(d['value']), d['ms_per_step'])"
done; done
for m in 0 1; do DDPPO_TCONV_BN128_AUTO=$m timeout 600 python bench.py --config rgbd --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('rgbd bn128auto $m', round(d['value']), d['ms_per_step'])"; done
