#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 900 python -m pytest tests/test_gpu_depth_layers.py -q -x -k conv2d > gpurun_out/pytest_conv.log 2>&1; echo "conv rc=$?"; tail -1 gpurun_out/pytest_conv.log
for i in 1 2; do
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_bn64.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_bn64.json')); print('bn64', d['value'], d['ms_per_step'])"
DDPPO_TCONV_BN128=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_bn128.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_bn128.json')); print('bn128', d['value'], d['ms_per_step'])"
done
